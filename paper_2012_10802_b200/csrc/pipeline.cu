// pipeline.cu — detect_potholes_pipeline (pipeline.cpp:47-109) on the device.
//
// The whole frame — bootstrap SGM at half resolution, road fit, PT SGM, road
// refit, disparity transform, SLIC + pooling, histogram/threshold and
// labelling — is enqueued on the context stream with no host synchronisation;
// the only host<->device traffic is the image upload and the result download.
// After the first (eager) run of a given (H, W, config, input type) the device
// part is captured into a CUDA graph and replayed on later calls.  Stage times
// come from CUDA events recorded between the stages (StageClock names,
// pipeline.cpp:64-104).
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <vector>

#include "abi_util.hpp"
#include "road.cuh"
#include "seg.cuh"
#include <cstdlib>

#include "sgm.cuh"

namespace rpdg {

namespace {

constexpr long long kPipelineObsCap = 100000;  // sample_observations cap (pipeline.cpp:66, :81)

struct FrameBuffers {
  float* left;
  float* right;
  uint8_t* left8;
  uint8_t* right8;
  float* hl;
  float* hr;
  float* b_d0;
  float* b_d1;
  double* b_shifts;
  float* d0;
  float* d1;
  double* shifts;
  float* d2;
  float* d3;
  int32_t* labels;
  int* n_potholes;
  FitOut* coarse;
  FitOut* fit;
  rpd_threshold* thr;
  unsigned long long* clamped;
  DevModel* flat;
  ObsBuffers obs;
  SlicOut sp;
  struct FrameScalars* scal;  // every scalar output + the status, one D2H copy
};

// The frame's scalar results gathered on the device at the end of the graph,
// so rpd_detect_fetch reads them (and the status word) with ONE small copy
// instead of seven.
struct FrameScalars {
  FitOut coarse, fit;
  rpd_threshold thr;
  unsigned long long clamped;
  int count, npot;
  DevStatus status;
};

__global__ void k_gather_scalars(const FitOut* coarse, const FitOut* fit, const rpd_threshold* thr,
                                 const unsigned long long* clamped, const int* count,
                                 const int* npot, const DevStatus* status, FrameScalars* out) {
  out->coarse = *coarse;
  out->fit = *fit;
  out->thr = *thr;
  out->clamped = *clamped;
  out->count = *count;
  out->npot = *npot;
  out->status = *status;
}

struct GraphKey {
  int h, w, u8, profile;
  rpd_config cfg;
  bool operator<(const GraphKey& o) const {
    return std::memcmp(this, &o, sizeof(GraphKey)) < 0;
  }
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  unsigned generation = 0;
  int kernels = 0;
  FrameBuffers fb{};
};

struct PipelineState {
  std::map<GraphKey, GraphEntry> graphs;
  FrameBuffers last{};
  bool have_last = false;
  int last_h = 0, last_w = 0;
};

PipelineState& state(rpd_ctx* ctx) {
  if (!ctx->pipeline) ctx->pipeline = new PipelineState();
  return *static_cast<PipelineState*>(ctx->pipeline);
}

__global__ void k_flat_model(DevModel* m) { *m = DevModel{0.0, 0.0, 0.0, 1.0, 0.0}; }

// Stage event: inside a stream capture it must become an external event-record
// node (a plain record would only act as a capture-internal dependency).
void record_stage(rpd_ctx* ctx, int i) { record_event(ctx, ctx->ev[i]); }

int count_kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  RPD_CK(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) RPD_CK(cudaGraphGetNodes(g, nodes.data(), &n));
  int k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    RPD_CK(cudaGraphNodeGetType(nd, &t));
    if (t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

FrameBuffers alloc_frame(rpd_ctx* ctx, int h, int w, int K) {
  const size_t n = size_t(h) * w;
  const size_t hn = size_t(h / 2) * (w / 2);
  FrameBuffers f{};
  Workspace& ws = ctx->ws;
  f.scal = ws.get<FrameScalars>("pl_scalars", 1);
  f.left = ws.get<float>("pl_left", n);
  f.right = ws.get<float>("pl_right", n);
  f.left8 = ws.get<uint8_t>("pl_left8", n);
  f.right8 = ws.get<uint8_t>("pl_right8", n);
  f.hl = ws.get<float>("pl_hl", std::max<size_t>(hn, 1));
  f.hr = ws.get<float>("pl_hr", std::max<size_t>(hn, 1));
  f.b_d0 = ws.get<float>("pl_bd0", n);
  f.b_d1 = ws.get<float>("pl_bd1", n);
  f.b_shifts = ws.get<double>("pl_bshifts", h);
  f.d0 = ws.get<float>("pl_d0", n);
  f.d1 = ws.get<float>("pl_d1", n);
  f.shifts = ws.get<double>("pl_shifts", h);
  f.d2 = ws.get<float>("pl_d2", n);
  f.d3 = ws.get<float>("pl_d3", n);
  f.labels = ws.get<int32_t>("pl_labels", n);
  f.n_potholes = ws.get<int>("pl_npot", 1);
  f.coarse = ws.get<FitOut>("pl_coarse", 1);
  f.fit = ws.get<FitOut>("pl_fit", 1);
  f.thr = ws.get<rpd_threshold>("pl_thr", 1);
  f.clamped = ws.get<unsigned long long>("pl_clamped", 1);
  f.flat = ws.get<DevModel>("pl_flat", 1);
  f.obs.uv = ws.get<uint32_t>("pl_obs_uv", kPipelineObsCap);
  f.obs.d = ws.get<float>("pl_obs_d", kPipelineObsCap);
  f.obs.count = ws.get<int>("pl_obs_count", 1);
  (void)K;
  return f;
}

// Enqueues the device part of one frame (everything after the upload).
// Debugging / cost attribution only (RPD_SKIP_STAGES bitmask, results are
// garbage): 1 = road fits, 2 = SLIC + pooling + detection, 4 = detection,
// 8 = bootstrap SGM, 16 = PT SGM.
int skip_stages() {
  static const int m = [] {
    const char* e = debug_knob("RPD_SKIP_STAGES");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}
// Marginal-cost attribution (RPD_DUP_STAGES, same bits): the stage is enqueued
// twice (idempotent: same inputs, same outputs), so the throughput drop is
// the stage's cost in the concurrent regime.
int dup_stages() {
  static const int m = [] {
    const char* e = debug_knob("RPD_DUP_STAGES");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

void enqueue_frame_body(rpd_ctx* ctx, FrameBuffers& f, int h, int w, bool u8,
                        const rpd_config& c);

void enqueue_frame(rpd_ctx* ctx, FrameBuffers& f, int h, int w, bool u8, const rpd_config& c) {
  enqueue_frame_body(ctx, f, h, w, u8, c);
  k_gather_scalars<<<1, 1, 0, ctx->stream>>>(f.coarse, f.fit, f.thr, f.clamped, f.sp.count,
                                             f.n_potholes, ctx->status, f.scal);
  RPD_LAUNCH_CHECK();
}

void enqueue_frame_body(rpd_ctx* ctx, FrameBuffers& f, int h, int w, bool u8,
                        const rpd_config& c) {
  cudaStream_t st = ctx->stream;
  const int skip = skip_stages();
  const int dup = dup_stages();
  const long long n = (long long)h * w;
  reset_status(ctx);
  ctx->agg_pass = 0;
  record_stage(ctx, 0);
  if (u8) {
    launch_u8_to_f32(f.left8, f.left, n, st, f.right8, f.right);
  }
  k_flat_model<<<1, 1, 0, st>>>(f.flat);
  RPD_LAUNCH_CHECK();
  // pipeline.cpp:57-63 bootstrap with a flat model, half resolution if >= 64
  const bool halve = h >= 64 && w >= 64;
  int bh = h, bw = w;
  if (halve) {
    bh = h / 2;
    bw = w / 2;
    launch_half_image(f.left, h, w, f.hl, st, f.right, f.hr);
    rpd_config boot = c;
    boot.d_max = (c.d_max + 1) / 2;
    for (int rep = 0; rep < ((dup & 8) ? 2 : 1) && !(skip & 8); ++rep)
      match_pair_dev(ctx, f.hl, f.hr, bh, bw, f.flat, boot, boot.d_max, f.b_d0, f.b_d1,
                     f.b_shifts);
  } else {
    match_pair_dev(ctx, f.left, f.right, h, w, f.flat, c, c.d_max, f.b_d0, f.b_d1, f.b_shifts);
  }
  record_stage(ctx, 1);
  // pipeline.cpp:66-73 coarse road fit (a0 *= 2 when halved)
  if (!(skip & 1))
    sample_observations_dev(ctx, f.b_d1, bh, bw, nullptr, kPipelineObsCap, f.obs,
                            kWhereSampleBoot);
  FitRequest fr;
  fr.mode = kFitRoad;
  fr.compact = true;
  fr.obs = f.obs;
  fr.kmax = kPipelineObsCap;
  fr.hi = c.roll_bracket;
  fr.tol = c.roll_tol;
  fr.a0_scale = halve ? 2.0 : 1.0;
  fr.where = kWhereFitBoot;
  fr.out = f.coarse;
  if (!(skip & 1)) fit_dev(ctx, fr);
  record_stage(ctx, 2);
  // pipeline.cpp:76 PT pass
  for (int rep = 0; rep < ((dup & 16) ? 2 : 1) && !(skip & 16); ++rep)
    match_pair_dev(ctx, f.left, f.right, h, w, &f.coarse->model, c, c.d_max_pt, f.d0, f.d1,
                   f.shifts);
  record_stage(ctx, 3);
  // pipeline.cpp:81-86 refit
  if (!(skip & 1))
    sample_observations_dev(ctx, f.d1, h, w, nullptr, kPipelineObsCap, f.obs, kWhereSamplePt);
  fr.a0_scale = 1.0;
  fr.where = kWhereFitPt;
  fr.out = f.fit;
  if (!(skip & 1)) fit_dev(ctx, fr);
  if (dup & 1) fit_dev(ctx, fr);
  record_stage(ctx, 4);
  // pipeline.cpp:89-91 disparity transformation
  RPD_CK(cudaMemsetAsync(f.clamped, 0, sizeof(unsigned long long), st));
  transform_disparity_dev(f.d1, h, w, &f.fit->model, c.delta_dt, f.d2, f.clamped, st);
  record_stage(ctx, 5);
  // pipeline.cpp:94-96 SLIC + pooling
  if (skip & 2) {
    f.sp.labels = f.labels;  // valid device buffers for the fetch
    f.sp.count = f.n_potholes;
    f.sp.centers = nullptr;
    record_stage(ctx, 6);
    record_stage(ctx, 7);
    return;
  }
  // slic + pool_superpixels (the pooling shares slic's final label pass)
  f.sp = slic_dev(ctx, f.d2, h, w, c.superpixels, c.compactness, c.slic_iterations, f.d3);
  if (dup & 2)
    f.sp = slic_dev(ctx, f.d2, h, w, c.superpixels, c.compactness, c.slic_iterations, f.d3);
  record_stage(ctx, 6);
  if (skip & 4) {
    record_stage(ctx, 7);
    return;
  }
  // pipeline.cpp:99-103 histogram, threshold, labelling
  const HistDev hd = build_histogram_dev(ctx, f.d2, h, w, c.hist_bin_width, c.tau_diag);
  find_threshold_dev(ctx, hd, c.hist_bin_width, c.delta_pd, c.tau_diag, f.thr,
                     kWhereThresholdEmpty);
  for (int rep = 0; rep < ((dup & 4) ? 2 : 1); ++rep)
    detect_potholes_dev(ctx, f.d3, f.sp.labels, f.sp.spacing, h, w, f.thr, c.border_margin,
                        c.min_superpixels, c.connectivity, f.labels, f.n_potholes);
  record_stage(ctx, 7);
}

// Runs one frame from device-resident inputs already in f.left/right (or
// f.left8/right8), replaying a captured graph when one matches.
void run_frame(rpd_ctx* ctx, int h, int w, bool u8, const rpd_config& c, FrameBuffers& out) {
  PipelineState& ps = state(ctx);
  GraphKey key;
  std::memset(&key, 0, sizeof(key));
  key.h = h;
  key.w = w;
  key.u8 = u8 ? 1 : 0;
  key.profile = ctx->profile ? 1 : 0;
  key.cfg = c;
  auto it = ps.graphs.find(key);
  if (it != ps.graphs.end() && it->second.exec && it->second.generation == ctx->ws.generation()) {
    RPD_CK(cudaGraphLaunch(it->second.exec, ctx->stream));
    out = it->second.fb;
    ctx->graph_replayed = 1;
    ctx->kernels_last_frame = it->second.kernels;
    return;
  }
  // eager run (allocates every workspace buffer)
  const unsigned gen0 = ctx->ws.generation();
  FrameBuffers f = alloc_frame(ctx, h, w, 0);
  enqueue_frame(ctx, f, h, w, u8, c);
  out = f;
  ctx->graph_replayed = 0;
  if (ctx->ws.generation() != gen0) return;  // buffers moved: capture next time
  // capture for the next call with the same key
  cudaGraph_t g = nullptr;
  FrameBuffers fg = f;
  RPD_CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  bool ok = true;
  try {
    enqueue_frame(ctx, fg, h, w, u8, c);
  } catch (...) {
    ok = false;
  }
  const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &g);
  if (!ok || ec != cudaSuccess || !g || ctx->ws.generation() != gen0) {
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    return;
  }
  const int kernels = count_kernel_nodes(g);
  ctx->kernels_last_frame = kernels;
  cudaGraphExec_t exec = nullptr;
  if (cudaGraphInstantiate(&exec, g, 0) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    return;
  }
  cudaGraphDestroy(g);
  GraphEntry& e = ps.graphs[key];
  if (e.exec) cudaGraphExecDestroy(e.exec);
  e.exec = exec;
  e.kernels = kernels;
  e.generation = ctx->ws.generation();
  e.fb = fg;
}

void fetch(rpd_ctx* ctx, const FrameBuffers& f, int h, int w, rpd_detect_out* out) {
  cudaStream_t st = ctx->stream;
  const size_t n = size_t(h) * w;
  // cudaMemcpyDefault: an output may be host memory or device memory of this
  // GPU (device-resident consumers take a device-to-device copy)
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    if (dst && bytes) RPD_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
  };
  d2h(out->d0, f.d0, sizeof(float) * n);
  d2h(out->d1, f.d1, sizeof(float) * n);
  d2h(out->d2, f.d2, sizeof(float) * n);
  d2h(out->d3, f.d3, sizeof(float) * n);
  d2h(out->labels, f.labels, sizeof(int32_t) * n);
  d2h(out->sp_labels, f.sp.labels, sizeof(int32_t) * n);
  FrameScalars* hs = static_cast<FrameScalars*>(ctx->pinned.get(sizeof(FrameScalars)));
  RPD_CK(cudaMemcpyAsync(hs, f.scal, sizeof(FrameScalars), cudaMemcpyDeviceToHost, st));
  RPD_CK(cudaStreamSynchronize(st));
  check_status(hs->status);
  const int count = hs->count;
  if (out->centers && out->centers_cap > 0 && count > 0) {
    const int m = std::min(out->centers_cap, count);
    RPD_CK(cudaMemcpyAsync(out->centers, f.sp.centers, sizeof(double) * 3 * size_t(m),
                           cudaMemcpyDefault, st));
    RPD_CK(cudaStreamSynchronize(st));
  }
  out->sp_count = count;
  out->sp_spacing = f.sp.spacing;
  auto to_fit = [](const FitOut& x) {
    rpd_road_fit r;
    r.model = rpd_road_model{x.a0, x.a1, x.phi};
    r.e0min = x.e0min;
    r.used = x.used;
    return r;
  };
  out->coarse_fit = to_fit(hs->coarse);
  out->fit = to_fit(hs->fit);
  out->threshold = hs->thr;
  out->clamped = (int64_t)hs->clamped;
  out->n_potholes = hs->npot;
  float ms[RPD_NUM_STAGES];
  for (int i = 0; i < RPD_NUM_STAGES; ++i) {
    RPD_CK(cudaEventElapsedTime(&ms[i], ctx->ev[i], ctx->ev[i + 1]));
    out->stage_ms[i] = ms[i];
  }
  float tot = 0;
  RPD_CK(cudaEventElapsedTime(&tot, ctx->ev[0], ctx->ev[RPD_NUM_STAGES]));
  out->total_ms = tot;
}

void check_pipeline_args(const rpd_config* cfg, int h, int w) {
  if (!cfg) throw InvalidArg("config: null");
  config_validate(*cfg);
  check_dims(h, w);
  if (h >= 65536 || w >= 65536) throw InvalidArg("detect: image side must be < 65536");
}

}  // namespace

}  // namespace rpdg

using namespace rpdg;

extern "C" {

rpd_status rpd_detect(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                      const rpd_config* cfg, rpd_detect_out* out) {
  return guard(ctx, [&] {
    check_pipeline_args(cfg, h, w);
    const size_t n = size_t(h) * w;
    float* l = ctx->ws.get<float>("pl_left", n);
    float* r = ctx->ws.get<float>("pl_right", n);
    RPD_CK(cudaMemcpyAsync(l, left, sizeof(float) * n, cudaMemcpyDefault, ctx->stream));
    RPD_CK(cudaMemcpyAsync(r, right, sizeof(float) * n, cudaMemcpyDefault, ctx->stream));
    FrameBuffers f;
    run_frame(ctx, h, w, false, *cfg, f);
    fetch(ctx, f, h, w, out);
  });
}

rpd_status rpd_detect_u8(rpd_ctx* ctx, const uint8_t* left, const uint8_t* right, int h, int w,
                         const rpd_config* cfg, rpd_detect_out* out) {
  return guard(ctx, [&] {
    check_pipeline_args(cfg, h, w);
    const size_t n = size_t(h) * w;
    uint8_t* l = ctx->ws.get<uint8_t>("pl_left8", n);
    uint8_t* r = ctx->ws.get<uint8_t>("pl_right8", n);
    RPD_CK(cudaMemcpyAsync(l, left, n, cudaMemcpyDefault, ctx->stream));
    RPD_CK(cudaMemcpyAsync(r, right, n, cudaMemcpyDefault, ctx->stream));
    FrameBuffers f;
    run_frame(ctx, h, w, true, *cfg, f);
    fetch(ctx, f, h, w, out);
  });
}

rpd_status rpd_detect_async_u8(rpd_ctx* ctx, const uint8_t* d_left, const uint8_t* d_right, int h,
                               int w, const rpd_config* cfg) {
  return guard(ctx, [&] {
    check_pipeline_args(cfg, h, w);
    const size_t n = size_t(h) * w;
    uint8_t* l = ctx->ws.get<uint8_t>("pl_left8", n);
    uint8_t* r = ctx->ws.get<uint8_t>("pl_right8", n);
    if (d_left != l)
      RPD_CK(cudaMemcpyAsync(l, d_left, n, cudaMemcpyDeviceToDevice, ctx->stream));
    if (d_right != r)
      RPD_CK(cudaMemcpyAsync(r, d_right, n, cudaMemcpyDeviceToDevice, ctx->stream));
    PipelineState& ps = state(ctx);
    run_frame(ctx, h, w, true, *cfg, ps.last);
    ps.have_last = true;
    ps.last_h = h;
    ps.last_w = w;
  });
}

rpd_status rpd_detect_async(rpd_ctx* ctx, const float* d_left, const float* d_right, int h, int w,
                            const rpd_config* cfg) {
  return guard(ctx, [&] {
    check_pipeline_args(cfg, h, w);
    const size_t n = size_t(h) * w;
    float* l = ctx->ws.get<float>("pl_left", n);
    float* r = ctx->ws.get<float>("pl_right", n);
    if (d_left != l)
      RPD_CK(cudaMemcpyAsync(l, d_left, sizeof(float) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    if (d_right != r)
      RPD_CK(cudaMemcpyAsync(r, d_right, sizeof(float) * n, cudaMemcpyDeviceToDevice,
                             ctx->stream));
    PipelineState& ps = state(ctx);
    run_frame(ctx, h, w, false, *cfg, ps.last);
    ps.have_last = true;
    ps.last_h = h;
    ps.last_w = w;
  });
}

rpd_status rpd_detect_async_host_u8(rpd_ctx* ctx, const uint8_t* left, const uint8_t* right,
                                    int h, int w, const rpd_config* cfg) {
  return guard(ctx, [&] {
    check_pipeline_args(cfg, h, w);
    const size_t n = size_t(h) * w;
    uint8_t* l = ctx->ws.get<uint8_t>("pl_left8", n);
    uint8_t* r = ctx->ws.get<uint8_t>("pl_right8", n);
    // asynchronous (DMA) when the host buffers are pinned (rpd_host_alloc)
    RPD_CK(cudaMemcpyAsync(l, left, n, cudaMemcpyDefault, ctx->stream));
    RPD_CK(cudaMemcpyAsync(r, right, n, cudaMemcpyDefault, ctx->stream));
    PipelineState& ps = state(ctx);
    run_frame(ctx, h, w, true, *cfg, ps.last);
    ps.have_last = true;
    ps.last_h = h;
    ps.last_w = w;
  });
}

rpd_status rpd_host_alloc(size_t bytes, void** out) {
  if (!out) return RPD_EINVAL;
  *out = nullptr;
  if (cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return RPD_ENOMEM;
  }
  return RPD_OK;
}

void rpd_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

rpd_status rpd_detect_fetch(rpd_ctx* ctx, rpd_detect_out* out) {
  return guard(ctx, [&] {
    PipelineState& ps = state(ctx);
    if (!ps.have_last) throw InvalidArg("rpd_detect_fetch: no frame in flight");
    fetch(ctx, ps.last, ps.last_h, ps.last_w, out);
  });
}

rpd_status rpd_input_buffers_u8(rpd_ctx* ctx, int h, int w, uint8_t** d_left, uint8_t** d_right) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    *d_left = ctx->ws.get<uint8_t>("pl_left8", n);
    *d_right = ctx->ws.get<uint8_t>("pl_right8", n);
  });
}

}  // extern "C"

namespace rpdg {
void pipeline_forget(rpd_ctx* ctx) {
  if (!ctx->pipeline) return;
  PipelineState* ps = static_cast<PipelineState*>(ctx->pipeline);
  for (auto& kv : ps->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  delete ps;
  ctx->pipeline = nullptr;
}
}  // namespace rpdg
