// abi_core.cu — context lifecycle, config and the SGM / perspective entry
// points of the C-ABI (include/rpd_b200.h).  Host buffers are copied to
// context-owned device workspaces; all device work is ordered on ctx->stream.
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "abi_util.hpp"
#include "sgm.cuh"

namespace rpdg {

bool rpd_sync_debug() {
  static const bool on = [] {
    const char* e = debug_knob("RPD_SYNC_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}

void reset_status(rpd_ctx* ctx) {
  RPD_CK(cudaMemsetAsync(ctx->status, 0, sizeof(DevStatus), ctx->stream));
}

static const char* status_message(int where) {
  switch (where) {
    case kWhereSampleBoot: return "road fit failed: sample_observations: fewer than 3 valid pixels";
    case kWhereFitBoot:
      return "road fit failed: fit_line: degenerate observations (singular normal matrix)";
    case kWhereSamplePt:
      return "road refit failed: sample_observations: fewer than 3 valid pixels";
    case kWhereFitPt:
      return "road refit failed: fit_line: degenerate observations (singular normal matrix)";
    case kWhereThresholdEmpty: return "find_road_threshold: all vectors excluded";
    case kWhereHistTooLarge: return "build_histogram: histogram too large for the device band";
    case kWhereSample: return "sample_observations: fewer than 3 valid pixels";
    case kWhereFit: return "fit_line: degenerate observations (singular normal matrix)";
    default: return "device failure";
  }
}

void record_event(rpd_ctx* ctx, cudaEvent_t ev) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  RPD_CK(cudaStreamIsCapturing(ctx->stream, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    RPD_CK(cudaEventRecordWithFlags(ev, ctx->stream, cudaEventRecordExternal));
  else
    RPD_CK(cudaEventRecord(ev, ctx->stream));
}

void sync_and_check(rpd_ctx* ctx) {
  DevStatus h{};
  RPD_CK(cudaMemcpyAsync(&h, ctx->status, sizeof(DevStatus), cudaMemcpyDeviceToHost,
                         ctx->stream));
  RPD_CK(cudaStreamSynchronize(ctx->stream));
  check_status(h);
}

void check_status(const DevStatus& h) {
  if (h.code == RPD_EDEGENERATE) throw Degenerate(status_message(h.where));
  if (h.code == RPD_EINVAL) throw InvalidArg(status_message(h.where));
  if (h.code == RPD_ENOMEM) throw CudaFail(status_message(h.where));
  if (h.code != 0) throw CudaFail(status_message(h.where));
}

}  // namespace rpdg

using namespace rpdg;

extern "C" {

int rpd_abi_version(void) { return RPD_ABI_VERSION; }

rpd_status rpd_ctx_create(int device, int, int, int, rpd_ctx** out) {
  if (!out) return RPD_EINVAL;
  *out = nullptr;
  rpd_ctx* ctx = new (std::nothrow) rpd_ctx();
  if (!ctx) return RPD_ENOMEM;
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->status, sizeof(DevStatus));
  if (e == cudaSuccess) e = cudaMemset(ctx->status, 0, sizeof(DevStatus));
  for (int i = 0; e == cudaSuccess && i <= RPD_NUM_STAGES; ++i) e = cudaEventCreate(&ctx->ev[i]);
  for (int i = 0; e == cudaSuccess && i < 4; ++i) e = cudaEventCreate(&ctx->agg_ev[i / 2][i % 2]);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount,
                                                   device);
  int major = 0;
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (e != cudaSuccess) {
    cudaGetLastError();
    rpd_ctx_destroy(ctx);
    return RPD_ECUDA;
  }
  if (major < 10) {  // built for sm_100a only
    rpd_ctx_destroy(ctx);
    return RPD_ECUDA;
  }
  *out = ctx;
  return RPD_OK;
}

void rpd_ctx_destroy(rpd_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  pipeline_forget(ctx);
  ctx->ws.release();
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& pr : ctx->agg_ev)
    for (auto& e : pr)
      if (e) cudaEventDestroy(e);
  if (ctx->status) cudaFree(ctx->status);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* rpd_last_error(const rpd_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

void* rpd_ctx_stream(rpd_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

rpd_status rpd_ctx_set_profiling(rpd_ctx* ctx, int enable) {
  return guard(ctx, [&] { ctx->profile = enable != 0; });
}

namespace {
__global__ void k_poke(unsigned char* p, size_t off) { p[off] = 0; }
}  // namespace

// Self-test of the guard mechanism (checked build): writes one byte just past
// a fresh workspace buffer; rpd_debug_guard_check must then report it.
rpd_status rpd_debug_guard_selftest(rpd_ctx* ctx, size_t bytes) {
  return guard(ctx, [&] {
#ifdef RPD_DEBUG_KNOBS
    unsigned char* p = ctx->ws.get<unsigned char>("guard_selftest", bytes);
    k_poke<<<1, 1, 0, ctx->stream>>>(p, bytes);
    RPD_LAUNCH_CHECK();
#else
    (void)bytes;
    throw InvalidArg("guard self-test: checked build only");
#endif
  });
}

rpd_status rpd_debug_guard_check(rpd_ctx* ctx, long long* corrupted, char* first, int cap) {
  return guard(ctx, [&] {
    RPD_CK(cudaStreamSynchronize(ctx->stream));
    std::string who;
    *corrupted = ctx->ws.check_guards(&who);
    if (first && cap > 0) {
      std::strncpy(first, who.c_str(), size_t(cap - 1));
      first[cap - 1] = 0;
    }
  });
}

rpd_status rpd_ctx_stats(rpd_ctx* ctx, rpd_stats* out) {
  return guard(ctx, [&] {
    RPD_CK(cudaStreamSynchronize(ctx->stream));
    rpd_stats s{};
    s.kernels_last_frame = ctx->kernels_last_frame;
    s.graph_replayed = ctx->graph_replayed;
    s.last_agg_kernel = ctx->last_agg_kernel;
    s.agg_segmented_ctas = ctx->agg_segmented_ctas;
    if (ctx->agg_reruns) {
      unsigned long long n = 0;
      RPD_CK(cudaMemcpy(&n, ctx->agg_reruns, sizeof(n), cudaMemcpyDeviceToHost));
      s.agg_segment_reruns = (int64_t)n;
    }
    if (ctx->slic_tiles) {
      unsigned long long n[4] = {0, 0, 0, 0};
      RPD_CK(cudaMemcpy(n, ctx->slic_tiles, sizeof(n), cudaMemcpyDeviceToHost));
      s.slic_tiles_assigned = (int64_t)n[0];
      s.slic_tiles_skipped = (int64_t)n[1];
      s.slic_centres_moved = (int64_t)n[2];
      s.slic_pixels_changed = (int64_t)n[3];
    }
    s.sgm_passes = ctx->profile ? ctx->agg_pass : 0;
    for (int i = 0; i < s.sgm_passes; ++i) {
      float ms = 0;
      RPD_CK(cudaEventElapsedTime(&ms, ctx->agg_ev[i][0], ctx->agg_ev[i][1]));
      s.sgm_agg_ms[i] = ms;
      s.sgm_agg_alg_bytes[i] = ctx->agg_alg_bytes[i];
      s.sgm_cells[i] = ctx->agg_cells[i];
    }
    *out = s;
  });
}

void rpd_config_default(rpd_config* cfg) {
  if (cfg) config_default(cfg);
}

rpd_status rpd_config_validate(rpd_ctx* ctx, const rpd_config* cfg) {
  return guard(ctx, [&] { config_validate(*cfg); });
}

rpd_status rpd_config_set(rpd_ctx* ctx, rpd_config* cfg, const char* key, const char* value) {
  return guard(ctx, [&] { config_set(cfg, key, value); });
}

// ------------------------------------------------------------ perspective --
rpd_status rpd_compute_row_shifts(rpd_ctx* ctx, const rpd_road_model* model, int w, int h,
                                  double delta_pt, double* shifts) {
  return guard(ctx, [&] {
    if (w < 2) throw InvalidArg("compute_row_shifts: width must be >= 2");
    if (h <= 0) return;
    DevModel* m = upload_model(ctx, *model);
    double* s = ctx->ws.get<double>("abi_shifts", h);
    launch_row_shifts(m, h, w, delta_pt, s, ctx->stream);
    download(ctx, shifts, s, sizeof(double) * h);
  });
}

rpd_status rpd_warp_right_image(rpd_ctx* ctx, const float* right, int h, int w,
                                const double* shifts, float* image, uint8_t* in_view) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    const float* r = upload(ctx, "abi_in0", right, n);
    const double* s = upload(ctx, "abi_shifts", shifts, size_t(h));
    float* o = ctx->ws.get<float>("abi_out0", n);
    uint8_t* iv = ctx->ws.get<uint8_t>("abi_out1", n);
    launch_warp_right(r, s, h, w, o, iv, ctx->stream);
    if (image) download(ctx, image, o, sizeof(float) * n);
    if (in_view) download(ctx, in_view, iv, n);
  });
}

rpd_status rpd_restore_disparity(rpd_ctx* ctx, const float* d0, int h, int w,
                                 const double* shifts, float* d1) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    const float* a = upload(ctx, "abi_in0", d0, n);
    const double* s = upload(ctx, "abi_shifts", shifts, size_t(h));
    float* o = ctx->ws.get<float>("abi_out0", n);
    launch_restore(a, s, h, w, o, ctx->stream);
    download(ctx, d1, o, sizeof(float) * n);
  });
}

// -------------------------------------------------------------------- SGM --
rpd_status rpd_census_cost_volume(rpd_ctx* ctx, const float* left, const float* right, int h,
                                  int w, int d_max, int window, const uint8_t* in_view,
                                  float* costs) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (window % 2 == 0) throw InvalidArg("census_cost_volume: window must be odd");
    if (window < 3 || window > 7) throw InvalidArg("census_cost_volume: window must be 3, 5 or 7");
    if (d_max >= w) throw InvalidArg("census_cost_volume: d_max >= width");
    if (d_max < 0) throw InvalidArg("census_cost_volume: d_max must be >= 0");
    const size_t n = size_t(h) * w;
    const float* l = upload(ctx, "abi_in0", left, n);
    const float* r = upload(ctx, "abi_in1", right, n);
    const uint8_t* iv = in_view ? upload(ctx, "abi_in2", in_view, n) : nullptr;
    uint64_t* cl = ctx->ws.get<uint64_t>("abi_cl", n);
    uint64_t* cr = ctx->ws.get<uint64_t>("abi_cr", n);
    launch_census(l, h, w, window, cl, ctx->stream);
    launch_census(r, h, w, window, cr, ctx->stream);
    const size_t cells = n * size_t(d_max + 1);
    float* c = ctx->ws.get<float>("abi_vol0", cells);
    launch_cost_f32(cl, cr, iv, h, w, d_max + 1, window, c, ctx->stream);
    download(ctx, costs, c, sizeof(float) * cells);
  });
}

rpd_status rpd_aggregate_costs(rpd_ctx* ctx, const float* costs, int h, int w, int d_max,
                               const int32_t* dirs, int ndirs, float l1, float l2, float* agg) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (d_max < 0 || ndirs < 0) throw InvalidArg("aggregate_costs: bad dimensions");
    const size_t cells = size_t(h) * w * size_t(d_max + 1);
    int paths = 0;
    const bool u8 = aggregate_u8_eligible(costs, cells, d_max + 1, dirs, ndirs, l1, l2, &paths);
    const float* c = upload(ctx, "abi_vol0", costs, cells);
    float* o = ctx->ws.get<float>("abi_vol1", cells);
    if (u8) {
      aggregate_u8_dev(ctx, c, h, w, d_max + 1, paths, l1, l2, o);
    } else {
      aggregate_f32(ctx, c, h, w, d_max + 1, dirs, ndirs, l1, l2, o);
      ctx->last_agg_kernel = kAggF32;
    }
    download(ctx, agg, o, sizeof(float) * cells);
  });
}

rpd_status rpd_swap_reference(rpd_ctx* ctx, const float* costs, int h, int w, int d_max,
                              float* right_costs) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (d_max < 0) throw InvalidArg("swap_reference: bad dimensions");
    const size_t cells = size_t(h) * w * size_t(d_max + 1);
    const float* c = upload(ctx, "abi_vol0", costs, cells);
    float* o = ctx->ws.get<float>("abi_vol1", cells);
    swap_reference_f32(ctx, c, h, w, d_max + 1, o);
    download(ctx, right_costs, o, sizeof(float) * cells);
  });
}

rpd_status rpd_select_disparity(rpd_ctx* ctx, const float* agg, int h, int w, int d_max,
                                float* disp) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (d_max < 0) throw InvalidArg("select_disparity: bad dimensions");
    const size_t n = size_t(h) * w;
    const float* a = upload(ctx, "abi_vol0", agg, n * size_t(d_max + 1));
    float* o = ctx->ws.get<float>("abi_out0", n);
    select_disparity_f32(a, h, w, d_max + 1, o, ctx->stream);
    download(ctx, disp, o, sizeof(float) * n);
  });
}

rpd_status rpd_consistency_filter(rpd_ctx* ctx, float* left, const float* right, int h, int w,
                                  double thr) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    float* l = upload(ctx, "abi_in0", left, n);
    const float* r = upload(ctx, "abi_in1", right, n);
    consistency_filter_dev(l, r, h, w, thr, ctx->stream);
    download(ctx, left, l, sizeof(float) * n);
  });
}

rpd_status rpd_match_pair(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                          const rpd_road_model* model, const rpd_config* cfg, int d_max,
                          float* d0, float* d1, double* shifts) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (cfg->sgm_paths != 4 && cfg->sgm_paths != 8)
      throw InvalidArg("config: sgm_paths must be 4 or 8");
    const size_t n = size_t(h) * w;
    const float* l = upload(ctx, "abi_in0", left, n);
    const float* r = upload(ctx, "abi_in1", right, n);
    DevModel* m = upload_model(ctx, *model);
    float* o0 = ctx->ws.get<float>("abi_out0", n);
    float* o1 = ctx->ws.get<float>("abi_out1", n);
    double* s = ctx->ws.get<double>("abi_shifts", h);
    match_pair_dev(ctx, l, r, h, w, m, *cfg, d_max, o0, o1, s);
    if (d0) download(ctx, d0, o0, sizeof(float) * n);
    if (d1) download(ctx, d1, o1, sizeof(float) * n);
    if (shifts) download(ctx, shifts, s, sizeof(double) * h);
  });
}

rpd_status rpd_match_pair_dump(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                               const rpd_road_model* model, const rpd_config* cfg, int d_max,
                               float* cost, float* agg_left, float* agg_right, float* disp_left,
                               float* disp_right) {
  const rpd_sgm_dump d{cost, nullptr, agg_left, agg_right, disp_left, disp_right};
  return rpd_match_pair_dump_ex(ctx, left, right, h, w, model, cfg, d_max, &d);
}

rpd_status rpd_match_pair_dump_ex(rpd_ctx* ctx, const float* left, const float* right, int h,
                                  int w, const rpd_road_model* model, const rpd_config* cfg,
                                  int d_max, const rpd_sgm_dump* out) {
  float* cost = out->cost;
  float* cost_right = out->cost_right;
  float* agg_left = out->agg_left;
  float* agg_right = out->agg_right;
  float* disp_left = out->disp_left;
  float* disp_right = out->disp_right;
  return guard(ctx, [&] {
    check_dims(h, w);
    if (cfg->sgm_paths != 4 && cfg->sgm_paths != 8)
      throw InvalidArg("config: sgm_paths must be 4 or 8");
    if (d_max < 0) throw InvalidArg("census_cost_volume: d_max must be >= 0");
    const size_t n = size_t(h) * w;
    const size_t cells = n * size_t(d_max + 1);
    const float* l = upload(ctx, "abi_in0", left, n);
    const float* r = upload(ctx, "abi_in1", right, n);
    DevModel* m = upload_model(ctx, *model);
    float* o0 = ctx->ws.get<float>("abi_out0", n);
    float* o1 = ctx->ws.get<float>("abi_out1", n);
    double* s = ctx->ws.get<double>("abi_shifts", h);
    MatchDump dump;
    dump.cost = cost ? ctx->ws.get<float>("abi_dump_cost", cells) : nullptr;
    dump.cost_right = cost_right ? ctx->ws.get<float>("abi_dump_costr", cells) : nullptr;
    dump.agg_left = agg_left ? ctx->ws.get<float>("abi_dump_aggl", cells) : nullptr;
    dump.agg_right = agg_right ? ctx->ws.get<float>("abi_dump_aggr", cells) : nullptr;
    dump.disp_left = disp_left ? ctx->ws.get<float>("abi_dump_dl", n) : nullptr;
    dump.disp_right = disp_right ? ctx->ws.get<float>("abi_dump_dr", n) : nullptr;
    match_pair_dev(ctx, l, r, h, w, m, *cfg, d_max, o0, o1, s, &dump);
    if (cost) download(ctx, cost, dump.cost, sizeof(float) * cells);
    if (cost_right) download(ctx, cost_right, dump.cost_right, sizeof(float) * cells);
    if (agg_left) download(ctx, agg_left, dump.agg_left, sizeof(float) * cells);
    if (agg_right) download(ctx, agg_right, dump.agg_right, sizeof(float) * cells);
    if (disp_left) download(ctx, disp_left, dump.disp_left, sizeof(float) * n);
    if (disp_right) download(ctx, disp_right, dump.disp_right, sizeof(float) * n);
    RPD_CK(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
