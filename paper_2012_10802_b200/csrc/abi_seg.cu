// abi_seg.cu — road-geometry and segmentation entry points of the C-ABI
// (include/rpd_b200.h).  Each call stages host buffers into context
// workspaces, runs the same device routines the pipeline uses, and copies the
// result back.
#include <vector>

#include "scan.cuh"
#include "abi_util.hpp"
#include "road.cuh"
#include "seg.cuh"
#include "sgm.cuh"

using namespace rpdg;

namespace rpdg {
void sincos_probe_dev(const double* x, int n, double* s, double* c, cudaStream_t st);
}

namespace {

FitOut run_fit(rpd_ctx* ctx, FitRequest req) {
  reset_status(ctx);
  FitOut* out = ctx->ws.get<FitOut>("abi_fit_out", 1);
  req.out = out;
  req.where = kWhereFit;
  fit_dev(ctx, req);
  FitOut h{};
  RPD_CK(cudaMemcpyAsync(&h, out, sizeof(FitOut), cudaMemcpyDeviceToHost, ctx->stream));
  sync_and_check(ctx);
  return h;
}

FitRequest double_request(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                          int64_t k) {
  if (k < 3) throw InvalidArg("fit_line: need at least 3 observations");
  FitRequest r;
  r.compact = false;
  r.k_host = k;
  r.dd = upload(ctx, "abi_obs_d", d, size_t(k));
  r.du = upload(ctx, "abi_obs_u", u, size_t(k));
  r.dv = upload(ctx, "abi_obs_v", v, size_t(k));
  return r;
}

}  // namespace

extern "C" {

rpd_status rpd_sample_observations(rpd_ctx* ctx, const float* d1, int h, int w,
                                   const rpd_rect_roi* roi, int64_t cap, double* d, double* u,
                                   double* v, int64_t* count) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (cap < 1) throw InvalidArg("sample_observations: cap must be >= 1");
    const size_t n = size_t(h) * w;
    const long long kmax = std::min<long long>(cap, (long long)n);
    const float* dd = upload(ctx, "abi_in0", d1, n);
    ObsBuffers obs{ctx->ws.get<uint32_t>("abi_so_uv", kmax), ctx->ws.get<float>("abi_so_d", kmax),
                   ctx->ws.get<int>("abi_so_count", 1)};
    reset_status(ctx);
    sample_observations_dev(ctx, dd, h, w, roi, cap, obs, kWhereSample);
    int k = 0;
    RPD_CK(cudaMemcpyAsync(&k, obs.count, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    sync_and_check(ctx);
    std::vector<uint32_t> uv(static_cast<size_t>(k));
    std::vector<float> df(static_cast<size_t>(k));
    download(ctx, uv.data(), obs.uv, sizeof(uint32_t) * k);
    download(ctx, df.data(), obs.d, sizeof(float) * k);
    for (int i = 0; i < k; ++i) {
      u[i] = double(uv[size_t(i)] & 0xFFFFu);
      v[i] = double(uv[size_t(i)] >> 16);
      d[i] = double(df[size_t(i)]);
    }
    *count = k;
  });
}

rpd_status rpd_fit_line(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                        int64_t k, double phi, rpd_line_fit* out) {
  return guard(ctx, [&] {
    FitRequest r = double_request(ctx, d, u, v, k);
    r.mode = kFitLine;
    r.phi = phi;
    const FitOut f = run_fit(ctx, r);
    *out = rpd_line_fit{rpd_road_model{f.a0, f.a1, f.phi}, f.e0min};
  });
}

rpd_status rpd_estimate_roll(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                             int64_t k, double lo, double hi, double tol, rpd_road_model* out) {
  return guard(ctx, [&] {
    if (tol <= 0) throw InvalidArg("estimate_roll: tol must be > 0");
    FitRequest r = double_request(ctx, d, u, v, k);
    r.mode = kEstimateRoll;
    r.lo = lo;
    r.hi = hi;
    r.tol = tol;
    const FitOut f = run_fit(ctx, r);
    *out = rpd_road_model{f.a0, f.a1, f.phi};
  });
}

rpd_status rpd_fit_road(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                        int64_t k, double bracket, double tol, rpd_road_fit* out) {
  return guard(ctx, [&] {
    if (tol <= 0) throw InvalidArg("estimate_roll: tol must be > 0");
    FitRequest r = double_request(ctx, d, u, v, k);
    r.mode = kFitRoad;
    r.hi = bracket;
    r.tol = tol;
    const FitOut f = run_fit(ctx, r);
    *out = rpd_road_fit{rpd_road_model{f.a0, f.a1, f.phi}, f.e0min, f.used};
  });
}

rpd_status rpd_transform_disparity(rpd_ctx* ctx, const float* d1, int h, int w,
                                   const rpd_road_model* model, double delta_dt, float* d2,
                                   int64_t* clamped) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    const float* a = upload(ctx, "abi_in0", d1, n);
    DevModel* m = upload_model(ctx, *model);
    float* o = ctx->ws.get<float>("abi_out0", n);
    unsigned long long* c = ctx->ws.get<unsigned long long>("abi_clamped", 1);
    RPD_CK(cudaMemsetAsync(c, 0, sizeof(unsigned long long), ctx->stream));
    transform_disparity_dev(a, h, w, m, delta_dt, o, c, ctx->stream);
    unsigned long long hc = 0;
    RPD_CK(cudaMemcpyAsync(&hc, c, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
    download(ctx, d2, o, sizeof(float) * n);
    if (clamped) *clamped = int64_t(hc);
  });
}

rpd_status rpd_slic(rpd_ctx* ctx, const float* d2, int h, int w, int p, double m, int iters,
                    int32_t* labels, rpd_center* centers, int cap, int32_t* count,
                    double* spacing) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    const float* a = upload(ctx, "abi_in0", d2, n);
    const SlicOut sp = slic_dev(ctx, a, h, w, p, m, iters);
    int k = 0;
    RPD_CK(cudaMemcpyAsync(&k, sp.count, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RPD_CK(cudaStreamSynchronize(ctx->stream));
    if (labels) download(ctx, labels, sp.labels, sizeof(int32_t) * n);
    if (centers && cap > 0 && k > 0)
      download(ctx, centers, sp.centers, sizeof(double) * 3 * size_t(std::min(cap, k)));
    if (count) *count = k;
    if (spacing) *spacing = sp.spacing;
  });
}

rpd_status rpd_pool_superpixels(rpd_ctx* ctx, const float* d2, const int32_t* lab, int count,
                                int h, int w, float* d3) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    if (count < 0) throw InvalidArg("pool_superpixels: negative count");
    for (size_t i = 0; i < n; ++i)
      if (lab[i] < 0 || lab[i] > count)
        throw InvalidArg("pool_superpixels: label out of range");
    const float* a = upload(ctx, "abi_in0", d2, n);
    const int32_t* l = upload(ctx, "abi_lab0", lab, n);
    float* o = ctx->ws.get<float>("abi_out0", n);
    pool_superpixels_dev(ctx, a, l, h, w, count, o);
    download(ctx, d3, o, sizeof(float) * n);
  });
}

rpd_status rpd_build_histogram(rpd_ctx* ctx, const float* d2, int h, int w, double bw,
                               int64_t* counts, int64_t cap_n, int64_t* n, double* origin,
                               int64_t* total) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t np = size_t(h) * w;
    const float* a = upload(ctx, "abi_in0", d2, np);
    reset_status(ctx);
    long long nn = 0, tt = 0;
    double oo = 0;
    try {
      build_histogram_full_dev(ctx, a, h, w, bw, &nn, &oo, &tt,
                               reinterpret_cast<long long*>(counts), cap_n);
    } catch (const Capacity&) {
      *n = nn;
      *origin = oo;
      *total = tt;
      throw;
    }
    sync_and_check(ctx);
    *n = nn;
    *origin = oo;
    *total = tt;
  });
}

rpd_status rpd_find_road_threshold(rpd_ctx* ctx, const int64_t* counts, int64_t n, double bw,
                                   double origin, int64_t total, double delta_pd, double tau,
                                   rpd_threshold* out) {
  return guard(ctx, [&] {
    if (n < 0) throw InvalidArg("find_road_threshold: negative size");
    if (n > 46341) throw InvalidArg("find_road_threshold: histogram too large");
    reset_status(ctx);
    const long long* c =
        upload(ctx, "abi_hist", reinterpret_cast<const long long*>(counts), size_t(n) * n);
    rpd_threshold* o = ctx->ws.get<rpd_threshold>("abi_thr", 1);
    threshold_from_full_dev(ctx, c, n, bw, origin, total, delta_pd, tau, o);
    rpd_threshold h{};
    RPD_CK(cudaMemcpyAsync(&h, o, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    sync_and_check(ctx);
    *out = h;
  });
}

rpd_status rpd_connected_components(rpd_ctx* ctx, const int32_t* mask, int h, int w, int conn,
                                    int32_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    const int32_t* m = upload(ctx, "abi_lab0", mask, n);
    int32_t* o = ctx->ws.get<int32_t>("abi_lab1", n);
    connected_components_dev(ctx, m, h, w, conn, o);
    download(ctx, out, o, sizeof(int32_t) * n);
  });
}

rpd_status rpd_detect_potholes(rpd_ctx* ctx, const float* d3, const int32_t* sp_labels,
                               double spacing, int h, int w, const rpd_threshold* thr, int margin,
                               int min_sp, int conn, int32_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const size_t n = size_t(h) * w;
    const float* a = upload(ctx, "abi_in0", d3, n);
    const int32_t* l = upload(ctx, "abi_lab0", sp_labels, n);
    const rpd_threshold* t = upload(ctx, "abi_thr_in", thr, 1);
    int32_t* o = ctx->ws.get<int32_t>("abi_lab1", n);
    detect_potholes_dev(ctx, a, l, spacing, h, w, t, margin, min_sp, conn, o, nullptr);
    download(ctx, out, o, sizeof(int32_t) * n);
  });
}

rpd_status rpd_debug_sincos(rpd_ctx* ctx, const double* x, int n, double* s, double* c) {
  return guard(ctx, [&] {
    if (n <= 0) return;
    const double* dx = upload(ctx, "abi_dbg_x", x, size_t(n));
    double* ds = ctx->ws.get<double>("abi_dbg_s", size_t(n));
    double* dc = ctx->ws.get<double>("abi_dbg_c", size_t(n));
    sincos_probe_dev(dx, n, ds, dc, ctx->stream);
    download(ctx, s, ds, sizeof(double) * size_t(n));
    download(ctx, c, dc, sizeof(double) * size_t(n));
  });
}

rpd_status rpd_debug_scan(rpd_ctx* ctx, const int32_t* in, int64_t n, int32_t* out,
                          int32_t* total) {
  return guard(ctx, [&] {
    if (n < 0) throw InvalidArg("scan: n < 0");
    int* dtot = ctx->ws.get<int>("abi_dbg_scan_total", 1);
    RPD_CK(cudaMemsetAsync(dtot, 0, sizeof(int), ctx->stream));
    if (n > 0) {
      const int* din = upload(ctx, "abi_dbg_scan_in", in, size_t(n));
      int* dout = ctx->ws.get<int>("abi_dbg_scan_out", size_t(n));
      scan_exclusive(ctx, ScanArrayIn{din}, dout, n, dtot);
      download(ctx, out, dout, sizeof(int) * size_t(n));
    }
    download(ctx, total, dtot, sizeof(int));
  });
}

}  // extern "C"
