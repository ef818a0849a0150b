// abi_geom3d.cu — 3-D reprojection and point-cloud error (road_geometry.cpp:
// 153-188 of the reference) on the device.
//
// * reproject / reproject_masked: flag -> exclusive scan -> scatter keeps the
//   reference's scan order; every coordinate is computed with the reference's
//   double expression order (no contraction: --fmad=false) and rounded to
//   float, so the points are bit-identical.
// * reproject_instances: all pothole clouds of a label map in one pass — a
//   stable radix sort of (label, pixel) pairs gives scan order within each
//   label (the CLI's per-pothole loop, rpd_cli.cpp:99-104).
// * closest_distance_error: brute force, one thread per test point against
//   shared-memory tiles of the truth cloud; the per-point minima are exact
//   (same double expressions), their sum is taken in double-double with
//   block partials in a fixed order, so the result is the correctly rounded
//   square root of a near-exact mean (the reference sums sequentially).
#include <cub/cub.cuh>

#include <vector>

#include "abi_util.hpp"

using namespace rpdg;

namespace {

struct Rig {
  double focal, baseline, cu, cv;
};

__device__ __forceinline__ rpd_point3 reproject_px(float d, int u, int v, const Rig& r) {
  const double z = r.focal * r.baseline / double(d);
  return rpd_point3{static_cast<float>((double(u) - r.cu) * z / r.focal),
                    static_cast<float>((double(v) - r.cv) * z / r.focal), static_cast<float>(z)};
}

__device__ __forceinline__ bool reprojectable(float d) { return d != kInvalid && d > 0.0f; }

__global__ void k_reproj_flags(const float* __restrict__ d1, const int32_t* __restrict__ labels,
                               int label, long long n, int* __restrict__ flags) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x)
    flags[p] = reprojectable(d1[p]) && (!labels || labels[p] == label) ? 1 : 0;
}

__global__ void k_reproj_scatter(const float* __restrict__ d1, const int* __restrict__ flags,
                                 const int* __restrict__ pos, int w, long long n, Rig rig,
                                 long long cap, rpd_point3* __restrict__ out,
                                 long long* __restrict__ count) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    if (flags[p] && pos[p] < cap) out[pos[p]] = reproject_px(d1[p], int(p % w), int(p / w), rig);
    if (p == n - 1) *count = (long long)pos[p] + flags[p];
  }
}

// keys: label (1..max_label) of reprojectable pixels, max_label + 1 otherwise
__global__ void k_instance_keys(const float* __restrict__ d1, const int32_t* __restrict__ labels,
                                int max_label, long long n, unsigned* __restrict__ keys,
                                int* __restrict__ idx) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int l = labels[p];
    keys[p] = (l >= 1 && l <= max_label && reprojectable(d1[p])) ? unsigned(l)
                                                                   : unsigned(max_label) + 1u;
    idx[p] = int(p);
  }
}

__global__ void k_instance_counts(const unsigned* __restrict__ keys, long long n, int max_label,
                                  unsigned long long* __restrict__ cnt) {
  for (long long p0 = blockIdx.x * (long long)blockDim.x; p0 < n;
       p0 += (long long)gridDim.x * blockDim.x) {
    const long long p = p0 + threadIdx.x;
    const int k = p < n ? int(keys[p]) : max_label + 1;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, k);
    if (k <= max_label && (threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&cnt[k], (unsigned long long)__popc(peers));
  }
}

__global__ void k_instance_points(const float* __restrict__ d1, const int* __restrict__ idx,
                                  int w, long long total, Rig rig, rpd_point3* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long p = idx[i];
    out[i] = reproject_px(d1[p], int(p % w), int(p / w), rig);
  }
}

constexpr int kCdeThreads = 256;
constexpr int kCdeTile = 1024;  // truth points per shared-memory tile

struct DDs {
  double hi, lo;
};
__device__ __forceinline__ DDs dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ DDs dd_plus(DDs a, DDs b) {
  DDs s = dd_two_sum(a.hi, b.hi);
  const DDs t = dd_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  double hi = s.hi + s.lo;
  double lo = s.lo - (hi - s.hi);
  lo += t.lo;
  const double h2 = hi + lo;
  return {h2, lo - (h2 - hi)};
}

__global__ void __launch_bounds__(kCdeThreads)
    k_cde(const rpd_point3* __restrict__ test, long long n, const rpd_point3* __restrict__ truth,
          long long m, DDs* __restrict__ part) {
  __shared__ float3 tile[kCdeTile];
  DDs acc{0.0, 0.0};
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < n;
       t0 += (long long)gridDim.x * blockDim.x) {
    const long long i = t0 + threadIdx.x;
    rpd_point3 p{0.f, 0.f, 0.f};
    if (i < n) p = test[i];
    double best = __longlong_as_double(0x7FF0000000000000ll);  // +inf (road_geometry.cpp:180)
    for (long long g0 = 0; g0 < m; g0 += kCdeTile) {
      __syncthreads();
      for (int j = threadIdx.x; j < kCdeTile && g0 + j < m; j += blockDim.x) {
        const rpd_point3 g = truth[g0 + j];
        tile[j] = make_float3(g.x, g.y, g.z);
      }
      __syncthreads();
      const int cnt = int(m - g0 < kCdeTile ? m - g0 : (long long)kCdeTile);
      for (int j = 0; j < cnt; ++j) {
        const float3 g = tile[j];
        const double dx = double(p.x) - double(g.x), dy = double(p.y) - double(g.y),
                     dz = double(p.z) - double(g.z);
        const double d2 = dx * dx + dy * dy + dz * dz;
        best = d2 < best ? d2 : best;  // std::min(best, d2)
      }
    }
    if (i < n) acc = dd_plus(acc, DDs{best, 0.0});
  }
  __shared__ DDs s[kCdeThreads];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int width = kCdeThreads / 2; width > 0; width >>= 1) {
    if (threadIdx.x < width) s[threadIdx.x] = dd_plus(s[threadIdx.x], s[threadIdx.x + width]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

Rig to_rig(const rpd_stereo_rig* r) {
  if (!r) throw InvalidArg("reproject: null rig");
  if (r->focal <= 0 || r->baseline <= 0) throw InvalidArg("reproject: bad rig");  // :154
  return Rig{r->focal, r->baseline, r->cu, r->cv};
}

long long reproject_impl(rpd_ctx* ctx, const float* d1, const int32_t* labels, int label, int h,
                         int w, const Rig& rig, rpd_point3* out, long long cap) {
  check_dims(h, w);
  cudaStream_t st = ctx->stream;
  const long long n = (long long)h * w;
  const float* dd = upload(ctx, "rp_d1", d1, size_t(n));
  const int32_t* dl = labels ? upload(ctx, "rp_labels", labels, size_t(n)) : nullptr;
  int* flags = ctx->ws.get<int>("rp_flags", size_t(n));
  int* pos = ctx->ws.get<int>("rp_pos", size_t(n));
  long long* count = ctx->ws.get<long long>("rp_count", 1);
  rpd_point3* dout = ctx->ws.get<rpd_point3>("rp_out", size_t(std::max<long long>(1, std::min<long long>(cap, n))));
  const int blocks = int(std::min<long long>((n + 255) / 256, ctx->sm_count * 16));
  k_reproj_flags<<<blocks, 256, 0, st>>>(dd, dl, label, n, flags);
  RPD_LAUNCH_CHECK();
  scan_exclusive_i32(ctx, flags, pos, n);
  k_reproj_scatter<<<blocks, 256, 0, st>>>(dd, flags, pos, w, n, rig, cap, dout, count);
  RPD_LAUNCH_CHECK();
  long long hc = 0;
  download(ctx, &hc, count, sizeof(hc));
  const long long k = std::min(hc, cap);
  if (k > 0) download(ctx, out, dout, sizeof(rpd_point3) * size_t(k));
  return hc;
}

}  // namespace

extern "C" {

rpd_stereo_rig rpd_rig_from_config(const rpd_config* cfg, int width, int height) {
  // pipeline.cpp:38-45
  rpd_stereo_rig r{700.0, 0.12, 0.0, 0.0};
  if (!cfg) return r;
  r.focal = cfg->focal;
  r.baseline = cfg->baseline;
  r.cu = cfg->cu >= 0 ? cfg->cu : width / 2.0;
  r.cv = cfg->cv >= 0 ? cfg->cv : height / 2.0;
  return r;
}

rpd_status rpd_reproject(rpd_ctx* ctx, const float* d1, int h, int w, const rpd_stereo_rig* rig,
                         rpd_point3* out, int64_t cap, int64_t* n) {
  return guard(ctx, [&] {
    if (!d1 || !n || (cap > 0 && !out)) throw InvalidArg("reproject: null buffer");
    const long long c = reproject_impl(ctx, d1, nullptr, 0, h, w, to_rig(rig), out, cap);
    *n = c;
    if (c > cap) throw Capacity("reproject: more points than cap");
  });
}

rpd_status rpd_reproject_masked(rpd_ctx* ctx, const float* d1, const int32_t* labels, int h,
                                int w, int label, const rpd_stereo_rig* rig, rpd_point3* out,
                                int64_t cap, int64_t* n) {
  return guard(ctx, [&] {
    if (!d1 || !labels || !n || (cap > 0 && !out)) throw InvalidArg("reproject: null buffer");
    const long long c = reproject_impl(ctx, d1, labels, label, h, w, to_rig(rig), out, cap);
    *n = c;
    if (c > cap) throw Capacity("reproject_masked: more points than cap");
  });
}

rpd_status rpd_reproject_instances(rpd_ctx* ctx, const float* d1, const int32_t* labels, int h,
                                   int w, int max_label, const rpd_stereo_rig* rig,
                                   rpd_point3* out, int64_t cap, int64_t* offsets) {
  return guard(ctx, [&] {
    if (!d1 || !labels || !offsets || (cap > 0 && !out))
      throw InvalidArg("reproject_instances: null buffer");
    if (max_label < 0) throw InvalidArg("reproject_instances: max_label < 0");
    check_dims(h, w);
    const Rig r = to_rig(rig);
    cudaStream_t st = ctx->stream;
    const long long n = (long long)h * w;
    const float* dd = upload(ctx, "rp_d1", d1, size_t(n));
    const int32_t* dl = upload(ctx, "rp_labels", labels, size_t(n));
    unsigned* keys = ctx->ws.get<unsigned>("rp_keys", size_t(n));
    unsigned* keys2 = ctx->ws.get<unsigned>("rp_keys2", size_t(n));
    int* idx = ctx->ws.get<int>("rp_idx", size_t(n));
    int* idx2 = ctx->ws.get<int>("rp_idx2", size_t(n));
    rpd_point3* dout = ctx->ws.get<rpd_point3>("rp_out", size_t(std::max<long long>(1, std::min<long long>(cap, n))));
    const int blocks = int(std::min<long long>((n + 255) / 256, ctx->sm_count * 16));
    k_instance_keys<<<blocks, 256, 0, st>>>(dd, dl, max_label, n, keys, idx);
    RPD_LAUNCH_CHECK();
    int bits = 1;
    while ((1ll << bits) <= (long long)max_label + 1) ++bits;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, idx, idx2, int(n), 0, bits,
                                    st);
    void* tmp = ctx->ws.get<uint8_t>("rp_sort", tmp_bytes);
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, idx, idx2, int(n), 0, bits, st);
    RPD_LAUNCH_CHECK();
    unsigned long long* dcnt = ctx->ws.get<unsigned long long>("rp_cnt", size_t(max_label) + 1);
    RPD_CK(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * (size_t(max_label) + 1), st));
    k_instance_counts<<<blocks, 256, 0, st>>>(keys, n, max_label, dcnt);
    RPD_LAUNCH_CHECK();
    std::vector<unsigned long long> hc(size_t(max_label) + 1);
    download(ctx, hc.data(), dcnt, sizeof(unsigned long long) * hc.size());
    std::vector<long long> ho(size_t(max_label) + 1, 0);  // ho[k] = end of label k
    for (int q = 1; q <= max_label; ++q) ho[size_t(q)] = ho[size_t(q) - 1] + (long long)hc[size_t(q)];
    const long long total = ho[size_t(max_label)];
    const long long k = std::min<long long>(total, cap);
    if (k > 0) {
      k_instance_points<<<blocks, 256, 0, st>>>(dd, idx2, w, k, r, dout);
      RPD_LAUNCH_CHECK();
      download(ctx, out, dout, sizeof(rpd_point3) * size_t(k));
    }
    for (size_t q = 0; q < ho.size(); ++q) offsets[q] = ho[q];
    if (total > cap) throw Capacity("reproject_instances: more points than cap");
  });
}

rpd_status rpd_closest_distance_error(rpd_ctx* ctx, const rpd_point3* test, int64_t n_test,
                                      const rpd_point3* truth, int64_t n_truth, double* out) {
  return guard(ctx, [&] {
    if (n_test <= 0 || n_truth <= 0 || !test || !truth)
      throw InvalidArg("closest_distance_error: empty cloud");  // :175-176
    if (!out) throw InvalidArg("closest_distance_error: null output");
    const rpd_point3* dt = upload(ctx, "cde_test", test, size_t(n_test));
    const rpd_point3* dg = upload(ctx, "cde_truth", truth, size_t(n_truth));
    const int blocks = int(std::min<long long>((n_test + kCdeThreads - 1) / kCdeThreads,
                                               ctx->sm_count * 8));
    DDs* part = ctx->ws.get<DDs>("cde_part", size_t(blocks));
    k_cde<<<blocks, kCdeThreads, 0, ctx->stream>>>(dt, n_test, dg, n_truth, part);
    RPD_LAUNCH_CHECK();
    std::vector<DDs> hp(static_cast<size_t>(blocks));
    download(ctx, hp.data(), part, sizeof(DDs) * hp.size());
    double hi = 0.0, lo = 0.0;  // the device's dd_plus over the block partials, in order
    for (const DDs& b : hp) {
      auto two_sum = [](double a, double c, double& s, double& e) {
        s = a + c;
        const double bb = s - a;
        e = (a - (s - bb)) + (c - bb);
      };
      double sh, sl, th, tl;
      two_sum(hi, b.hi, sh, sl);
      two_sum(lo, b.lo, th, tl);
      sl += th;
      const double h2 = sh + sl;
      double l2 = sl - (h2 - sh);
      l2 += tl;
      hi = h2 + l2;
      lo = l2 - (hi - h2);
    }
    *out = std::sqrt(hi / static_cast<double>(n_test));
  });
}

}  // extern "C"
