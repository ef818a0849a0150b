// road.cu — road-model fit (fit_line / estimate_roll / fit_road), observation
// sampling and disparity transformation for sm_100a.
//
// Reference: /root/reference/proj/src/road_geometry.cpp:12-151.
//
// The whole golden-section roll search (18 iterations + trimming + second
// search at the default bracket/tol) runs inside ONE launch of an 8-CTA thread
// block cluster (8 x 1024 threads).  The observations (<= 100 000, 8 B each in
// the compact format) are staged once into the CTAs' shared memory; every
// fit_line probe is two cluster-wide reductions whose partials are exchanged
// through distributed shared memory (DSMEM).  No host round trip per probe.
//
// Reduction order (shared with the CPU oracle, oracle/rpd_oracle.cpp
// lane_tree_sum): element i belongs to lane i mod 8192 (lane = CTA*1024 +
// thread) and is added sequentially; lanes are then combined by an adjacent-
// pairwise binary tree (warp shuffles, then CTA, then the 8 cluster partials).
// Eigen's own SIMD order (road_geometry.cpp:20-24, 37) is not reproducible
// without Eigen; the reference tests pin these sums to 1e-9 relative.

#include <algorithm>

#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include "road.cuh"

namespace cg = cooperative_groups;

namespace rpdg {

// ------------------------------------------------ double-double sin/cos ----
namespace {
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__device__ __forceinline__ DD quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ DD two_prod(double a, double b) {
  const double p = a * b;
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DD dd_mul(DD a, DD b) {
  DD p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo;
  p.lo += a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ DD dd_div_d(DD a, double b) {
  const double q1 = a.hi / b;
  const DD p = two_prod(q1, b);
  DD r = two_sum(a.hi, -p.hi);
  r.lo -= p.lo;
  r.lo += a.lo;
  const double q2 = (r.hi + r.lo) / b;
  return quick_two_sum(q1, q2);
}
}  // namespace

__device__ void dd_sincos(double x, double* s_out, double* c_out) {
  const DD pio2 = {1.5707963267948966, 6.123233995736766e-17};
  const double kf = rint(x / pio2.hi);
  DD r = {x, 0.0};
  if (kf != 0.0) {
    const DD kp = dd_mul(pio2, DD{kf, 0.0});
    r = dd_add(r, DD{-kp.hi, -kp.lo});
  }
  const DD x2 = dd_mul(r, r);
  DD st = r, ss = r;        // sin series
  DD ct = {1.0, 0.0}, cs = ct;  // cos series
  for (int n = 1; n <= 24; ++n) {
    st = dd_div_d(dd_mul(st, x2), -double((2 * n) * (2 * n + 1)));
    ct = dd_div_d(dd_mul(ct, x2), -double((2 * n - 1) * (2 * n)));
    ss = dd_add(ss, st);
    cs = dd_add(cs, ct);
    if (fabs(st.hi) < 1e-40 && fabs(ct.hi) < 1e-40) break;
  }
  const int q = int((long long)kf & 3);
  const double sv = ss.hi, cv = cs.hi;
  switch (q) {
    case 0: *s_out = sv; *c_out = cv; break;
    case 1: *s_out = cv; *c_out = -sv; break;
    case 2: *s_out = -sv; *c_out = -cv; break;
    default: *s_out = -cv; *c_out = sv; break;
  }
}

// ------------------------------------------------- sample_observations ----
struct RoiPred {
  int u0, v0, u1, v1;
};

__global__ void k_sample_flags(const float* __restrict__ d1, int h, int w, RoiPred r,
                               int* __restrict__ flags) {
  const long long n = (long long)h * w;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int u = int(p % w), v = int(p / w);
    flags[p] = (u >= r.u0 && u < r.u1 && v >= r.v0 && v < r.v1 && d1[p] != kInvalid) ? 1 : 0;
  }
}

__global__ void k_sample_scatter(const int* __restrict__ flags, const int* __restrict__ pos,
                                 long long n, int* __restrict__ list, int* __restrict__ total) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    if (flags[p]) list[pos[p]] = int(p);
    if (p == n - 1) *total = pos[p] + flags[p];
  }
}

// road_geometry.cpp:119-133: k = min(n, cap); obs_i = valid[floor(i*n/k)].
__global__ void k_sample_gather(const float* __restrict__ d1, int w, const int* __restrict__ list,
                                const int* __restrict__ total, long long cap,
                                uint32_t* __restrict__ uv, float* __restrict__ d,
                                int* __restrict__ count, DevStatus* st, int where) {
  const long long n = *total;
  const long long k = n < cap ? n : cap;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i == 0) {
    *count = n < 3 ? 0 : int(k);
    if (n < 3) set_status(st, RPD_EDEGENERATE, where, n);
  }
  if (n < 3 || i >= k) return;
  const int p = list[(i * n) / k];
  uv[i] = uint32_t(p % w) | (uint32_t(p / w) << 16);
  d[i] = d1[p];
}

void sample_observations_dev(rpd_ctx* ctx, const float* d1, int h, int w, const rpd_rect_roi* roi,
                             long long cap, ObsBuffers obs, int where) {
  if (w >= 65536 || h >= 65536) throw InvalidArg("sample_observations: image side >= 65536");
  RoiPred r{0, 0, w, h};
  if (roi) {  // road_geometry.cpp:106-111
    const int u0 = std::clamp(roi->u0, 0, w), v0 = std::clamp(roi->v0, 0, h);
    const int ww = std::clamp(roi->width, 0, w - u0), hh = std::clamp(roi->height, 0, h - v0);
    r = RoiPred{u0, v0, u0 + ww, v0 + hh};
  }
  cudaStream_t st = ctx->stream;
  const long long n = (long long)h * w;
  int* flags = ctx->ws.get<int>("so_flags", n);
  int* pos = ctx->ws.get<int>("so_pos", n);
  int* list = ctx->ws.get<int>("so_list", n);
  int* total = ctx->ws.get<int>("so_total", 1);
  const int blocks = int(std::min<long long>((n + 255) / 256, ctx->sm_count * 16));
  k_sample_flags<<<blocks, 256, 0, st>>>(d1, h, w, r, flags);
  RPD_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flags, pos, int(n), st);
  void* tmp = ctx->ws.get<uint8_t>("so_cub", tmp_bytes);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags, pos, int(n), st);
  RPD_LAUNCH_CHECK();
  k_sample_scatter<<<blocks, 256, 0, st>>>(flags, pos, n, list, total);
  RPD_LAUNCH_CHECK();
  const long long gmax = std::min<long long>(cap, n);
  k_sample_gather<<<std::max(1, cdiv(gmax, 256)), 256, 0, st>>>(
      d1, w, list, total, cap, obs.uv, obs.d, obs.count, ctx->status, where);
  RPD_LAUNCH_CHECK();
}

// ----------------------------------------------------------- fit kernel ----
constexpr int kFitCtas = 8;
constexpr int kFitThreads = 1024;
constexpr int kFitLanes = kFitCtas * kFitThreads;  // == oracle kFitLanes
constexpr int kFitDynSmem = 192 * 1024;
constexpr int kRowsCompact = kFitDynSmem / (kFitThreads * 8);   // 24
constexpr int kRowsDouble = kFitDynSmem / (kFitThreads * 24);   // 8
constexpr int kMaxRowsTrim = 64;

struct FitKParams {
  FitRequest r;
  DevStatus* status;
  // trimming scratch (same format as the input)
  uint32_t* scr_uv;
  float* scr_d;
  double* scr_dd;
  double* scr_du;
  double* scr_dv;
};

struct FitShared {
  double warp_part[32][4];
  double cta_part[2][4];
  double bcast[4];
  double sc[2];
  int row_cnt[kMaxRowsTrim];
  int row_base[kMaxRowsTrim];
  int warp_cnt[32];
};

struct LineFitD {
  double a0, a1, phi, e0min, c, s;
};

struct FitState {
  const FitKParams* P;
  FitShared* S;
  unsigned char* dyn;
  bool compact;
  bool staged;
  long long k;
  int rows;
  int lane;
  int slot;
  // current (global) source when not staged
  const uint32_t* g_uv;
  const float* g_d;
  const double* g_dd;
  const double* g_du;
  const double* g_dv;
};

__device__ __forceinline__ void fit_get(const FitState& F, int m, long long i, double& d, double& u,
                                        double& v) {
  if (F.compact) {
    uint32_t uv;
    float df;
    if (F.staged) {
      const uint2 e = reinterpret_cast<const uint2*>(F.dyn)[m * kFitThreads + threadIdx.x];
      uv = e.x;
      df = __uint_as_float(e.y);
    } else {
      uv = F.g_uv[i];
      df = F.g_d[i];
    }
    u = double(uv & 0xFFFFu);
    v = double(uv >> 16);
    d = double(df);
  } else {
    if (F.staged) {
      const double* e = reinterpret_cast<const double*>(F.dyn) + 3 * (m * kFitThreads + threadIdx.x);
      d = e[0];
      u = e[1];
      v = e[2];
    } else {
      d = F.g_dd[i];
      u = F.g_du[i];
      v = F.g_dv[i];
    }
  }
}

// Stage the current source into shared memory (when it fits).
__device__ void fit_stage(FitState& F) {
  F.rows = int((F.k + kFitLanes - 1) / kFitLanes);
  F.staged = F.rows <= (F.compact ? kRowsCompact : kRowsDouble);
  if (!F.staged) return;
  for (int m = 0; m < F.rows; ++m) {
    const long long i = (long long)m * kFitLanes + F.lane;
    if (i >= F.k) break;
    if (F.compact) {
      reinterpret_cast<uint2*>(F.dyn)[m * kFitThreads + threadIdx.x] =
          make_uint2(F.g_uv[i], __float_as_uint(F.g_d[i]));
    } else {
      double* e = reinterpret_cast<double*>(F.dyn) + 3 * (m * kFitThreads + threadIdx.x);
      e[0] = F.g_dd[i];
      e[1] = F.g_du[i];
      e[2] = F.g_dv[i];
    }
  }
  __syncthreads();
}

// Cluster-wide sum of NV doubles in the fixed adjacent-pairwise lane order.
template <int NV>
__device__ void cluster_sum(FitState& F, double (&x)[NV]) {
  cg::cluster_group cl = cg::this_cluster();
  FitShared& S = *F.S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1)
#pragma unroll
    for (int q = 0; q < NV; ++q) x[q] += __shfl_down_sync(0xFFFFFFFFu, x[q], off);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) S.warp_part[warp][q] = x[q];
  __syncthreads();
  if (warp == 0) {
    double y[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) y[q] = S.warp_part[lane][q];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1)
#pragma unroll
      for (int q = 0; q < NV; ++q) y[q] += __shfl_down_sync(0xFFFFFFFFu, y[q], off);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NV; ++q) S.cta_part[F.slot][q] = y[q];
  }
  cl.sync();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double p[kFitCtas];
#pragma unroll
      for (int r = 0; r < kFitCtas; ++r) p[r] = *cl.map_shared_rank(&S.cta_part[F.slot][q], r);
#pragma unroll
      for (int width = 1; width < kFitCtas; width *= 2)
#pragma unroll
        for (int j = 0; j < kFitCtas; j += 2 * width) p[j] += p[j + width];
      S.bcast[q] = p[0];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) x[q] = S.bcast[q];
  F.slot ^= 1;
}

__device__ double fit_sum_d(FitState& F) {
  double x[1] = {0.0};
  for (int m = 0; m < F.rows; ++m) {
    const long long i = (long long)m * kFitLanes + F.lane;
    if (i >= F.k) break;
    double d, u, v;
    fit_get(F, m, i, d, u, v);
    x[0] += d;
  }
  cluster_sum<1>(F, x);
  return x[0];
}

// fit_line, road_geometry.cpp:12-39.  Returns false when the normal matrix is
// singular (the reference throws runtime_error).
__device__ bool fit_probe(FitState& F, double phi, double sd, LineFitD& out) {
  FitShared& S = *F.S;
  if (threadIdx.x == 0) {
    double s, c;
    dd_sincos(phi, &s, &c);
    S.sc[0] = s;
    S.sc[1] = c;
  }
  __syncthreads();
  const double s = S.sc[0], c = S.sc[1];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int m = 0; m < F.rows; ++m) {
    const long long i = (long long)m * kFitLanes + F.lane;
    if (i >= F.k) break;
    double d, u, v;
    fit_get(F, m, i, d, u, v);
    const double t = c * v - s * u;
    acc[0] += t;
    acc[1] += t * t;
    acc[2] += d * t;
  }
  cluster_sum<3>(F, acc);
  const double kk = double(F.k);
  const double st = acc[0], stt = acc[1], sdt = acc[2];
  const double det = kk * stt - st * st;
  const double prod = kk * stt;
  const double scale = (prod < 1.0) ? 1.0 : prod;
  if (fabs(det) < 1e-12 * scale) return false;
  const double a0 = (stt * sd - st * sdt) / det;
  const double a1 = (kk * sdt - st * sd) / det;
  double e[1] = {0.0};
  for (int m = 0; m < F.rows; ++m) {
    const long long i = (long long)m * kFitLanes + F.lane;
    if (i >= F.k) break;
    double d, u, v;
    fit_get(F, m, i, d, u, v);
    const double t = c * v - s * u;
    const double r = d - a0 - a1 * t;
    e[0] += r * r;
  }
  cluster_sum<1>(F, e);
  out = LineFitD{a0, a1, phi, e[0], c, s};
  return true;
}

// estimate_roll, road_geometry.cpp:41-68 (golden section, f1 < f2 branch).
__device__ bool fit_golden(FitState& F, double lo, double hi, double tol, LineFitD& out) {
  const double sd = fit_sum_d(F);
  constexpr double g = 0.6180339887498949;
  double a = lo, b = hi;
  double x1 = b - g * (b - a), x2 = a + g * (b - a);
  LineFitD f;
  if (!fit_probe(F, x1, sd, f)) return false;
  double f1 = f.e0min;
  if (!fit_probe(F, x2, sd, f)) return false;
  double f2 = f.e0min;
  while (b - a > tol) {
    if (f1 < f2) {
      b = x2;
      x2 = x1;
      f2 = f1;
      x1 = b - g * (b - a);
      if (!fit_probe(F, x1, sd, f)) return false;
      f1 = f.e0min;
    } else {
      a = x1;
      x1 = x2;
      f1 = f2;
      x2 = a + g * (b - a);
      if (!fit_probe(F, x2, sd, f)) return false;
      f2 = f.e0min;
    }
  }
  return fit_probe(F, 0.5 * (a + b), sd, out);
}

// Stable cluster-wide compaction of the survivors of fit_road's trimming
// (road_geometry.cpp:83-97) into the scratch buffers.  Returns the new count.
__device__ long long fit_trim(FitState& F, const LineFitD& first, double rms) {
  cg::cluster_group cl = cg::this_cluster();
  FitShared& S = *F.S;
  const FitKParams& P = *F.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double lim = 3.0 * rms;
  const int rank = int(cl.block_rank());
  // keep bits of this thread's rows
  unsigned long long keep = 0;
  for (int m = 0; m < F.rows; ++m) {
    const long long i = (long long)m * kFitLanes + F.lane;
    if (i >= F.k) break;
    double d, u, v;
    fit_get(F, m, i, d, u, v);
    const double r = d - (first.a0 + first.a1 * (v * first.c - u * first.s));
    if (fabs(r) <= lim) keep |= 1ull << m;
  }
  // per-row counts of this CTA (rows <= kMaxRowsTrim enforced by the host)
  for (int m = 0; m < F.rows; ++m) {
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, (keep >> m) & 1ull);
    if (lane == 0) S.warp_cnt[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int q = 0; q < 32; ++q) t += S.warp_cnt[q];
      S.row_cnt[m] = t;
    }
    __syncthreads();
  }
  cl.sync();  // row counts of every CTA are visible
  if (threadIdx.x == 0) {
    long long base = 0;
    for (int m = 0; m < F.rows; ++m) {
      long long mine = 0;
      for (int r = 0; r < kFitCtas; ++r) {
        const int cnt = *cl.map_shared_rank(&S.row_cnt[m], r);
        if (r == rank) mine = base;
        base += cnt;
      }
      S.row_base[m] = int(mine);
    }
    S.bcast[0] = double(base);
  }
  cl.sync();  // peers finished reading row_cnt
  const long long kept = (long long)S.bcast[0];
  if (kept < 3 || kept == F.k) return kept;
  // scatter survivors in element order
  for (int m = 0; m < F.rows; ++m) {
    const bool kb = (keep >> m) & 1ull;
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, kb);
    if (lane == 0) S.warp_cnt[warp] = __popc(bal);
    __syncthreads();
    int woff = 0;
    for (int q = 0; q < warp; ++q) woff += S.warp_cnt[q];
    const long long i = (long long)m * kFitLanes + F.lane;
    if (kb && i < F.k) {
      const long long dst = S.row_base[m] + woff + __popc(bal & ((1u << lane) - 1u));
      double d, u, v;
      fit_get(F, m, i, d, u, v);
      if (F.compact) {
        P.scr_uv[dst] = uint32_t(u) | (uint32_t(v) << 16);
        P.scr_d[dst] = float(d);
      } else {
        P.scr_dd[dst] = d;
        P.scr_du[dst] = u;
        P.scr_dv[dst] = v;
      }
    }
    __syncthreads();
  }
  __threadfence();
  cl.sync();
  F.k = kept;
  F.g_uv = P.scr_uv;
  F.g_d = P.scr_d;
  F.g_dd = P.scr_dd;
  F.g_du = P.scr_du;
  F.g_dv = P.scr_dv;
  fit_stage(F);
  return kept;
}

__global__ void __launch_bounds__(kFitThreads, 1) k_fit(const __grid_constant__ FitKParams P) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ FitShared S;
  cg::cluster_group cl = cg::this_cluster();
  const FitRequest& R = P.r;
  FitState F;
  F.P = &P;
  F.S = &S;
  F.dyn = dyn;
  F.compact = R.compact;
  F.lane = int(cl.block_rank()) * kFitThreads + threadIdx.x;
  F.slot = 0;
  F.g_uv = R.obs.uv;
  F.g_d = R.obs.d;
  F.g_dd = R.dd;
  F.g_du = R.du;
  F.g_dv = R.dv;
  const bool failed_before = P.status->code != 0;
  F.k = R.compact ? (long long)(failed_before ? 0 : *R.obs.count) : R.k_host;
  FitOut res{};
  bool ok = !failed_before && F.k >= 3;
  if (ok) {
    fit_stage(F);
    LineFitD f{};
    long long used = F.k;
    if (R.mode == kFitLine) {
      const double sd = fit_sum_d(F);
      ok = fit_probe(F, R.phi, sd, f);
    } else if (R.mode == kEstimateRoll) {
      ok = fit_golden(F, R.lo, R.hi, R.tol, f);
    } else {
      ok = fit_golden(F, -R.hi, R.hi, R.tol, f);  // fit_road: first = fit_line(obs, m.phi)
      if (ok) {
        const double rms = sqrt(f.e0min / double(F.k));
        if (!(rms <= 0.0)) {
          const long long k0 = F.k;
          const long long kept = fit_trim(F, f, rms);
          if (kept >= 3 && kept != k0) {
            ok = fit_golden(F, -R.hi, R.hi, R.tol, f);
            used = kept;
          }
        }
      }
    }
    if (ok) {
      res.a0 = f.a0 * R.a0_scale;
      res.a1 = f.a1;
      res.phi = f.phi;
      res.e0min = f.e0min;
      res.used = used;
      res.model = DevModel{res.a0, f.a1, f.phi, f.c, f.s};
    }
  }
  if (!ok && !failed_before && cl.block_rank() == 0 && threadIdx.x == 0)
    set_status(P.status, RPD_EDEGENERATE, R.where);
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    if (!ok) res = FitOut{0.0, 0.0, 0.0, 0.0, 0, DevModel{0.0, 0.0, 0.0, 1.0, 0.0}};
    *R.out = res;
  }
  cl.sync();  // keep shared memory alive until every peer is done with DSMEM
}

void fit_dev(rpd_ctx* ctx, const FitRequest& req) {
  RPD_CK(cudaFuncSetAttribute(k_fit, cudaFuncAttributeMaxDynamicSharedMemorySize, kFitDynSmem));
  RPD_CK(cudaFuncSetAttribute(k_fit, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
  if (!req.compact && req.k_host > (long long)kMaxRowsTrim * kFitLanes)
    throw InvalidArg("fit: too many observations for the device fit (max 524288)");
  FitKParams P{};
  P.r = req;
  P.status = ctx->status;
  const long long scratch = req.compact ? (long long)kMaxRowsTrim * kFitLanes
                                        : std::max<long long>(req.k_host, 1);
  if (req.mode == kFitRoad) {
    if (req.compact) {
      P.scr_uv = ctx->ws.get<uint32_t>("fit_scr_uv", scratch);
      P.scr_d = ctx->ws.get<float>("fit_scr_d", scratch);
    } else {
      P.scr_dd = ctx->ws.get<double>("fit_scr_dd", scratch);
      P.scr_du = ctx->ws.get<double>("fit_scr_du", scratch);
      P.scr_dv = ctx->ws.get<double>("fit_scr_dv", scratch);
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kFitCtas);
  cfg.blockDim = dim3(kFitThreads);
  cfg.dynamicSmemBytes = kFitDynSmem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kFitCtas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RPD_CK(cudaLaunchKernelEx(&cfg, k_fit, P));
}

// --------------------------------------------------- transform_disparity --
__global__ void k_transform(const float* __restrict__ d1, int h, int w,
                            const DevModel* __restrict__ model, double delta,
                            float* __restrict__ d2, unsigned long long* __restrict__ clamped) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  bool clamp = false;
  if (u < w) {
    const size_t i = size_t(v) * w + u;
    const float x = d1[i];
    if (x != kInvalid) {
      const DevModel m = *model;
      double y = double(x) - road_at(m, double(u), double(v)) + delta;
      if (y < 0) {
        y = 0;
        clamp = true;
      }
      d2[i] = float(y);
    } else {
      d2[i] = x;
    }
  }
  const unsigned bal = __ballot_sync(0xFFFFFFFFu, clamp);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(clamped, (unsigned long long)__popc(bal));
}

void transform_disparity_dev(const float* d1, int h, int w, const DevModel* model, double delta_dt,
                             float* d2, unsigned long long* clamped, cudaStream_t st) {
  k_transform<<<dim3(cdiv(w, 128), h), 128, 0, st>>>(d1, h, w, model, delta_dt, d2, clamped);
  RPD_LAUNCH_CHECK();
}

}  // namespace rpdg
