// road.cu — road-model fit (fit_line / estimate_roll / fit_road), observation
// sampling and disparity transformation for sm_100a.
//
// Reference: /root/reference/proj/src/road_geometry.cpp:12-151.
//
// The whole fit_road (golden-section roll search, trimming, second search)
// runs inside ONE cooperative launch of 64 co-resident CTAs (one per SM,
// 128 summation lanes each). The observations (<= 524 288) are staged once in
// shared memory as exact doubles; the searches run on double-double moments
// (one pass), only the reported residual energies need further passes. Every
// pass ends in one grid-wide reduction whose CTA partials are exchanged
// through flag-tagged 64-bit words in L2 (no barrier, no host round trip).
//
// Reduction order (shared with the CPU oracle, oracle/rpd_oracle.cpp
// lane_tree_sum / moments): element i belongs to lane i mod 8192 (lane =
// CTA*128 + thread) and is added sequentially; lanes are then combined by an
// adjacent-pairwise binary tree (warp shuffles, CTA, then the 64 CTA
// partials). Eigen's own SIMD order (road_geometry.cpp:20-24, 37) is not
// reproducible without Eigen; the reference tests pin these sums to 1e-9.

#include <algorithm>


#include <cub/cub.cuh>

#include <mutex>
#include <vector>

#include "road.cuh"
#include "sincos_table.cuh"
#include "scan.cuh"


// k_fit's code size: with both input kinds' copies of the fit inlined it was
// ~44 k SASS instructions (~700 KB); one copy is 22 k.  Out-of-line helpers
// (RPD_FIT_NOINLINE_ON) shrink it to 11 k and the serial fit, but measured
// slower in the concurrent regime.
#ifndef RPD_FIT_NOINLINE_ON
#define RPD_FIT_NOINLINE_ON 0  // 1: 10.9 k instead of 22.4 k instructions, fit 0.111 -> 0.096 ms serial, but -1 % frames/s
#endif
#if RPD_FIT_NOINLINE_ON
#define RPD_FIT_NOINLINE __noinline__
#else
#define RPD_FIT_NOINLINE
#endif

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
// (-1)^n / (2n+1)! and (-1)^n / (2n)! as exact double-double constants.
constexpr int kTaylorTerms = 18;  // enough for |x| <= pi/4 at ~1e-36
__constant__ double c_sin_hi[kTaylorTerms] = {1.0, -0.16666666666666666, 0.008333333333333333, -0.0001984126984126984, 2.7557319223985893e-06, -2.505210838544172e-08, 1.6059043836821613e-10, -7.647163731819816e-13, 2.8114572543455206e-15, -8.22063524662433e-18, 1.9572941063391263e-20, -3.868170170630684e-23, 6.446950284384474e-26, -9.183689863795546e-29, 1.1309962886447716e-31, -1.216125041553518e-34, 1.151633562077195e-37, -9.67759295863189e-41};
__constant__ double c_sin_lo[kTaylorTerms] = {0.0, -9.25185853854297e-18, 1.1564823173178714e-19, -1.7209558293420705e-22, -1.858393274046472e-22, 1.448814070935912e-24, 1.2585294588752098e-26, -7.03872877733453e-30, 1.6508842730861433e-31, -2.2141894119604265e-34, -1.3643503830087908e-36, 8.843177655482344e-40, -1.9330404233703465e-42, -1.4303150396787322e-45, 1.0498015412959506e-47, -5.586290567888806e-51, -6.09957445788454e-54, -3.202295548645562e-57};
__constant__ double c_cos_hi[kTaylorTerms] = {1.0, -0.5, 0.041666666666666664, -0.001388888888888889, 2.48015873015873e-05, -2.755731922398589e-07, 2.08767569878681e-09, -1.1470745597729725e-11, 4.779477332387385e-14, -1.5619206968586225e-16, 4.110317623312165e-19, -8.896791392450574e-22, 1.6117375710961184e-24, -2.4795962632247976e-27, 3.279889237069838e-30, -3.7699876288159054e-33, 3.8003907548547434e-36, -3.387157535521162e-39};
__constant__ double c_cos_lo[kTaylorTerms] = {0.0, 0.0, 2.3129646346357427e-18, 5.300543954373577e-20, 2.1511947866775882e-23, -2.3767714622250297e-23, -1.20734505911326e-25, -2.0655512752830745e-28, 4.399205485834081e-31, -1.1910679660273754e-32, 1.4412973378659527e-36, 7.911402614872376e-38, -3.6846573564509766e-41, 1.2953730964765229e-43, 1.5117542744029879e-46, -2.5870347832750324e-49, 1.7457158024652518e-52, -5.09056148151085e-56};
}  // namespace

// Correctly rounded sin/cos (with overwhelming probability).  Fast path for
// the roll angles (|x| <= 0.75): x = a_k + r with a_k = k/256 (r exact,
// |r| <= 2^-9).  sin(r) = r - r^3/6 + O(r^5) and cos(r) = 1 - r^2/2 + O(r^4):
// the leading terms in double-double from the exact r^2 = p + e (two_prod),
// the tails (< 2^-38 |r| and < 2^-40) in double, so sin/cos(r) are
// double-doubles good to ~2^-90 relative; the addition formulas with
// tabulated double-double sin/cos(a_k) (sincos_table.cuh) combine them.  A
// short dependent chain: the roll search's latency (tree batches, final
// probes) is dominated by this function.  Otherwise: reduction by pi/2 and an
// 18-term double-double series.
__device__ RPD_FIT_NOINLINE void dd_sincos(double x, double* s_out, double* c_out) {
  if (fabs(x) <= 0.75) {
    if (x == 0.0) {  // keeps the sign of zero
      *s_out = x;
      *c_out = 1.0;
      return;
    }
    const double kf = rint(x * 256.0);
    const double r = x - kf * 0.00390625;  // exact
    const double p = r * r;
    const double e = __fma_rn(r, r, -p);  // r^2 = p + e exactly
    // sin(r) = r - r * (r^2/3!) + r * p * S, S = r^2/5! - r^4/7! + r^6/9!: the
    // r^3 term in double-double from the exact r^2, the rest (< 2^-38 |r|) in
    // double
    const DD d6 = dd_mul(DD{p, e}, DD{0.16666666666666666, 9.25185853854297e-18});
    const DD t3 = dd_mul(d6, DD{r, 0.0});
    const double S =
        p * (0.008333333333333333 + p * (-0.0001984126984126984 + p * 2.7557319223985893e-06));
    const DD sr = dd_add(dd_add(DD{r, 0.0}, DD{-t3.hi, -t3.lo}), DD{(r * p) * S, 0.0});
    // cos(r) = 1 - (p + e)/2 + Q, Q = r^4/4! - r^6/6! + r^8/8!
    const double Q = (p * p) * (0.041666666666666664 +
                                p * (-0.001388888888888889 + p * 2.48015873015873e-05));
    const DD c0 = two_sum(1.0, -0.5 * p);
    const DD cr = quick_two_sum(c0.hi, c0.lo + (Q - 0.5 * e));
    const int idx = int(kf) + kSinTab256Half;
    const DD sa = {c_t256_sin_hi[idx], c_t256_sin_lo[idx]};
    const DD ca = {c_t256_cos_hi[idx], c_t256_cos_lo[idx]};
    const DD sx = dd_add(dd_mul(sa, cr), dd_mul(ca, sr));
    const DD m = dd_mul(sa, sr);
    const DD cx = dd_add(dd_mul(ca, cr), DD{-m.hi, -m.lo});
    *s_out = sx.hi;
    *c_out = cx.hi;
    return;
  }
  const DD pio2 = {1.5707963267948966, 6.123233995736766e-17};
  const double kf = rint(x / pio2.hi);
  DD r = {x, 0.0};
  if (kf != 0.0) {
    const DD kp = dd_mul(pio2, DD{kf, 0.0});
    r = dd_add(r, DD{-kp.hi, -kp.lo});
  }
  const DD x2 = dd_mul(r, r);
  DD ps = {c_sin_hi[kTaylorTerms - 1], c_sin_lo[kTaylorTerms - 1]};
  DD pc = {c_cos_hi[kTaylorTerms - 1], c_cos_lo[kTaylorTerms - 1]};
#pragma unroll
  for (int n = kTaylorTerms - 2; n >= 0; --n) {
    ps = dd_add(dd_mul(ps, x2), DD{c_sin_hi[n], c_sin_lo[n]});
    pc = dd_add(dd_mul(pc, x2), DD{c_cos_hi[n], c_cos_lo[n]});
  }
  const DD ss = dd_mul(ps, r), cs = pc;
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


// Sample flag of pixel p (road_geometry.cpp:112-117): in the ROI and a valid
// disparity.  load8 feeds the scan; the scatter re-evaluates it.
struct SampleFlagIn {
  const float* d1;
  int w;
  RoiPred r;
  __device__ __forceinline__ int at(int u, int v, long long p) const {
    return (u >= r.u0 && u < r.u1 && v >= r.v0 && v < r.v1 && d1[p] != kInvalid) ? 1 : 0;
  }
  __device__ __forceinline__ void load8(long long base, long long n, int (&f)[8]) const {
    int v = int(base / w), u = int(base - (long long)v * w);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      f[k] = base + k < n ? at(u, v, base + k) : 0;
      if (++u == w) {
        u = 0;
        ++v;
      }
    }
  }
};

__global__ void k_sample_scatter(const SampleFlagIn in, const int* __restrict__ pos, long long n,
                                 int* __restrict__ list) {
  // four pixels per thread (launched with max(1, cdiv(n, 1024)) blocks of 256)
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 >= n) return;
  int v = int(p0 / in.w), u = int(p0 - (long long)v * in.w);
  for (long long p = p0; p < min(n, p0 + 4); ++p) {
    if (in.at(u, v, p)) list[pos[p]] = int(p);
    if (++u == in.w) {
      u = 0;
      ++v;
    }
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
  int* pos = ctx->ws.get<int>("so_pos", n);
  int* list = ctx->ws.get<int>("so_list", n);
  int* total = ctx->ws.get<int>("so_total", 1);
  // flags -> scan (+ total) -> scatter, the flags evaluated in place
  const SampleFlagIn in{d1, w, r};
  scan_exclusive(ctx, in, pos, n, total);
  k_sample_scatter<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(in, pos, n, list);
  RPD_LAUNCH_CHECK();
  const long long gmax = std::min<long long>(cap, n);
  k_sample_gather<<<std::max(1, cdiv(gmax, 256)), 256, 0, st>>>(
      d1, w, list, total, cap, obs.uv, obs.d, obs.count, ctx->status, where);
  RPD_LAUNCH_CHECK();
}

// ----------------------------------------------------------- fit kernel ----
// One cooperative grid of kFitCtas CTAs (co-resident, one per SM) runs a whole
// fit.  CTA c owns lanes [c*kFitSweep, (c+1)*kFitSweep) of the 8192 summation
// lanes; its observations (rows m: element m*8192 + lane) are staged once in
// shared memory as exact doubles.
//
// The golden-section search evaluates fit_line's energy from the observation
// moments (n, Σu, Σv, Σd, Σuu, Σvv, Σuv, Σdu, Σdv, Σdd) in double-double
// arithmetic: the products are exact (two_prod) and the moments are summed in
// double-double in the fixed lane order, so one pass over the data replaces
// one pass per probe and the expanded energy keeps ~30 significant digits
// (the cancellation the reference avoids with its residual form,
// road_geometry.cpp:35-37, is harmless at that precision).  The reported
// e0min of every final fit_line is still the residual form in double, summed
// in the lane order.  Trimming (road_geometry.cpp:83-97) masks elements in
// place; the survivors keep their lanes.  A fit_road is therefore four
// grid-wide reductions (moments, residual, survivor moments, residual); each
// CTA combines the kFitCtas CTA partials with the same pairwise tree, so all CTAs
// hold bit-identical sums and run the scalar search redundantly.
// oracle/rpd_oracle.cpp restates exactly this arithmetic.
#ifndef RPD_FIT_CTAS
#define RPD_FIT_CTAS 64  // 64 x 128 threads: +1 % frames/s and a faster serial fit than 128 x 64
#endif
constexpr int kFitCtas = RPD_FIT_CTAS;
constexpr int kFitSweep = 8192 / kFitCtas;         // summation lanes per CTA
constexpr int kFitSweepWarps = kFitSweep / 32;
constexpr int kFitThreads = kFitSweep;
constexpr int kFitLanes = kFitCtas * kFitSweep;    // == oracle kFitLanes (8192)
// rows of staged observations (64: 524288 observations), within ~200 KB of shared memory
constexpr int kMaxRowsSmem = (200 * 1024) / (kFitSweep * 3 * 8);
constexpr int kMaxRows = kMaxRowsSmem < 64 ? kMaxRowsSmem : 64;
constexpr int kMaxNV = 20;                         // doubles per reduction (10 DD moments)
constexpr int kPartReplicas = 8;  // copies of the CTA partials (spreads the polling over L2)
constexpr int kPartWords = 2 * kPartReplicas * kFitCtas * kMaxNV * 2;
static_assert((kFitSweepWarps & (kFitSweepWarps - 1)) == 0, "warps");
static_assert((kFitCtas & (kFitCtas - 1)) == 0 && kFitCtas / 2 <= kFitSweep, "ctas");

// dynamic shared memory for `rows` staged rows (SoA doubles d | u | v)
__host__ __device__ constexpr int fit_dyn_smem(int rows) {
  return rows * kFitSweep * 3 * int(sizeof(double));
}

struct FitKParams {
  FitRequest r;
  DevStatus* status;
  unsigned long long* part;  // [2][kPartReplicas][kFitCtas][kMaxNV][2] flag-tagged partials
  int trace;                 // debug (RPD_FIT_TRACE=1): per-phase clock64 trace of CTA 0
  int rows_cap;              // staged rows the dynamic shared memory holds
};

struct FitShared {
  double warp_part[kFitSweepWarps][kMaxNV];
  double red[kFitSweepWarps][kMaxNV];
  DD g_e[kFitThreads];  // golden-search decision tree: node energies
  int g_bad[kFitThreads];  // node probe degenerate
  long long tr[512];
  int ntr;
};

struct FitState {
  const FitKParams* P;
  FitShared* S;
  double* e;     // staged SoA doubles: d | u | v, each [rows_cap][kFitSweep]
  int rstride;   // rows_cap * kFitSweep
  long long k;
  int rows;      // rows this lane owns
  int lane;
  unsigned calls;  // grid reductions so far (the exchange flag)
};

__device__ __forceinline__ void fit_tr(FitState& F, int tag) {
  if (F.P->trace && blockIdx.x == 0 && threadIdx.x == 0 && F.S->ntr < 512)
    F.S->tr[F.S->ntr++] = ((long long)tag << 48) | (clock64() & 0xFFFFFFFFFFFFll);
}

constexpr unsigned kSpinLimit = 1u << 24;  // ~seconds: a lost peer traps, never hangs

// ----- double-double arithmetic (Dekker / Knuth; restated in the oracle) ----
__device__ __forceinline__ DD dd_add_d(DD a, double b) {
  DD s = two_sum(a.hi, b);
  s.lo += a.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DD dd_neg(DD a) { return DD{-a.hi, -a.lo}; }
__device__ __forceinline__ DD dd_sub(DD a, DD b) { return dd_add(a, dd_neg(b)); }
__device__ __forceinline__ DD dd_mul_d(DD a, double b) {
  DD p = two_prod(a.hi, b);
  p.lo = __fma_rn(a.lo, b, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
// product with fused low-order terms (the fit's arithmetic; dd_sincos keeps dd_mul)
__device__ __forceinline__ DD dd_mulf(DD a, DD b) {
  DD p = two_prod(a.hi, b.hi);
  p.lo = __fma_rn(a.hi, b.lo, p.lo);
  p.lo = __fma_rn(a.lo, b.hi, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ DD dd_div(DD a, DD b) {
  const double q1 = a.hi / b.hi;
  DD r = dd_sub(a, dd_mul_d(b, q1));
  const double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul_d(b, q2));
  const double q3 = r.hi / b.hi;
  return dd_add_d(quick_two_sum(q1, q2), q3);
}
__device__ __forceinline__ bool dd_lt(DD a, DD b) {
  return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}

// Moments in double-double: su, sv, sd, suu, svv, suv, sdu, sdv, sdd, n.
constexpr int kNMom = 10;
struct Moments {
  DD m[kNMom];
};

// Stage the first k elements of the request's input into shared memory.
template <bool COMPACT>
__device__ void fit_stage(FitState& F, const FitRequest& R) {
  const int rows_total = int((F.k + kFitLanes - 1) / kFitLanes);
  const long long full = F.k / kFitLanes;
  F.rows = int(full) + (F.lane < F.k - full * kFitLanes ? 1 : 0);
  constexpr int U = 8;  // loads in flight per thread
  for (int m0 = 0; m0 < rows_total; m0 += U) {
    double d[U], u[U], v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long i = (long long)(m0 + j) * kFitLanes + F.lane;
      if (m0 + j < F.rows) {
        if (COMPACT) {
          const uint32_t uv = __ldcg(R.obs.uv + i);
          u[j] = double(uv & 0xFFFFu);
          v[j] = double(uv >> 16);
          d[j] = double(__ldcg(R.obs.d + i));
        } else {
          d[j] = __ldcg(R.dd + i);
          u[j] = __ldcg(R.du + i);
          v[j] = __ldcg(R.dv + i);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (m0 + j < F.rows) {
        const int o = (m0 + j) * kFitSweep + threadIdx.x;
        F.e[o] = d[j];
        F.e[F.rstride + o] = u[j];
        F.e[2 * F.rstride + o] = v[j];
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void fit_get(const FitState& F, int m, double& d, double& u, double& v) {
  const int o = m * kFitSweep + threadIdx.x;
  d = F.e[o];
  u = F.e[F.rstride + o];
  v = F.e[2 * F.rstride + o];
}

// Grid-wide sum of NV values (doubles, or NV/2 double-doubles when DD) in the
// fixed adjacent-pairwise lane order.  CTA partials are exchanged without a
// barrier: each double travels as two 64-bit words (flag << 32 | 32 data
// bits), each single-copy atomic, so a reader that sees the call's flag in
// both words holds the value (the LL protocol of NCCL).  Slots alternate by
// call parity: a CTA rewrites a slot only after every CTA has published the
// following call, i.e. finished reading this one.
template <int NV, bool DDV>
__device__ RPD_FIT_NOINLINE void grid_sum(FitState& F, double (&x)[NV]) {
  static_assert(NV <= kMaxNV && (!DDV || NV % 2 == 0), "values");
  // Every step below runs element by element (one double, or one
  // double-double when DDV): the per-element trees are those of the
  // all-elements formulation, but only one element's temporaries are live
  // (the register footprint sets how many other CTAs share the fit's SMs).
  constexpr int ST = DDV ? 2 : 1;
  FitShared& S = *F.S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned flag = ++F.calls;
  unsigned long long* part =
      F.P->part + size_t(flag & 1u) * (kPartReplicas * kFitCtas * kMaxNV * 2);
  const unsigned long long ftag = (unsigned long long)flag << 32;
  // a[0..ST) += b[0..ST)
  auto plus = [](double* a, const double* b) {
    if (DDV) {
      const DD r = dd_add(DD{a[0], a[1]}, DD{b[0], b[1]});
      a[0] = r.hi;
      a[1] = r.lo;
    } else {
      a[0] += b[0];
    }
  };
  fit_tr(F, 3);
#pragma unroll
  for (int q = 0; q < NV; q += ST) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      double o[ST];
#pragma unroll
      for (int c = 0; c < ST; ++c) o[c] = __shfl_down_sync(0xFFFFFFFFu, x[q + c], off);
      plus(&x[q], o);
    }
  }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) S.warp_part[warp][q] = x[q];
  __syncthreads();
  if (threadIdx.x < NV) {  // thread q publishes value q of the CTA partial
    const int q = threadIdx.x;
    const int e = q - q % ST;
    double p[kFitSweepWarps][ST];
#pragma unroll
    for (int r = 0; r < kFitSweepWarps; ++r)
#pragma unroll
      for (int c = 0; c < ST; ++c) p[r][c] = S.warp_part[r][e + c];
#pragma unroll
    for (int width = 1; width < kFitSweepWarps; width *= 2)
#pragma unroll
      for (int j = 0; j < kFitSweepWarps; j += 2 * width) plus(p[j], p[j + width]);
    const double val = p[0][q - e];
    const unsigned long long bits = (unsigned long long)__double_as_longlong(val);
    const unsigned long long w0 = ftag | (bits & 0xFFFFFFFFull), w1 = ftag | (bits >> 32);
#pragma unroll
    for (int rep = 0; rep < kPartReplicas; ++rep) {
      unsigned long long* dst = part + ((size_t(rep) * kFitCtas + blockIdx.x) * kMaxNV + q) * 2;
      asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(w0), "l"(w1)
                   : "memory");
    }
  }
  fit_tr(F, 4);
  // combine the kFitCtas partials: thread j holds pair (2j, 2j+1)
  constexpr int kPairs = kFitCtas / 2;
  if (threadIdx.x < kPairs) {
    const unsigned long long* src =
        part + (size_t(blockIdx.x % kPartReplicas) * kFitCtas + 2 * threadIdx.x) * kMaxNV * 2;
    unsigned spins = 0;
    constexpr int kW = kPairs < 32 ? kPairs : 32;
    constexpr unsigned kWMask = kW == 32 ? 0xFFFFFFFFu : ((1u << kW) - 1u);
#pragma unroll 1
    for (int q = 0; q < NV; q += ST) {
      double y[ST], b[ST];
      while (true) {  // element q of both partials, polled until the call's flag shows
        unsigned long long w[2][ST][2];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int t = 0; t < ST; ++t)
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                         : "=l"(w[c][t][0]), "=l"(w[c][t][1])
                         : "l"(src + (c * kMaxNV + q + t) * 2)
                         : "memory");
        bool ready = true;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int t = 0; t < ST; ++t)
            ready &= (w[c][t][0] >> 32) == flag && (w[c][t][1] >> 32) == flag;
        if (ready) {
#pragma unroll
          for (int t = 0; t < ST; ++t) {
            y[t] = __longlong_as_double(
                (long long)((w[0][t][0] & 0xFFFFFFFFull) | (w[0][t][1] << 32)));
            b[t] = __longlong_as_double(
                (long long)((w[1][t][0] & 0xFFFFFFFFull) | (w[1][t][1] << 32)));
          }
          break;
        }
        if (++spins > kSpinLimit) __trap();
      }
      plus(y, b);
#pragma unroll
      for (int off = 1; off < kW; off <<= 1) {
        double o[ST];
#pragma unroll
        for (int t = 0; t < ST; ++t) o[t] = __shfl_down_sync(kWMask, y[t], off);
        plus(y, o);
      }
      if (lane == 0)
#pragma unroll
        for (int t = 0; t < ST; ++t) S.red[warp][q + t] = y[t];
    }
    fit_tr(F, 41);
  }
  __syncthreads();
  constexpr int kRW = (kPairs + 31) / 32;
#pragma unroll
  for (int q = 0; q < NV; q += ST) {
    double p[kRW][ST];
#pragma unroll
    for (int r = 0; r < kRW; ++r)
#pragma unroll
      for (int t = 0; t < ST; ++t) p[r][t] = S.red[r][q + t];
#pragma unroll
    for (int width = 1; width < kRW; width *= 2)
#pragma unroll
      for (int j = 0; j < kRW; j += 2 * width) plus(p[j], p[j + width]);
#pragma unroll
    for (int t = 0; t < ST; ++t) x[q + t] = p[0][t];
  }
  __syncthreads();  // S.red / S.warp_part reusable
  fit_tr(F, 5);
}

// Moments of the elements whose row bit is set in `mask` (this lane's rows).
__device__ RPD_FIT_NOINLINE Moments fit_moments(FitState& F, unsigned long long mask) {
  DD acc[kNMom];
#pragma unroll
  for (int q = 0; q < kNMom; ++q) acc[q] = DD{0.0, 0.0};
  for (int m = 0; m < F.rows; ++m) {
    if (!((mask >> m) & 1ull)) continue;
    double d, u, v;
    fit_get(F, m, d, u, v);
    acc[0] = dd_add_d(acc[0], u);
    acc[1] = dd_add_d(acc[1], v);
    acc[2] = dd_add_d(acc[2], d);
    acc[3] = dd_add(acc[3], two_prod(u, u));
    acc[4] = dd_add(acc[4], two_prod(v, v));
    acc[5] = dd_add(acc[5], two_prod(u, v));
    acc[6] = dd_add(acc[6], two_prod(d, u));
    acc[7] = dd_add(acc[7], two_prod(d, v));
    acc[8] = dd_add(acc[8], two_prod(d, d));
    acc[9] = dd_add_d(acc[9], 1.0);
  }
  double x[2 * kNMom];
#pragma unroll
  for (int q = 0; q < kNMom; ++q) {
    x[2 * q] = acc[q].hi;
    x[2 * q + 1] = acc[q].lo;
  }
  grid_sum<2 * kNMom, true>(F, x);
  Moments M;
#pragma unroll
  for (int q = 0; q < kNMom; ++q) M.m[q] = DD{x[2 * q], x[2 * q + 1]};
  return M;
}

// fit_line at (c, s) = (cos phi, sin phi) from the moments
// (road_geometry.cpp:16-37), in double-double: the angle-dependent sums
// st = c Sv - s Su, stt = c^2 Svv - 2cs Suv + s^2 Suu, sdt = c Sdv - s Sdu,
// det = n stt - st^2 (singular test as :26-29), and either the minimal
// energy  E = Sdd - (stt Sd^2 - 2 st Sd sdt + n sdt^2) / det  (the search) or
// the coefficients a0 = (stt Sd - st sdt)/det, a1 = (n sdt - st Sd)/det.
struct LineSums {
  DD N, T1, T2, TD, det;
};
__device__ __forceinline__ bool line_sums(const Moments& M, double c, double s, LineSums& o) {
  o.N = M.m[9];
  const DD cc = two_prod(c, c), ss = two_prod(s, s), cs = two_prod(c, s);
  o.T1 = dd_sub(dd_mul_d(M.m[1], c), dd_mul_d(M.m[0], s));
  o.T2 = dd_add(dd_sub(dd_mulf(cc, M.m[4]), dd_mul_d(dd_mulf(cs, M.m[5]), 2.0)),
                dd_mulf(ss, M.m[3]));
  o.TD = dd_sub(dd_mul_d(M.m[7], c), dd_mul_d(M.m[6], s));
  const DD nT2 = dd_mulf(o.N, o.T2);
  o.det = dd_sub(nT2, dd_mulf(o.T1, o.T1));
  const double scale = nT2.hi < 1.0 ? 1.0 : nT2.hi;
  return !(fabs(o.det.hi) < 1e-12 * scale);
}
__device__ RPD_FIT_NOINLINE bool line_energy(const Moments& M, double c, double s, DD& e) {
  LineSums L;
  if (!line_sums(M, c, s, L)) return false;
  const DD D1 = M.m[2];
  DD q = dd_mulf(L.T2, dd_mulf(D1, D1));
  q = dd_sub(q, dd_mul_d(dd_mulf(dd_mulf(L.T1, D1), L.TD), 2.0));
  q = dd_add(q, dd_mulf(L.N, dd_mulf(L.TD, L.TD)));
  e = dd_sub(M.m[8], dd_div(q, L.det));
  return true;
}
__device__ RPD_FIT_NOINLINE bool line_coef(const Moments& M, double c, double s, DD& a0, DD& a1) {
  LineSums L;
  if (!line_sums(M, c, s, L)) return false;
  const DD D1 = M.m[2];
  a0 = dd_div(dd_sub(dd_mulf(L.T2, D1), dd_mulf(L.T1, L.TD)), L.det);
  a1 = dd_div(dd_sub(dd_mulf(L.N, L.TD), dd_mulf(L.T1, D1)), L.det);
  return true;
}

struct LineFitD {
  double a0, a1, phi, e0min, c, s;
};

// Final fit_line at phi: a0/a1 from the moments (rounded), e0min in the
// reference's residual form over the masked elements (one grid reduction).
__device__ bool fit_line_final(FitState& F, const Moments& M, double phi, double c, double s,
                               unsigned long long mask, LineFitD& out) {
  DD A0, A1;
  if (!line_coef(M, c, s, A0, A1)) return false;
  fit_tr(F, 13);
  const double a0 = A0.hi, a1 = A1.hi;
  double acc[1] = {0.0};
  for (int m = 0; m < F.rows; ++m) {
    if (!((mask >> m) & 1ull)) continue;
    double d, u, v;
    fit_get(F, m, d, u, v);
    const double t = c * v - s * u;
    const double r = d - a0 - a1 * t;
    acc[0] += r * r;
  }
  grid_sum<1, false>(F, acc);
  out = LineFitD{a0, a1, phi, acc[0], c, s};
  return true;
}

// Golden-section bracket state of estimate_roll (road_geometry.cpp:41-68).
struct GState {
  double a, b, x1, x2;
};
constexpr double kGolden = 0.6180339887498949;

// The f1 < f2 (br) / else update; returns the newly evaluated point.
__device__ __forceinline__ double g_advance(GState& s, bool br) {
  if (br) {
    s.b = s.x2;
    s.x2 = s.x1;
    s.x1 = s.b - kGolden * (s.b - s.a);
    return s.x1;
  }
  s.a = s.x1;
  s.x1 = s.x2;
  s.x2 = s.a + kGolden * (s.b - s.a);
  return s.x2;
}

// estimate_roll on moments.  The search walks a binary decision tree: from
// the current state, the next point is fixed (the pending comparison is
// known) and every later point depends on the comparisons in between.  Each
// batch evaluates a 63-node subtree (6 iterations) in parallel — thread t of
// the CTA takes node t (level floor(log2 t), path bits t - 2^level, MSB
// first) and computes its point's sin/cos and energy — into a shared table;
// the walk then only compares.  The first batch holds the two initial probes
// (nodes 0, 1) and the 62 nodes of the five iterations after them.  All
// threads (and CTAs) follow the same decisions.  Returns the final midpoint
// and its sin/cos.
__device__ bool fit_golden(FitState& F, const Moments& M, double lo, double hi, double tol,
                           double& phi, double& cphi, double& sphi) {
  static_assert((kFitThreads & (kFitThreads - 1)) == 0 && kFitThreads >= 64, "tree batch size");
  constexpr int kTreeLv = kFitThreads == 64 ? 6 : (kFitThreads == 128 ? 7 : (kFitThreads == 256 ? 8 : 9));
  FitShared& S = *F.S;
  const int t = threadIdx.x;
  GState st{lo, hi, hi - kGolden * (hi - lo), lo + kGolden * (hi - lo)};
  auto eval_node = [&](double x) {
    double bs, bc;
    dd_sincos(x, &bs, &bc);
    DD e{0.0, 0.0};
    const bool ok = line_energy(M, bc, bs, e);
    S.g_e[t] = e;
    S.g_bad[t] = ok ? 0 : 1;
  };
  // batch 0: initial probes and the tree below them
  {
    double x;
    if (t < 2) {
      x = t == 0 ? st.x1 : st.x2;
    } else {
      GState g = st;
      const int lv = 31 - __clz(t);
      const int bits = t - (1 << lv);
      x = 0.0;
      for (int j = lv - 1; j >= 0; --j) x = g_advance(g, ((bits >> j) & 1) != 0);
    }
    fit_tr(F, 6);
    eval_node(x);
    __syncthreads();
    fit_tr(F, 8);
  }
  if (S.g_bad[0] | S.g_bad[1]) return false;
  DD f1 = S.g_e[0], f2 = S.g_e[1];
  int node = 1, left = kTreeLv - 1;  // the tree below the probes: children of virtual node 1
  bool br = dd_lt(f1, f2);
  node = 2 * node + (br ? 1 : 0);
  while (st.b - st.a > tol) {
    if (left == 0) {  // new batch from the current state (br known)
      __syncthreads();  // everyone is done with the previous table
      GState g = st;
      double x = g_advance(g, br);
      const int lv = t == 0 ? 0 : 31 - __clz(t);
      const int bits = t - (1 << lv);
      for (int j = lv - 1; j >= 0; --j) x = g_advance(g, ((bits >> j) & 1) != 0);
      fit_tr(F, 6);
      eval_node(x);
      __syncthreads();
      fit_tr(F, 8);
      node = 1;
      left = kTreeLv;
    }
    if (S.g_bad[node]) return false;  // fit_line throws on this probe
    g_advance(st, br);
    if (br)
      f2 = f1;
    else
      f1 = f2;
    if (br)
      f1 = S.g_e[node];
    else
      f2 = S.g_e[node];
    --left;
    br = dd_lt(f1, f2);
    node = 2 * node + (br ? 1 : 0);
  }
  fit_tr(F, 10);
  phi = 0.5 * (st.a + st.b);
  dd_sincos(phi, &sphi, &cphi);
  fit_tr(F, 11);
  __syncthreads();  // the table is free for the next search
  fit_tr(F, 12);
  return true;
}

// The fit after staging (one copy for both input kinds: the kernel's code
// size is what the instruction caches of the SMs it shares see).
__device__ RPD_FIT_NOINLINE void fit_run(FitState& F, const FitKParams& P, FitOut& res, bool& ok) {
  const FitRequest& R = P.r;
  fit_tr(F, 1);
  const unsigned long long all = F.rows >= 64 ? ~0ull : ((1ull << F.rows) - 1ull);
  const Moments M = fit_moments(F, all);
  LineFitD f{};
  long long used = F.k;
  double phi = 0.0, c = 1.0, s = 0.0;
  if (R.mode == kFitLine) {
    phi = R.phi;
    dd_sincos(phi, &s, &c);
    ok = fit_line_final(F, M, phi, c, s, all, f);
  } else {
    const double lo = R.mode == kEstimateRoll ? R.lo : -R.hi;
    ok = fit_golden(F, M, lo, R.hi, R.tol, phi, c, s) && fit_line_final(F, M, phi, c, s, all, f);
    fit_tr(F, 2);
    if (ok && R.mode == kFitRoad) {
      const double rms = sqrt(f.e0min / double(F.k));
      if (!(rms <= 0.0)) {
        // road_geometry.cpp:83-97: keep |d - road(u, v)| <= 3 rms, in place
        const double lim = 3.0 * rms;
        unsigned long long keep = 0;
        for (int m = 0; m < F.rows; ++m) {
          double d, u, v;
          fit_get(F, m, d, u, v);
          const double r = d - (f.a0 + f.a1 * (v * f.c - u * f.s));
          if (fabs(r) <= lim) keep |= 1ull << m;
        }
        const Moments M2 = fit_moments(F, keep);
        const long long kept = (long long)M2.m[9].hi;
        if (kept >= 3 && kept != F.k) {
          ok = fit_golden(F, M2, -R.hi, R.hi, R.tol, phi, c, s) &&
               fit_line_final(F, M2, phi, c, s, keep, f);
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

#ifndef RPD_FIT_MINB
#define RPD_FIT_MINB 8  // 128 registers: the fit shares its SMs with other streams (+1.5 % frames/s over 1)
#endif
__global__ void __launch_bounds__(kFitThreads, RPD_FIT_MINB * 64 / kFitThreads) k_fit(const __grid_constant__ FitKParams P) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ FitShared S;
  const FitRequest& R = P.r;
  FitState F;
  F.P = &P;
  F.S = &S;
  F.e = reinterpret_cast<double*>(dyn);
  F.rstride = P.rows_cap * kFitSweep;
  F.lane = int(blockIdx.x) * kFitSweep + int(threadIdx.x);
  F.calls = 0;
  if (threadIdx.x == 0) S.ntr = 0;
  __syncthreads();
  fit_tr(F, 0);
  const bool failed_before = P.status->code != 0;
  F.k = R.compact ? (long long)(failed_before ? 0 : *R.obs.count) : R.k_host;
  FitOut res{};
  bool ok = !failed_before && F.k >= 3;
  if (ok && F.k > (long long)P.rows_cap * kFitLanes) {  // host sizes rows_cap from the cap
    ok = false;
    if (blockIdx.x == 0 && threadIdx.x == 0) set_status(P.status, RPD_EINVAL, R.where, F.k);
  }
  if (ok) {
    if (R.compact)
      fit_stage<true>(F, R);
    else
      fit_stage<false>(F, R);
    fit_run(F, P, res, ok);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (!ok && !failed_before) set_status(P.status, RPD_EDEGENERATE, R.where);
    if (!ok) res = FitOut{0.0, 0.0, 0.0, 0.0, 0, DevModel{0.0, 0.0, 0.0, 1.0, 0.0}};
    *R.out = res;
  }
  fit_tr(F, 9);
  if (P.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = S.tr[0] & 0xFFFFFFFFFFFFll;
    for (int i = 0; i < S.ntr; ++i) {
      const long long t = S.tr[i] & 0xFFFFFFFFFFFFll;
      printf("FITTR %d %d %lld\n", i, int(S.tr[i] >> 48), t - t0);
    }
  }
}

void fit_dev(rpd_ctx* ctx, const FitRequest& req) {
  // Function attributes are per device: one setup per device, thread-safe
  // (contexts on several devices and host threads share this code).
  static std::mutex attr_mu;
  static std::vector<char> attr_done;
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    if ((int)attr_done.size() <= ctx->device) attr_done.resize(ctx->device + 1, 0);
    if (!attr_done[ctx->device]) {
      RPD_CK(cudaFuncSetAttribute(k_fit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  fit_dyn_smem(kMaxRows)));
      int per_sm = 0;
      RPD_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit, kFitThreads,
                                                           fit_dyn_smem(kMaxRows)));
      if (per_sm * ctx->sm_count < kFitCtas)
        throw CudaFail("fit: device cannot co-schedule the fit grid");
      attr_done[ctx->device] = 1;
    }
  }
  if (!req.compact && req.k_host > (long long)kMaxRows * kFitLanes)
    throw InvalidArg("fit: too many observations for the device fit (max " +
                     std::to_string((long long)kMaxRows * kFitLanes) + ")");
  // Shared memory sized to the request's observation cap (13 rows for the
  // pipeline's 100 000).  With the moment-based search the fit makes only
  // four grid-wide exchanges, so sharing its SMs with other streams' CTAs now
  // pays (measured +1.7 % frames/s over reserving the 64-row maximum; the
  // opposite held for the per-probe design, profiles/r1_notes.md).
  const long long kcap = req.compact ? (req.kmax > 0 ? req.kmax : (long long)kMaxRows * kFitLanes)
                                     : req.k_host;
  const int rows_cap = int(std::min<long long>(
      kMaxRows, std::max<long long>(1, (kcap + kFitLanes - 1) / kFitLanes)));
  FitKParams P{};
  P.r = req;
  P.status = ctx->status;
  P.rows_cap = rows_cap;
  static const bool trace = debug_knob("RPD_FIT_TRACE") != nullptr;
  P.trace = trace ? 1 : 0;
  P.part = ctx->ws.get<unsigned long long>("fit_part", kPartWords);
  RPD_CK(cudaMemsetAsync(P.part, 0, sizeof(unsigned long long) * kPartWords, ctx->stream));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kFitCtas);
  cfg.blockDim = dim3(kFitThreads);
  cfg.dynamicSmemBytes = fit_dyn_smem(rows_cap);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RPD_CK(cudaLaunchKernelEx(&cfg, k_fit, P));
}

// --------------------------------------------------- transform_disparity --
__global__ void k_transform(const float* __restrict__ d1, int h, int w,
                            const DevModel* __restrict__ model, double delta,
                            float* __restrict__ d2, unsigned long long* __restrict__ clamped) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned nclamp = 0;
  for (int v = blockIdx.y; v < h; v += gridDim.y) {  // rows strided over gridDim.y
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
    nclamp += __popc(__ballot_sync(0xFFFFFFFFu, clamp));
  }
  if ((threadIdx.x & 31) == 0 && nclamp) atomicAdd(clamped, (unsigned long long)nclamp);
}

void transform_disparity_dev(const float* d1, int h, int w, const DevModel* model, double delta_dt,
                             float* d2, unsigned long long* clamped, cudaStream_t st) {
  k_transform<<<dim3(cdiv(w, 128), std::max(1, cdiv(h, 4))), 128, 0, st>>>(d1, h, w, model,
                                                                           delta_dt, d2, clamped);
  RPD_LAUNCH_CHECK();
}

}  // namespace rpdg

// ------------------------------------------------------------ debug hook --
namespace rpdg {
__global__ void k_sincos_probe(const double* __restrict__ x, int n, double* __restrict__ s,
                               double* __restrict__ c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dd_sincos(x[i], &s[i], &c[i]);
}
void sincos_probe_dev(const double* x, int n, double* s, double* c, cudaStream_t st) {
  k_sincos_probe<<<cdiv(n, 128), 128, 0, st>>>(x, n, s, c);
  RPD_LAUNCH_CHECK();
}
}  // namespace rpdg
