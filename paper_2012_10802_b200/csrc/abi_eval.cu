// abi_eval.cu — evaluation metrics (evaluation.hpp:14-149 of the reference;
// SURVEY.md §8(f) row 1) on the device: the per-pixel passes run as CUDA
// kernels with deterministic block partials; the tiny summaries (counts, the
// instance intersection table) are finished on the host with the reference's
// own arithmetic.
//
// * pep / rmse: one pass counts the pixels valid in both maps and those with
//   |est - gt| > eps, and sums the squared errors in double-double (block
//   partials combined in a fixed order), so the rmse is the correctly rounded
//   square root of a sum accurate to ~1e-30 relative (the reference's
//   sequential double sum differs by up to ~n ulp).
// * pixel_metrics: exact integer confusion counts.
// * instance_metrics: label maxima, areas and the dense prediction x truth
//   intersection table by (warp-aggregated) integer atomics; the greedy IoU
//   matching runs on the host exactly as evaluation.hpp:124-147.
#include <algorithm>
#include <climits>
#include <cmath>
#include <vector>

#include "abi_util.hpp"

using namespace rpdg;

namespace {

constexpr int kEvalBlocks = 592;  // 4 x 148 SMs, grid-stride
constexpr int kEvalThreads = 256;

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

struct DispPartial {
  unsigned long long q, bad;
  double hi, lo;
};

__global__ void __launch_bounds__(kEvalThreads)
    k_eval_disp(const float* __restrict__ est, const float* __restrict__ gt, long long n,
                double eps, DispPartial* __restrict__ part) {
  unsigned long long q = 0, bad = 0;
  DDs sum{0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float a = est[i], b = gt[i];
    if (a == kInvalid || b == kInvalid) continue;
    ++q;
    const double e = double(a) - double(b);
    if (fabs(e) > eps) ++bad;
    const double p = e * e;
    sum = dd_plus(sum, DDs{p, __fma_rn(e, e, -p)});  // exact square
  }
  // fixed-order block reduction
  __shared__ DispPartial s[kEvalThreads];
  s[threadIdx.x] = DispPartial{q, bad, sum.hi, sum.lo};
  __syncthreads();
  for (int width = kEvalThreads / 2; width > 0; width >>= 1) {
    if (threadIdx.x < width) {
      DispPartial& x = s[threadIdx.x];
      const DispPartial y = s[threadIdx.x + width];
      x.q += y.q;
      x.bad += y.bad;
      const DDs r = dd_plus(DDs{x.hi, x.lo}, DDs{y.hi, y.lo});
      x.hi = r.hi;
      x.lo = r.lo;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

struct ConfPartial {
  unsigned long long tp, fp, fn;
};

__global__ void __launch_bounds__(kEvalThreads)
    k_confusion(const int32_t* __restrict__ pred, const int32_t* __restrict__ gtm, long long n,
                ConfPartial* __restrict__ part) {
  unsigned long long tp = 0, fp = 0, fn = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const bool p = pred[i] != 0, g = gtm[i] != 0;
    tp += p && g;
    fp += p && !g;
    fn += !p && g;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    tp += __shfl_xor_sync(0xFFFFFFFFu, tp, off);
    fp += __shfl_xor_sync(0xFFFFFFFFu, fp, off);
    fn += __shfl_xor_sync(0xFFFFFFFFu, fn, off);
  }
  __shared__ ConfPartial s[kEvalThreads / 32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = ConfPartial{tp, fp, fn};
  __syncthreads();
  if (threadIdx.x == 0) {
    ConfPartial c{0, 0, 0};
    for (int w = 0; w < kEvalThreads / 32; ++w) {
      c.tp += s[w].tp;
      c.fp += s[w].fp;
      c.fn += s[w].fn;
    }
    part[blockIdx.x] = c;
  }
}

__global__ void __launch_bounds__(kEvalThreads)
    k_label_max(const int32_t* __restrict__ a, const int32_t* __restrict__ b, long long n,
                int* __restrict__ mx) {
  int ma = INT_MIN, mb = INT_MIN;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    ma = max(ma, a[i]);
    mb = max(mb, b[i]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    ma = max(ma, __shfl_xor_sync(0xFFFFFFFFu, ma, off));
    mb = max(mb, __shfl_xor_sync(0xFFFFFFFFu, mb, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&mx[0], ma);
    atomicMax(&mx[1], mb);
  }
}

// Areas of every positive label and the dense intersection table
// inter[p * (ng + 1) + g] (evaluation.hpp:106-113).
__global__ void __launch_bounds__(kEvalThreads)
    k_instance_counts(const int32_t* __restrict__ pred, const int32_t* __restrict__ gti,
                      long long n, int ng, unsigned long long* __restrict__ area_p,
                      unsigned long long* __restrict__ area_g,
                      unsigned long long* __restrict__ inter) {
  for (long long i0 = blockIdx.x * (long long)blockDim.x; i0 < n;
       i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    int p = 0, g = 0;
    if (i < n) {
      p = pred[i];
      g = gti[i];
    }
    // neighbouring pixels mostly share labels: one atomic per distinct key per warp
    const int kp = p > 0 ? p : -1, kg = g > 0 ? g : -1;
    const long long ki = (p > 0 && g > 0) ? (long long)p * (ng + 1) + g : -1;
    unsigned peers = __match_any_sync(0xFFFFFFFFu, kp);
    if (kp > 0 && (threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&area_p[kp], (unsigned long long)__popc(peers));
    peers = __match_any_sync(0xFFFFFFFFu, kg);
    if (kg > 0 && (threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&area_g[kg], (unsigned long long)__popc(peers));
    peers = __match_any_sync(0xFFFFFFFFu, ki);
    if (ki >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&inter[ki], (unsigned long long)__popc(peers));
  }
}

void check_shape(int h, int w) { check_dims(h, w); }

DispPartial disp_pass(rpd_ctx* ctx, const float* est, const float* gt, int h, int w, double eps) {
  check_shape(h, w);
  const long long n = (long long)h * w;
  const float* de = upload(ctx, "ev_est", est, size_t(n));
  const float* dg = upload(ctx, "ev_gt", gt, size_t(n));
  DispPartial* part = ctx->ws.get<DispPartial>("ev_part", kEvalBlocks);
  k_eval_disp<<<kEvalBlocks, kEvalThreads, 0, ctx->stream>>>(de, dg, n, eps, part);
  RPD_LAUNCH_CHECK();
  std::vector<DispPartial> hp(kEvalBlocks);
  download(ctx, hp.data(), part, sizeof(DispPartial) * kEvalBlocks);
  // fixed-order combination of the block partials (same double-double sum)
  DispPartial t{0, 0, 0.0, 0.0};
  auto two_sum = [](double a, double b, double& s, double& e) {
    s = a + b;
    const double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
  };
  for (const DispPartial& b : hp) {  // the device's dd_plus, block order
    t.q += b.q;
    t.bad += b.bad;
    double sh, sl, th, tl;
    two_sum(t.hi, b.hi, sh, sl);
    two_sum(t.lo, b.lo, th, tl);
    sl += th;
    const double hi = sh + sl;
    double lo = sl - (hi - sh);
    lo += tl;
    t.hi = hi + lo;
    t.lo = lo - (t.hi - hi);
  }
  return t;
}

}  // namespace

extern "C" {

rpd_status rpd_pep(rpd_ctx* ctx, const float* est, const float* gt, int h, int w, double eps,
                   double* out) {
  return guard(ctx, [&] {
    if (!est || !gt || !out) throw InvalidArg("pep: null buffer");
    const DispPartial t = disp_pass(ctx, est, gt, h, w, eps);
    if (t.q == 0) throw Degenerate("pep: no overlapping valid pixels");
    *out = 100.0 * static_cast<double>(t.bad) / static_cast<double>(t.q);
  });
}

rpd_status rpd_rmse(rpd_ctx* ctx, const float* est, const float* gt, int h, int w, double* out) {
  return guard(ctx, [&] {
    if (!est || !gt || !out) throw InvalidArg("rmse: null buffer");
    const DispPartial t = disp_pass(ctx, est, gt, h, w, 0.0);
    if (t.q == 0) throw Degenerate("rmse: no overlapping valid pixels");
    *out = std::sqrt(t.hi / static_cast<double>(t.q));
  });
}

double rpd_fscore(double precision, double recall) {
  const double s = precision + recall;
  return s > 0 ? 2.0 * precision * recall / s : 0.0;
}

rpd_status rpd_pixel_metrics(rpd_ctx* ctx, const int32_t* pred, const int32_t* gt_mask, int h,
                             int w, rpd_pixel_report* out) {
  return guard(ctx, [&] {
    if (!pred || !gt_mask || !out) throw InvalidArg("pixel_metrics: null buffer");
    check_shape(h, w);
    const long long n = (long long)h * w;
    const int32_t* dp = upload(ctx, "ev_pred", pred, size_t(n));
    const int32_t* dg = upload(ctx, "ev_gtm", gt_mask, size_t(n));
    ConfPartial* part = ctx->ws.get<ConfPartial>("ev_conf", kEvalBlocks);
    k_confusion<<<kEvalBlocks, kEvalThreads, 0, ctx->stream>>>(dp, dg, n, part);
    RPD_LAUNCH_CHECK();
    std::vector<ConfPartial> hp(kEvalBlocks);
    download(ctx, hp.data(), part, sizeof(ConfPartial) * kEvalBlocks);
    long long tp = 0, fp = 0, fn = 0;
    for (const ConfPartial& b : hp) {
      tp += (long long)b.tp;
      fp += (long long)b.fp;
      fn += (long long)b.fn;
    }
    rpd_pixel_report m{};
    m.counts = rpd_confusion{tp, fp, fn, n - tp - fp - fn};
    // evaluation.hpp:82-88
    const rpd_confusion& c = m.counts;
    const long long total = c.n_tp + c.n_fp + c.n_fn + c.n_tn;
    m.degenerate_precision = c.n_tp + c.n_fp == 0;
    m.degenerate_recall = c.n_tp + c.n_fn == 0;
    m.precision =
        m.degenerate_precision ? 0.0 : static_cast<double>(c.n_tp) / double(c.n_tp + c.n_fp);
    m.recall = m.degenerate_recall ? 0.0 : static_cast<double>(c.n_tp) / double(c.n_tp + c.n_fn);
    m.accuracy = total > 0 ? static_cast<double>(c.n_tp + c.n_tn) / double(total) : 0.0;
    m.fscore = rpd_fscore(m.precision, m.recall);
    *out = m;
  });
}

rpd_status rpd_instance_metrics(rpd_ctx* ctx, const int32_t* pred, const int32_t* gt_instances,
                                int h, int w, double iou_min, rpd_instance_report* out) {
  return guard(ctx, [&] {
    if (!pred || !gt_instances || !out) throw InvalidArg("instance_metrics: null buffer");
    check_shape(h, w);
    const long long n = (long long)h * w;
    const int32_t* dp = upload(ctx, "ev_pred", pred, size_t(n));
    const int32_t* dg = upload(ctx, "ev_gti", gt_instances, size_t(n));
    int* mx = ctx->ws.get<int>("ev_max", 2);
    const int init[2] = {INT_MIN, INT_MIN};
    RPD_CK(cudaMemcpyAsync(mx, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    k_label_max<<<kEvalBlocks, kEvalThreads, 0, ctx->stream>>>(dp, dg, n, mx);
    RPD_LAUNCH_CHECK();
    int hm[2];
    download(ctx, hm, mx, sizeof(hm));
    const int np = std::max(hm[0], 0), ng = std::max(hm[1], 0);
    const long long cells = (long long)(np + 1) * (ng + 1);
    if (cells > (1ll << 26))
      throw Capacity("instance_metrics: (max pred + 1) * (max truth + 1) exceeds 2^26");
    unsigned long long* area_p = ctx->ws.get<unsigned long long>("ev_area_p", size_t(np) + 1);
    unsigned long long* area_g = ctx->ws.get<unsigned long long>("ev_area_g", size_t(ng) + 1);
    unsigned long long* inter = ctx->ws.get<unsigned long long>("ev_inter", size_t(cells));
    RPD_CK(cudaMemsetAsync(area_p, 0, sizeof(unsigned long long) * (np + 1), ctx->stream));
    RPD_CK(cudaMemsetAsync(area_g, 0, sizeof(unsigned long long) * (ng + 1), ctx->stream));
    RPD_CK(cudaMemsetAsync(inter, 0, sizeof(unsigned long long) * cells, ctx->stream));
    k_instance_counts<<<kEvalBlocks, kEvalThreads, 0, ctx->stream>>>(dp, dg, n, ng, area_p,
                                                                     area_g, inter);
    RPD_LAUNCH_CHECK();
    std::vector<unsigned long long> ap(static_cast<size_t>(np) + 1), ag(static_cast<size_t>(ng) + 1),
        it(static_cast<size_t>(cells));
    RPD_CK(cudaMemcpyAsync(ap.data(), area_p, sizeof(unsigned long long) * ap.size(),
                           cudaMemcpyDeviceToHost, ctx->stream));
    RPD_CK(cudaMemcpyAsync(ag.data(), area_g, sizeof(unsigned long long) * ag.size(),
                           cudaMemcpyDeviceToHost, ctx->stream));
    download(ctx, it.data(), inter, sizeof(unsigned long long) * it.size());
    // evaluation.hpp:115-147
    struct Pair {
      double iou;
      int p, g;
    };
    std::vector<Pair> pairs;
    for (int p = 1; p <= np; ++p)
      for (int g = 1; g <= ng; ++g) {
        const long long i = (long long)it[size_t(p) * (ng + 1) + g];
        if (i == 0) continue;
        const double iou = static_cast<double>(i) /
                           static_cast<double>((long long)ap[size_t(p)] + (long long)ag[size_t(g)] - i);
        pairs.push_back({iou, p, g});
      }
    std::sort(pairs.begin(), pairs.end(), [](const Pair& a, const Pair& b) {
      if (a.iou != b.iou) return a.iou > b.iou;
      if (a.p != b.p) return a.p < b.p;
      return a.g < b.g;
    });
    std::vector<char> used_p(size_t(np) + 1, 0), used_g(size_t(ng) + 1, 0);
    rpd_instance_report rep{0, 0, 0};
    for (const Pair& pr : pairs) {
      if (pr.iou < iou_min) break;
      if (used_p[size_t(pr.p)] || used_g[size_t(pr.g)]) continue;
      used_p[size_t(pr.p)] = 1;
      used_g[size_t(pr.g)] = 1;
      ++rep.correct;
    }
    for (int p = 1; p <= np; ++p)
      if (!used_p[size_t(p)]) ++rep.incorrect;
    for (int g = 1; g <= ng; ++g)
      if (!used_g[size_t(g)]) ++rep.misdetection;
    *out = rep;
  });
}

}  // extern "C"
