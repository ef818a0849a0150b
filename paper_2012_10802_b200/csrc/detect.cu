// detect.cu — 2-D histogram, adaptive road threshold, connected components and
// pothole labelling for sm_100a.
//
// Reference: /root/reference/proj/src/segmentation.cpp:251-434.
//
//  * build_histogram (:251-296): vectors (D2(p), sum8/8) with the neighbour
//    sum in row-major order in double; lo/hi by atomic min/max on ordered
//    bit patterns; the pipeline stores only the diagonal band |i-j| <= band
//    (band = ceil(tau/bw)+1), everything outside is provably excluded by the
//    |g1-g2| > tau test of find_road_threshold and is only counted.
//  * find_road_threshold (:298-359): single CTA.  Keys (g1+g2)/2 are grouped
//    by i+j (groups are separated by bw/2, far above rounding), each group's
//    exact-double keys are sorted and merged, prefix sums run sequentially in
//    the reference's order, the 2-means split is an argmin with first-index
//    tie break.
//  * connected_components (:361-390) / detect_potholes (:392-434): union-find
//    rooted at the minimum raster index; labels are ranks of roots, i.e.
//    first-encounter scan order.  Distinct superpixels per component are
//    counted with an open-addressing hash set of (root, superpixel) pairs.

#include <cfloat>
#include <cmath>

#include <cub/cub.cuh>

#include "ccl.cuh"
#include "scan.cuh"

namespace rpdg {

namespace {

__device__ __forceinline__ long long ordered(double x) {
  const long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFll);
}
__device__ __forceinline__ double unordered(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7FFFFFFFFFFFFFFFll));
}

// One histogram vector at interior pixel (u, v): returns false when any of the
// nine samples is invalid (segmentation.cpp:257-271).
__device__ __forceinline__ bool hist_vector(const float* __restrict__ d2, int w, int u, int v,
                                            double& x, double& y) {
  const float c = d2[size_t(v) * w + u];
  if (c == kInvalid) return false;
  double sum = 0.0;
  for (int dv = -1; dv <= 1; ++dv)
    for (int du = -1; du <= 1; ++du) {
      if (du == 0 && dv == 0) continue;
      const float q = d2[size_t(v + dv) * w + (u + du)];
      if (q == kInvalid) return false;
      sum += q;
    }
  x = double(c);
  y = sum / 8.0;
  return true;
}

// meta: [0] n, [1] total, [2] excluded outside band, [3] lo key, [4] hi key
__global__ void k_hist_range(const float* __restrict__ d2, int h, int w,
                             long long* __restrict__ meta) {
  // rows strided over gridDim.y: one atomic triple per block (the three
  // counters are single hot addresses)
  const int u = blockIdx.x * blockDim.x + threadIdx.x + 1;
  long long lo = 0x7FFFFFFFFFFFFFFFll, hi = (long long)0x8000000000000000ull;
  unsigned long long cnt = 0;
  for (int v = blockIdx.y + 1; v + 1 < h; v += gridDim.y) {
    double x = 0, y = 0;
    const bool ok = u + 1 < w && hist_vector(d2, w, u, v, x, y);
    if (ok) {
      lo = min(lo, min(ordered(x), ordered(y)));
      hi = max(hi, max(ordered(x), ordered(y)));
      ++cnt;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, off));
    hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, off));
    cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, off);
  }
  __shared__ long long s_lo[32], s_hi[32];
  __shared__ unsigned long long s_cnt[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
    s_cnt[warp] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c = 0;
    for (int q = 0; q < int(blockDim.x >> 5); ++q) {
      lo = min(lo, s_lo[q]);
      hi = max(hi, s_hi[q]);
      c += s_cnt[q];
    }
    if (c) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&meta[1]), c);
      atomicMin(&meta[3], lo);
      atomicMax(&meta[4], hi);
    }
  }
}

__global__ void k_hist_setup(long long* __restrict__ meta, double bw, double* __restrict__ origin,
                             long long cap_rows, DevStatus* st, int where) {
  if (meta[1] == 0) {
    meta[0] = 0;
    *origin = 0.0;
    return;
  }
  const double lo = unordered(meta[3]), hi = unordered(meta[4]);
  const double o = floor(lo / bw) * bw;
  *origin = o;
  const long long n = (long long)floor((hi - o) / bw) + 1;
  meta[0] = n;
  if (n > cap_rows || n < 1) {
    set_status(st, RPD_ENOMEM, where, n);
    meta[0] = 0;
  }
}

__global__ void k_hist_clear(long long* __restrict__ band, const long long* __restrict__ meta,
                             int stride) {
  const long long total = meta[0] * stride;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    band[i] = 0;
}

// inv_bw != 0: bw is a power of two and (x - o) / bw == (x - o) * inv_bw
// exactly (both are the correctly rounded value of the same real number).
__global__ void k_hist_bin(const float* __restrict__ d2, int h, int w, double bw, double inv_bw,
                           const double* __restrict__ origin, long long* __restrict__ meta,
                           long long* __restrict__ band, int half) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const long long n = meta[0];
  const double o = *origin;
  unsigned outside_cnt = 0;
  for (int v = blockIdx.y + 1; v + 1 < h; v += gridDim.y) {
    double x = 0, y = 0;
    const bool ok = n > 0 && u + 1 < w && hist_vector(d2, w, u, v, x, y);
    long long slot = -1;
    if (ok) {
      const double qx = inv_bw != 0.0 ? (x - o) * inv_bw : (x - o) / bw;
      const double qy = inv_bw != 0.0 ? (y - o) * inv_bw : (y - o) / bw;
      long long i = (long long)floor(qx), j = (long long)floor(qy);
      i = i < n - 1 ? i : n - 1;
      j = j < n - 1 ? j : n - 1;
      const long long dj = j - i;
      if (dj < -half || dj > half)
        ++outside_cnt;
      else
        slot = i * (2 * half + 1) + (dj + half);
    }
    // neighbouring pixels mostly share a bin: one atomic per distinct bin per warp
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, slot);
    if (slot >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(reinterpret_cast<unsigned long long*>(&band[slot]),
                (unsigned long long)__popc(peers));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) outside_cnt += __shfl_xor_sync(0xFFFFFFFFu, outside_cnt, off);
  if ((threadIdx.x & 31) == 0 && outside_cnt)
    atomicAdd(reinterpret_cast<unsigned long long*>(&meta[2]), (unsigned long long)outside_cnt);
}

// Full n x n histogram -> band storage (ABI path), band = n - 1.
__global__ void k_full_to_band(const long long* __restrict__ full, long long n,
                               long long* __restrict__ band) {
  const long long stride = 2 * n - 1;
  const long long total = n * n;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long i = q / n, j = q % n;
    band[i * stride + (j - i + n - 1)] = full[q];
  }
}

__global__ void k_band_to_full(const long long* __restrict__ band, const long long* __restrict__ meta,
                               int half, long long* __restrict__ full) {
  const long long n = meta[0];
  const long long total = n * n;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long i = q / n, j = q % n;
    const long long dj = j - i;
    full[q] = (dj < -half || dj > half) ? 0 : band[i * (2 * half + 1) + dj + half];
  }
}

// --------------------------------------------------- find_road_threshold --
constexpr int kThrThreads = 1024;
constexpr int kMaxGroup = 64;  // distinct keys per i+j group kept in registers

struct ThrArgs {
  const long long* band;
  const long long* meta;  // n, total, excluded_outside
  const double* origin;
  int half;
  double bw, tau, delta_pd;
  double* xs;      // scratch keys (capacity cap_keys)
  long long* ws;   // scratch weights
  int* gcount;     // per group distinct count (capacity 2n)
  long long cap_keys;
  double* pw;      // prefix scratch (cap_keys + 1 each)
  double* pwx;
  double* pwxx;
  rpd_threshold* out;
  DevStatus* status;
  int where;
};

// Collect one group's in-tau keys (sorted, merged) into local arrays.
__device__ int thr_group(const ThrArgs& a, long long n, double o, long long s, double* kx,
                         long long* kw, long long& excl) {
  int m = 0;
  long long ilo = s - (n - 1) > 0 ? s - (n - 1) : 0;
  long long ihi = s < n - 1 ? s : n - 1;
  // only |j - i| = |s - 2i| <= half is stored
  const long long blo = (s - a.half + 1) >> 1, bhi = (s + a.half) >> 1;
  ilo = ilo > blo ? ilo : blo;
  ihi = ihi < bhi ? ihi : bhi;
  for (long long i = ilo; i <= ihi; ++i) {
    const long long j = s - i;
    const long long dj = j - i;
    if (dj < -a.half || dj > a.half) continue;
    const long long c = a.band[i * (2 * a.half + 1) + dj + a.half];
    if (c == 0) continue;
    const double g1 = o + (double(i) + 0.5) * a.bw;
    const double g2 = o + (double(j) + 0.5) * a.bw;
    if (fabs(g1 - g2) > a.tau) {
      excl += c;
      continue;
    }
    const double key = (g1 + g2) / 2.0;
    int pos = 0;
    while (pos < m && kx[pos] < key) ++pos;
    if (pos < m && kx[pos] == key) {
      kw[pos] += c;
      continue;
    }
    if (m == kMaxGroup) continue;  // cannot happen for band <= 31
    for (int q = m; q > pos; --q) {
      kx[q] = kx[q - 1];
      kw[q] = kw[q - 1];
    }
    kx[pos] = key;
    kw[pos] = c;
    ++m;
  }
  return m;
}

__global__ void __launch_bounds__(kThrThreads) k_threshold(const __grid_constant__ ThrArgs a) {
  using Scan = cub::BlockScan<long long, kThrThreads>;
  using Red = cub::BlockReduce<long long, kThrThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ typename Red::TempStorage red_tmp;
  __shared__ long long s_base, s_excl, s_m;
  if (a.status->code != 0) {
    if (threadIdx.x == 0) *a.out = rpd_threshold{0, 0, 0, 0, 0, 0};
    return;
  }
  const long long n = a.meta[0];
  const double o = *a.origin;
  const long long groups = n > 0 ? 2 * n - 1 : 0;
  if (threadIdx.x == 0) {
    s_base = 0;
    s_excl = 0;
  }
  __syncthreads();
  // pass 1: distinct counts per group
  long long excl_local = 0;
  for (long long g0 = 0; g0 < groups; g0 += blockDim.x) {
    const long long s = g0 + threadIdx.x;
    long long cnt = 0;
    if (s < groups) {
      double kx[kMaxGroup];
      long long kw[kMaxGroup];
      cnt = thr_group(a, n, o, s, kx, kw, excl_local);
      a.gcount[s] = int(cnt);
    }
    long long off, tot;
    Scan(scan_tmp).ExclusiveSum(cnt, off, tot);
    if (s < groups && cnt > 0) {
      // pass 2 inline: write this group's keys at base + off
      double kx[kMaxGroup];
      long long kw[kMaxGroup];
      long long dummy = 0;
      const int m = thr_group(a, n, o, s, kx, kw, dummy);
      const long long base = s_base + off;
      for (int q = 0; q < m && base + q < a.cap_keys; ++q) {
        a.xs[base + q] = kx[q];
        a.ws[base + q] = kw[q];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += tot;
    __syncthreads();
  }
  const long long excl_in = Red(red_tmp).Sum(excl_local);
  if (threadIdx.x == 0) {
    s_excl = excl_in + a.meta[2];
    s_m = s_base;
  }
  __syncthreads();
  const long long m = s_m;
  if (m == 0) {
    if (threadIdx.x == 0) {
      set_status(a.status, RPD_EDEGENERATE, a.where);
      *a.out = rpd_threshold{0, 0, 0, 0, 0, 0};
    }
    return;
  }
  if (m > a.cap_keys) {
    if (threadIdx.x == 0) set_status(a.status, RPD_ENOMEM, kWhereHistTooLarge, m);
    return;
  }
  const long long total = a.meta[1];
  rpd_threshold res{};
  res.excluded_fraction = total > 0 ? double(s_excl) / double(total) : 0.0;
  if (m < 2) {
    if (threadIdx.x == 0) {
      res.degenerate = 1;
      res.mu1 = res.mu2 = res.t_r = a.xs[0];
      res.t_s = res.t_r - a.delta_pd;
      *a.out = res;
    }
    return;
  }
  // prefix sums in the reference's sequential order
  if (threadIdx.x == 0) {
    double pw = 0, pwx = 0, pwxx = 0;
    a.pw[0] = a.pwx[0] = a.pwxx[0] = 0.0;
    for (long long i = 0; i < m; ++i) {
      const double wi = double(a.ws[i]);
      const double xi = a.xs[i];
      pw = pw + wi;
      pwx = pwx + wi * xi;
      pwxx = pwxx + wi * xi * xi;
      a.pw[i + 1] = pw;
      a.pwx[i + 1] = pwx;
      a.pwxx[i + 1] = pwxx;
    }
  }
  __syncthreads();
  // split scan: lexicographic min of (sse, split)
  double best_e = __longlong_as_double(0x7FF0000000000000ll);
  long long best_s = 1;
  for (long long sp = 1 + threadIdx.x; sp < m; sp += blockDim.x) {
    const double n1 = a.pw[sp] - a.pw[0], s1 = a.pwx[sp] - a.pwx[0], q1 = a.pwxx[sp] - a.pwxx[0];
    const double n2 = a.pw[m] - a.pw[sp], s2 = a.pwx[m] - a.pwx[sp], q2 = a.pwxx[m] - a.pwxx[sp];
    const double e = (q1 - s1 * s1 / n1) + (q2 - s2 * s2 / n2);
    if (e < best_e) {
      best_e = e;
      best_s = sp;
    }
  }
  // block argmin with first-index tie break
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double oe = __shfl_xor_sync(0xFFFFFFFFu, best_e, off);
    const long long os = __shfl_xor_sync(0xFFFFFFFFu, best_s, off);
    if (oe < best_e || (oe == best_e && os < best_s)) {
      best_e = oe;
      best_s = os;
    }
  }
  __shared__ double w_e[32];
  __shared__ long long w_s[32];
  if (lane == 0) {
    w_e[threadIdx.x >> 5] = best_e;
    w_s[threadIdx.x >> 5] = best_s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double be = w_e[0];
    long long bs = w_s[0];
    for (int q = 1; q < int(blockDim.x >> 5); ++q)
      if (w_e[q] < be || (w_e[q] == be && w_s[q] < bs)) {
        be = w_e[q];
        bs = w_s[q];
      }
    // no split evaluated as finite keeps split 1 (reference initialisation)
    const long long sp = (be < __longlong_as_double(0x7FF0000000000000ll)) ? bs : 1;
    res.mu1 = (a.pwx[sp] - a.pwx[0]) / (a.pw[sp] - a.pw[0]);
    res.mu2 = (a.pwx[m] - a.pwx[sp]) / (a.pw[m] - a.pw[sp]);
    res.t_r = res.mu2;
    res.t_s = res.t_r - a.delta_pd;
    *a.out = res;
  }
}

// ------------------------------------------------------------ labelling ----
// Elementwise passes take four pixels per thread (one 16-byte access per
// array; workspace buffers are 256-byte aligned), launched with ew4_blocks(n).
// Root flag of pixel p (a kept component's representative): parent[p] == p.
struct RootFlagIn {
  const int* parent;
  const unsigned char* keep;  // nullptr: every component
  __device__ __forceinline__ void load8(long long base, long long n, int (&f)[8]) const {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long p = base + k;
      f[k] = p < n && parent[p] == p && (!keep || keep[p]) ? 1 : 0;
    }
  }
};

__global__ void k_root_relabel(const int* __restrict__ parent,
                               const unsigned char* __restrict__ keep,
                               const int* __restrict__ rank, long long n, int32_t* __restrict__ out) {
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  auto lab = [&](int r) { return (r >= 0 && (!keep || keep[r])) ? rank[r] + 1 : 0; };
  if (p0 + 3 < n && (reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
    const int4 r = *reinterpret_cast<const int4*>(parent + p0);
    *reinterpret_cast<int4*>(out + p0) = make_int4(lab(r.x), lab(r.y), lab(r.z), lab(r.w));
    return;
  }
  for (long long p = p0; p < min(n, p0 + 4); ++p) out[p] = lab(parent[p]);
}


__global__ void k_detect_mask(const float* __restrict__ d3, long long n,
                              const rpd_threshold* __restrict__ thr, int32_t* __restrict__ mask) {
  const double ts = thr->t_s;
  auto in = [&](float x) { return (x != kInvalid && double(x) < ts) ? 1 : 0; };
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 + 3 < n && (reinterpret_cast<uintptr_t>(d3) & 15u) == 0) {
    const float4 x = *reinterpret_cast<const float4*>(d3 + p0);
    *reinterpret_cast<int4*>(mask + p0) = make_int4(in(x.x), in(x.y), in(x.z), in(x.w));
    return;
  }
  for (long long p = p0; p < min(n, p0 + 4); ++p) mask[p] = in(d3[p]);
}

constexpr unsigned long long kEmpty = 0xFFFFFFFFFFFFFFFFull;

__global__ void k_detect_stats(const int* __restrict__ parent, const int32_t* __restrict__ sp,
                               int h, int w, int margin, int* __restrict__ area,
                               unsigned char* __restrict__ border,
                               unsigned long long* __restrict__ table, unsigned long long tmask,
                               int* __restrict__ nsp) {
  const long long n = (long long)h * w;
  for (long long p0 = (long long)blockIdx.x * blockDim.x; p0 < n;
       p0 += (long long)gridDim.x * blockDim.x) {
    const long long p = p0 + threadIdx.x;
    const int r = p < n ? parent[p] : -1;
    if (!__any_sync(0xFFFFFFFFu, r >= 0)) continue;  // all background (most of the mask)
    const RunInfo ri = run_info(r);
    if (ri.head) atomicAdd(&area[r], ri.end - int(threadIdx.x & 31) + 1);  // run length
    if (r >= 0) {
      const int u = int(p % w), v = int(p / w);
      if (u < margin || u >= w - margin || v < margin || v >= h - margin) border[r] = 1;
    }
    // (root, superpixel) pairs: run heads of equal pairs insert into the set
    const int s = p < n ? sp[p] : 0;
    const int prs = __shfl_up_sync(0xFFFFFFFFu, s, 1);
    const int prr = __shfl_up_sync(0xFFFFFFFFu, r, 1);
    const bool head = r >= 0 && ((threadIdx.x & 31) == 0 || prr != r || prs != s);
    if (head) {
      const unsigned long long key = ((unsigned long long)(unsigned)r << 32) | (unsigned)s;
      unsigned long long hsh = key * 0x9E3779B97F4A7C15ull;
      unsigned long long slot = (hsh >> 20) & tmask;
      while (true) {
        const unsigned long long old = atomicCAS(&table[slot], kEmpty, key);
        if (old == kEmpty) {
          atomicAdd(&nsp[r], 1);
          break;
        }
        if (old == key) break;
        slot = (slot + 1) & tmask;
      }
    }
  }
}

__global__ void k_detect_keep(const int* __restrict__ parent, const int* __restrict__ area,
                              const unsigned char* __restrict__ border, const int* __restrict__ nsp,
                              long long n, long long min_area, int min_sp,
                              unsigned char* __restrict__ keep) {
  // four pixels per thread (launched with max(1, cdiv(n, 1024)) blocks of 256)
  auto root = [&](long long p) {
    keep[p] = (!border[p] && (long long)area[p] >= min_area && nsp[p] >= min_sp) ? 1 : 0;
  };
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 + 3 < n) {
    const int4 r = *reinterpret_cast<const int4*>(parent + p0);
    if (r.x == p0) root(p0);
    if (r.y == p0 + 1) root(p0 + 1);
    if (r.z == p0 + 2) root(p0 + 2);
    if (r.w == p0 + 3) root(p0 + 3);
    return;
  }
  for (long long p = p0; p < n; ++p)
    if (parent[p] == p) root(p);
}

}  // namespace


namespace {
__global__ void k_hist_init(long long* meta) {
  meta[0] = 0;
  meta[1] = 0;
  meta[2] = 0;
  meta[3] = 0x7FFFFFFFFFFFFFFFll;
  meta[4] = (long long)0x8000000000000000ull;
}
}  // namespace

constexpr long long kHistCapRows = 1 << 16;

static HistDev hist_alloc(rpd_ctx* ctx, int half, long long cap_rows, const char* tag,
                          bool with_bins = true) {
  HistDev hd;
  hd.half = half;
  hd.cap_rows = cap_rows;
  hd.meta = ctx->ws.get<long long>(std::string("hist_meta_") + tag, 5);
  hd.origin = ctx->ws.get<double>(std::string("hist_origin_") + tag, 1);
  hd.bins = with_bins ? ctx->ws.get<long long>(std::string("hist_bins_") + tag,
                                               size_t(cap_rows) * size_t(2 * half + 1))
                      : nullptr;
  return hd;
}

static void hist_range(rpd_ctx* ctx, const HistDev& hd, const float* d2, int h, int w, double bw,
                       int where) {
  cudaStream_t st = ctx->stream;
  k_hist_init<<<1, 1, 0, st>>>(hd.meta);
  RPD_LAUNCH_CHECK();
  if (h >= 3 && w >= 3) {
    const int gx = cdiv(w - 2, 128);
    const int gy = std::max(1, std::min(h - 2, cdiv(ctx->sm_count * 8, gx)));
    k_hist_range<<<dim3(gx, gy), 128, 0, st>>>(d2, h, w, hd.meta);
    RPD_LAUNCH_CHECK();
  }
  k_hist_setup<<<1, 1, 0, st>>>(hd.meta, bw, hd.origin, hd.cap_rows, ctx->status, where);
  RPD_LAUNCH_CHECK();
}

static void hist_bin(rpd_ctx* ctx, const HistDev& hd, const float* d2, int h, int w, double bw) {
  cudaStream_t st = ctx->stream;
  const int stride = 2 * hd.half + 1;
  k_hist_clear<<<ctx->sm_count * 4, 256, 0, st>>>(hd.bins, hd.meta, stride);
  RPD_LAUNCH_CHECK();
  if (h >= 3 && w >= 3) {
    // one row per block (the band atomics are spread over bins; the single
    // outside counter is aggregated per warp)
    int ex = 0;
    const double inv = (bw > 0.0 && std::frexp(bw, &ex) == 0.5) ? 1.0 / bw : 0.0;
    // rows strided over gridDim.y (about 4 rows per block)
    const int gy = std::max(1, cdiv(h - 2, 4));
    k_hist_bin<<<dim3(cdiv(w - 2, 128), gy), 128, 0, st>>>(d2, h, w, bw, inv, hd.origin, hd.meta,
                                                           hd.bins, hd.half);
    RPD_LAUNCH_CHECK();
  }
}

HistDev build_histogram_dev(rpd_ctx* ctx, const float* d2, int h, int w, double bw, double tau) {
  if (!(bw > 0)) throw InvalidArg("build_histogram: bin_width must be > 0");
  double hb = std::ceil(tau / bw) + 1.0;
  if (!(hb >= 1.0)) hb = 1.0;
  if (hb > 4096.0) throw InvalidArg("build_histogram: tau / bin_width too large for the band");
  HistDev hd = hist_alloc(ctx, int(hb), kHistCapRows, "pipe");
  hist_range(ctx, hd, d2, h, w, bw, kWhereHistTooLarge);
  hist_bin(ctx, hd, d2, h, w, bw);
  return hd;
}

void build_histogram_full_dev(rpd_ctx* ctx, const float* d2, int h, int w, double bw,
                              long long* n_out, double* origin_out, long long* total_out,
                              long long* counts_host, long long cap_n) {
  if (!(bw > 0)) throw InvalidArg("build_histogram: bin_width must be > 0");
  cudaStream_t st = ctx->stream;
  // range pass first (host needs n to size the full matrix)
  HistDev probe = hist_alloc(ctx, 0, 1LL << 40, "abi_probe", false);
  hist_range(ctx, probe, d2, h, w, bw, kWhereHistTooLarge);
  long long meta[5];
  double origin = 0;
  RPD_CK(cudaMemcpyAsync(meta, probe.meta, sizeof(meta), cudaMemcpyDeviceToHost, st));
  RPD_CK(cudaMemcpyAsync(&origin, probe.origin, sizeof(double), cudaMemcpyDeviceToHost, st));
  RPD_CK(cudaStreamSynchronize(st));
  const long long n = meta[0];
  *n_out = n;
  *origin_out = origin;
  *total_out = meta[1];
  if (n > cap_n) throw Capacity("build_histogram: counts buffer too small");
  if (n == 0 || !counts_host) return;
  if (n > 46341) throw InvalidArg("build_histogram: histogram too large");
  HistDev hd = hist_alloc(ctx, int(n - 1), n, "abi_full");
  hist_range(ctx, hd, d2, h, w, bw, kWhereHistTooLarge);
  hist_bin(ctx, hd, d2, h, w, bw);
  long long* full = ctx->ws.get<long long>("hist_abi_dense", size_t(n) * n);
  k_band_to_full<<<ctx->sm_count * 4, 256, 0, st>>>(hd.bins, hd.meta, hd.half, full);
  RPD_LAUNCH_CHECK();
  RPD_CK(cudaMemcpyAsync(counts_host, full, sizeof(long long) * size_t(n) * n,
                         cudaMemcpyDeviceToHost, st));
  RPD_CK(cudaStreamSynchronize(st));
}

void find_threshold_dev(rpd_ctx* ctx, const HistDev& hd, double bw, double delta_pd, double tau,
                        rpd_threshold* out, int where) {
  const long long cap_keys = std::max<long long>(1024, 2 * hd.cap_rows * 4);
  ThrArgs a{};
  a.band = hd.bins;
  a.meta = hd.meta;
  a.origin = hd.origin;
  a.half = hd.half;
  a.bw = bw;
  a.tau = tau;
  a.delta_pd = delta_pd;
  a.cap_keys = cap_keys;
  a.xs = ctx->ws.get<double>("thr_xs", cap_keys);
  a.ws = ctx->ws.get<long long>("thr_ws", cap_keys);
  a.gcount = ctx->ws.get<int>("thr_gcount", 2 * hd.cap_rows + 1);
  a.pw = ctx->ws.get<double>("thr_pw", cap_keys + 1);
  a.pwx = ctx->ws.get<double>("thr_pwx", cap_keys + 1);
  a.pwxx = ctx->ws.get<double>("thr_pwxx", cap_keys + 1);
  a.out = out;
  a.status = ctx->status;
  a.where = where;
  k_threshold<<<1, kThrThreads, 0, ctx->stream>>>(a);
  RPD_LAUNCH_CHECK();
}

void threshold_from_full_dev(rpd_ctx* ctx, const long long* counts_dev, long long n, double bw,
                             double origin, long long total, double delta_pd, double tau,
                             rpd_threshold* out) {
  cudaStream_t st = ctx->stream;
  HistDev hd = hist_alloc(ctx, int(std::max<long long>(n - 1, 0)), std::max<long long>(n, 1),
                          "abi_thr");
  if (n > 0) {
    k_full_to_band<<<ctx->sm_count * 4, 256, 0, st>>>(counts_dev, n, hd.bins);
    RPD_LAUNCH_CHECK();
  }
  const long long meta[5] = {n, total, 0, 0, 0};
  RPD_CK(cudaMemcpyAsync(hd.meta, meta, sizeof(meta), cudaMemcpyHostToDevice, st));
  RPD_CK(cudaMemcpyAsync(hd.origin, &origin, sizeof(double), cudaMemcpyHostToDevice, st));
  RPD_CK(cudaStreamSynchronize(st));
  find_threshold_dev(ctx, hd, bw, delta_pd, tau, out, kWhereThresholdEmpty);
}

// ------------------------------------------------------------------- CCL ---
void connected_components_dev(rpd_ctx* ctx, const int32_t* mask, int h, int w, int connectivity,
                              int32_t* out) {
  cudaStream_t st = ctx->stream;
  const long long n = (long long)h * w;
  int* parent = ctx->ws.get<int>("ccl_parent", n);
  int* pos = ctx->ws.get<int>("ccl_pos", n);
  uf_label(SameMask{mask}, h, w, connectivity == 4 ? 0 : 1, parent, ctx->sm_count, st);
  scan_exclusive(ctx, RootFlagIn{parent, nullptr}, pos, n);
  k_root_relabel<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(parent, nullptr, pos, n, out);
  RPD_LAUNCH_CHECK();
}

void detect_potholes_dev(rpd_ctx* ctx, const float* d3, const int32_t* sp_labels, double spacing,
                         int h, int w, const rpd_threshold* thr_dev, int border_margin,
                         int min_superpixels, int connectivity, int32_t* out, int* n_out) {
  cudaStream_t st = ctx->stream;
  const long long n = (long long)h * w;
  const int gblocks = int(std::max<long long>(1, std::min<long long>((n + 255) / 256,
                                                                      ctx->sm_count * 16)));
  int32_t* mask = ctx->ws.get<int32_t>("det_mask", n);
  int* parent = ctx->ws.get<int>("det_parent", n);
  int* area = ctx->ws.get<int>("det_area", n);
  unsigned char* border = ctx->ws.get<unsigned char>("det_border", n);
  unsigned char* keep = ctx->ws.get<unsigned char>("det_keep", n);
  int* nsp = ctx->ws.get<int>("det_nsp", n);
  int* pos = ctx->ws.get<int>("det_pos", n);
  unsigned long long tsize = 1024;
  while (tsize < 2ull * (unsigned long long)n) tsize <<= 1;
  unsigned long long* table = ctx->ws.get<unsigned long long>("det_table", tsize);
  k_detect_mask<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(d3, n, thr_dev, mask);
  RPD_LAUNCH_CHECK();
  uf_label(SameMask{mask}, h, w, connectivity == 4 ? 0 : 1, parent, ctx->sm_count, st);
  RPD_CK(cudaMemsetAsync(area, 0, sizeof(int) * n, st));
  RPD_CK(cudaMemsetAsync(border, 0, n, st));
  RPD_CK(cudaMemsetAsync(keep, 0, n, st));
  RPD_CK(cudaMemsetAsync(nsp, 0, sizeof(int) * n, st));
  RPD_CK(cudaMemsetAsync(table, 0xFF, sizeof(unsigned long long) * tsize, st));
  k_detect_stats<<<gblocks, 256, 0, st>>>(parent, sp_labels, h, w, border_margin, area, border,
                                          table, tsize - 1, nsp);
  RPD_LAUNCH_CHECK();
  const long long min_area = (long long)(spacing * spacing);  // segmentation.cpp:418
  k_detect_keep<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(parent, area, border, nsp, n, min_area, min_superpixels,
                                         keep);
  RPD_LAUNCH_CHECK();
  scan_exclusive(ctx, RootFlagIn{parent, keep}, pos, n, n_out);
  k_root_relabel<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(parent, keep, pos, n, out);
  RPD_LAUNCH_CHECK();
}

}  // namespace rpdg
