// ccl.cuh — union-find connected-component labelling and warp run
// reductions shared by SLIC connectivity and pothole labelling.
//
// Components are rooted at their MINIMUM raster index (union links the larger
// root under the smaller), so "first encounter in scan order"
// (segmentation.cpp:104-124, 370-388) is a rank of roots by index.
#pragma once

#include "seg.cuh"

namespace rpdg {

__device__ __forceinline__ int uf_find(const int* parent, int p) {
  int q = parent[p];
  while (q != p) {
    p = q;
    q = parent[p];
  }
  return p;
}

// find with path halving in global memory (benign races: a write only
// re-points a node to one of its ancestors)
__device__ __forceinline__ int uf_find_halve(int* parent, int p) {
  int q = __ldcg(parent + p);
  while (q != p) {
    const int r = __ldcg(parent + q);
    if (r != q) parent[p] = r;
    p = q;
    q = r;
  }
  return p;
}

__device__ __forceinline__ void uf_union(int* parent, int a, int b) {
  while (true) {
    a = uf_find_halve(parent, a);
    b = uf_find_halve(parent, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&parent[a], b);
    if (old == a) return;
    a = old;
  }
}

// Same-class predicate for the CCL kernels.
struct SameLabel {  // SLIC pieces: equal superpixel label (all pixels foreground)
  const int32_t* lab;
  __device__ bool fg(int) const { return true; }
  __device__ bool same(int p, int q) const { return lab[p] == lab[q]; }
  __device__ int key(int p) const { return lab[p]; }  // class of a foreground pixel
};
struct SameMask {  // binary mask components
  const int32_t* mask;
  __device__ bool fg(int p) const { return mask[p] != 0; }
  __device__ bool same(int p, int q) const { return mask[q] != 0; }
  __device__ int key(int) const { return 0; }
};

__global__ void k_uf_flatten(int h, int w, int* parent);

// Block-based union-find: each 32x16 tile is labelled in shared memory
// (local roots = minimum local index = minimum raster index inside the tile),
// then only tile-border pixels union across tiles in global memory.
constexpr int kTileW = 32, kTileH = 16;

// find with path halving: every write re-points a node to one of its own
// ancestors, so concurrent halving by other threads is benign.
__device__ __forceinline__ int uf_find_s(int* lab, int p) {
  int q = lab[p];
  while (q != p) {
    const int r = lab[q];
    if (r != q) lab[p] = r;
    p = q;
    q = r;
  }
  return p;
}

__device__ __forceinline__ void uf_union_s(int* lab, int a, int b) {
  while (true) {
    a = uf_find_s(lab, a);
    b = uf_find_s(lab, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&lab[a], b);
    if (old == a) return;
    a = old;
  }
}

// A warp is one tile row (kTileW == 32): each same-class run of the row is
// linked to its first pixel directly (ballot of run starts), so only the
// links to the row above need unions, and a union is skipped when an earlier
// direction of this pixel or the previous lane joins the same pair of
// current ancestors (the pair's sets are then already linked).
template <typename Pred>
__global__ void __launch_bounds__(kTileW* kTileH)
    k_uf_local(Pred pr, int h, int w, int conn8, int* __restrict__ parent) {
  static_assert(kTileW == 32, "a warp is one tile row");
  __shared__ int lab[kTileW * kTileH];
  __shared__ int cls[kTileW * kTileH];
  const int tx = threadIdx.x % kTileW, ty = threadIdx.x / kTileW;
  const int u0 = blockIdx.x * kTileW, v0 = blockIdx.y * kTileH;
  const int u = u0 + tx, v = v0 + ty;
  const bool in = u < w && v < h;
  const int p = v * w + u;
  const int i = threadIdx.x;
  const bool fg = in && pr.fg(p);
  const int key = fg ? pr.key(p) : 0;
  const int kl = __shfl_up_sync(0xFFFFFFFFu, key, 1);
  const bool fgl = __shfl_up_sync(0xFFFFFFFFu, fg, 1);
  const unsigned starts = __ballot_sync(0xFFFFFFFFu, fg && (tx == 0 || !fgl || kl != key));
  const int head = 31 - __clz(starts & (0xFFFFFFFFu >> (31 - tx)));
  lab[i] = fg ? ty * kTileW + head : -1;
  cls[i] = key;
  if (!__syncthreads_or(fg)) {  // all-background tile (most of a pothole mask)
    if (in) parent[p] = -1;
    return;
  }
  if (ty > 0) {  // warp-uniform
    // directions: N, NW, NE (8-connectivity); the W link is the run
    bool need[3];
    int j[3];
    j[0] = i - kTileW;
    j[1] = i - kTileW - 1;
    j[2] = i - kTileW + 1;
    need[0] = fg && lab[j[0]] >= 0 && cls[j[0]] == key;
    need[1] = fg && conn8 && tx > 0 && lab[j[1]] >= 0 && cls[j[1]] == key;
    need[2] = fg && conn8 && tx + 1 < kTileW && lab[j[2]] >= 0 && cls[j[2]] == key;
    const int ra = fg ? lab[i] : 0;
    unsigned long long pk[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int rb = need[d] ? lab[j[d]] : 0;
      const unsigned lo = unsigned(min(ra, rb)), hi = unsigned(max(ra, rb));
      pk[d] = need[d] ? ((unsigned long long)lo << 32 | hi) : ~0ull - d;
    }
    unsigned long long pv[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) pv[d] = __shfl_up_sync(0xFFFFFFFFu, pk[d], 1);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (!need[d] || (pk[d] >> 32) == (pk[d] & 0xFFFFFFFFull)) continue;
      bool dup = false;
#pragma unroll
      for (int e = 0; e < d; ++e) dup |= pk[e] == pk[d];
      if (tx > 0) {
#pragma unroll
        for (int e = 0; e < 3; ++e) dup |= pv[e] == pk[d];
      }
      if (!dup) uf_union_s(lab, i, j[d]);
    }
  }
  __syncthreads();
  if (in) {
    if (fg) {
      const int r = uf_find_s(lab, i);
      parent[p] = (v0 + r / kTileW) * w + (u0 + r % kTileW);
    } else {
      parent[p] = -1;
    }
  }
}

// Cross-tile unions.  Threads cover only the tile-border pixels: every pixel
// of each tile's top row (part A), then the left / right columns of the other
// rows (part B); each does the unions whose neighbour lies in another tile.
// One warp per tile, tiles in raster order (the order the unions reach the
// shared roots keeps the trees shallow): pass 0 = the tile's top row, pass 1 =
// its left (lanes 0-14) and right (lanes 15-29) columns below the top row.
constexpr int kBorderWarps = 8;
template <typename Pred>
__global__ void __launch_bounds__(32 * kBorderWarps)
    k_uf_border(Pred pr, int h, int w, int conn8, int* parent) {
  const int ncol = (w + kTileW - 1) / kTileW, nrow = (h + kTileH - 1) / kTileH;
  const int tile = blockIdx.x * kBorderWarps + int(threadIdx.x >> 5);
  if (tile >= ncol * nrow) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int u0 = (tile % ncol) * kTileW, v0 = (tile / ncol) * kTileH;
  for (int pass = 0; pass < 2; ++pass) {
    int u, v;
    if (pass == 0) {
      u = u0 + lane;
      v = v0;
    } else {
      u = lane < kTileH - 1 ? u0 : u0 + kTileW - 1;
      v = v0 + 1 + (lane < kTileH - 1 ? lane : lane - (kTileH - 1));
    }
    bool act = u < w && v < h && (pass == 0 || lane < 2 * (kTileH - 1));
    const int tx = u % kTileW;
    const bool left = tx == 0, top = v % kTileH == 0, right = tx == kTileW - 1;
    const int p = v * w + u;
    act = act && pr.fg(p);
    int q[4];
    bool need[4];
    q[0] = p - 1;
    q[1] = p - w;
    q[2] = p - w - 1;
    q[3] = p - w + 1;
    need[0] = act && left && u > 0 && pr.same(p, p - 1);
    need[1] = act && v > 0 && top && pr.same(p, p - w);
    need[2] = act && v > 0 && conn8 && (top || left) && u > 0 && pr.same(p, p - w - 1);
    need[3] = act && v > 0 && conn8 && (top || right) && u + 1 < w && pr.same(p, p - w + 1);
    // A union is skipped when an earlier direction of this pixel or any
    // direction of the previous lane's pixel joins the same pair of current
    // ancestors: that union links the same two sets (ancestors never leave a
    // set), so the result is unchanged and the shared roots see fewer atomics.
    const int rp = act ? __ldcg(parent + p) : -1;
    unsigned long long key[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int rq = need[d] ? __ldcg(parent + q[d]) : -2;
      const unsigned lo = unsigned(min(rp, rq)), hi = unsigned(max(rp, rq));
      key[d] = need[d] ? ((unsigned long long)lo << 32 | hi) : ~0ull - d;
    }
    unsigned long long prev[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) prev[d] = __shfl_up_sync(0xFFFFFFFFu, key[d], 1);
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      if (!need[d] || (key[d] >> 32) == (key[d] & 0xFFFFFFFFull)) continue;
      bool dup = false;
#pragma unroll
      for (int e = 0; e < d; ++e) dup |= key[e] == key[d];
      if (lane > 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) dup |= prev[e] == key[d];
      }
      if (!dup) uf_union(parent, p, q[d]);
    }
  }
}

template <typename Pred>
void uf_label(Pred pr, int h, int w, int conn8, int* parent, int /*sm_count*/, cudaStream_t st) {
  const long long n = (long long)h * w;
  const dim3 tiles(cdiv(w, kTileW), cdiv(h, kTileH));
  k_uf_local<<<tiles, kTileW * kTileH, 0, st>>>(pr, h, w, conn8, parent);
  RPD_LAUNCH_CHECK();
  k_uf_border<<<cdiv(tiles.x * tiles.y, kBorderWarps), 32 * kBorderWarps, 0, st>>>(pr, h, w, conn8,
                                                                                   parent);
  RPD_LAUNCH_CHECK();
  k_uf_flatten<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(h, w, parent);
  RPD_LAUNCH_CHECK();
}

// Segmented (contiguous-run) warp sum: lanes with equal `key` in a contiguous
// run are summed into the run's first lane; returns true on that lane.
// key < 0 lanes are skipped.
template <typename T>
__device__ __forceinline__ T shfl_down_any(T x, int off) {
  return __shfl_down_sync(0xFFFFFFFFu, x, off);
}
__device__ __forceinline__ Acc128 shfl_down_any(Acc128 x, int off) {
  Acc128 r;
  r.lo = __shfl_down_sync(0xFFFFFFFFu, x.lo, off);
  r.hi = __shfl_down_sync(0xFFFFFFFFu, x.hi, off);
  return r;
}
__device__ __forceinline__ Acc128 acc_add(Acc128 a, Acc128 b) {
  Acc128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}
template <typename T>
__device__ __forceinline__ T plus_(T a, T b) {
  return a + b;
}
__device__ __forceinline__ Acc128 plus_(Acc128 a, Acc128 b) { return acc_add(a, b); }

struct RunInfo {
  int end;    // last lane of this lane's run
  bool head;  // first lane of its run (and key >= 0)
};

__device__ __forceinline__ RunInfo run_info(int key) {
  const int lane = threadIdx.x & 31;
  const int nxt = __shfl_down_sync(0xFFFFFFFFu, key, 1);
  const int prv = __shfl_up_sync(0xFFFFFFFFu, key, 1);
  const bool tail = lane == 31 || nxt != key;
  const unsigned tails = __ballot_sync(0xFFFFFFFFu, tail);
  RunInfo r;
  r.end = lane + __ffs(tails >> lane) - 1;
  r.head = key >= 0 && (lane == 0 || prv != key);
  return r;
}

// As run_info, but a lane with brk set also starts a new run (row starts:
// a run then lies in one image row, so its count and coordinate sums follow
// from its bounds).
__device__ __forceinline__ RunInfo run_info_brk(int key, bool brk) {
  const int lane = threadIdx.x & 31;
  const int nxt = __shfl_down_sync(0xFFFFFFFFu, key, 1);
  const int prv = __shfl_up_sync(0xFFFFFFFFu, key, 1);
  const unsigned brks = __ballot_sync(0xFFFFFFFFu, brk);
  const bool tail = lane == 31 || nxt != key || ((brks >> (lane + 1)) & 1u);
  const unsigned tails = __ballot_sync(0xFFFFFFFFu, tail);
  RunInfo r;
  r.end = lane + __ffs(tails >> lane) - 1;
  r.head = key >= 0 && (lane == 0 || prv != key || brk);
  return r;
}

template <typename T>
__device__ __forceinline__ T run_sum(T x, const RunInfo& ri) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T o = shfl_down_any(x, off);
    if (lane + off <= ri.end) x = plus_(x, o);
  }
  return x;
}

// Exact 128-bit sums accumulated with fire-and-forget reductions: v = a2*2^64
// + a1*2^32 + a0 where every added term of a0 / a1 is < 2^32 (no carries to
// track), a2 takes the signed top word.
struct __align__(16) AccSum {
  unsigned long long a0, a1;
  long long a2;
  long long pad;
};

__device__ __forceinline__ void red_add_acc(AccSum* s, Acc128 x) {
  atomicAdd(&s->a0, x.lo & 0xFFFFFFFFull);
  atomicAdd(&s->a1, x.lo >> 32);
  atomicAdd(reinterpret_cast<unsigned long long*>(&s->a2), (unsigned long long)x.hi);
}

__device__ __forceinline__ Acc128 acc_value(const AccSum& s) {
  const unsigned long long lo = s.a0 + (s.a1 << 32);
  const long long carry = lo < s.a0 ? 1 : 0;
  return Acc128{lo, s.a2 + (long long)(s.a1 >> 32) + carry};
}

__device__ __forceinline__ void atomic_add_acc(Acc128* a, Acc128 x) {
  const unsigned long long old = atomicAdd(&a->lo, x.lo);
  const unsigned long long carry = (old + x.lo) < old ? 1ull : 0ull;
  const unsigned long long hi = (unsigned long long)x.hi + carry;
  if (hi) atomicAdd(reinterpret_cast<unsigned long long*>(&a->hi), hi);
}

// Exact fixed-point image of a float: x * 2^100 as a signed 128-bit integer.
// Exact for 2^-77 <= |x| < 2^27 (and 0); anything else sets *inexact.
__device__ __forceinline__ Acc128 to_fixed(float x, int* inexact) {
  Acc128 r{0ull, 0ll};
  if (x == 0.0f) return r;
  const uint32_t b = __float_as_uint(x);
  const int e = int((b >> 23) & 0xFFu);
  unsigned long long m = b & 0x7FFFFFu;
  int ex;
  if (e == 0) {
    ex = -149;
  } else {
    m |= 0x800000u;
    ex = e - 150;
  }
  int s = ex + 100;
  if (s < 0) {
    *inexact = 1;
    m = (-s >= 64) ? 0 : (m >> (-s));
    s = 0;
  }
  if (s > 103) {
    *inexact = 1;
    s = 103;
  }
  if (s < 64) {
    r.lo = m << s;
    r.hi = (s > 40) ? (long long)(m >> (64 - s)) : 0;
  } else {
    r.lo = 0;
    r.hi = (long long)(m << (s - 64));
  }
  if (b >> 31) {
    r.lo = ~r.lo + 1ull;
    r.hi = ~r.hi + (r.lo == 0 ? 1 : 0);
  }
  return r;
}

// Warp run sum of `x` (per contiguous key run, see run_info) added to the
// run's AccSum by its head lane.  Fast path when every participating value is
// 0 or has an exponent field in [117, 140] (2^-10 <= |x| < 2^14): such values
// are multiples of 2^-33 below 2^14, so every partial sum of <= 32 of them is
// a multiple of 2^-33 below 2^19 — 52 significant bits — and the run is summed
// EXACTLY in double (one DADD per step); the head converts it to the integer
// s = sum * 2^40 (< 2^59) that lands in the accumulator as s * 2^60 (a1 and
// a2 words; its a0 part is zero).  Otherwise the 128-bit fixed-point path.
// Both give the same exact total.
__device__ __forceinline__ void run_add_value(AccSum* sx, int key, bool active, float x,
                                              const RunInfo& ri, int* inexact) {
  const uint32_t b = __float_as_uint(x);
  const int e = int((b >> 23) & 0xFFu);
  const bool zero = !active || (b << 1) == 0u;
  const bool fast = zero || (e >= 117 && e <= 140);
  if (__all_sync(0xFFFFFFFFu, fast)) {
    double d = zero ? 0.0 : double(x);
    d = run_sum(d, ri);
    if (ri.head) {
      const long long v = __double2ll_rz(d * 1099511627776.0);  // exact: d * 2^40
      const unsigned long long a1 = ((unsigned long long)v << 60) >> 32;
      if (a1) atomicAdd(&sx[key].a1, a1);
      atomicAdd(reinterpret_cast<unsigned long long*>(&sx[key].a2), (unsigned long long)(v >> 4));
    }
  } else {
    int bad = 0;
    Acc128 ax = active ? to_fixed(x, &bad) : Acc128{0ull, 0ll};
    if (bad) atomicOr(inexact, 1);
    ax = run_sum(ax, ri);
    if (ri.head) red_add_acc(&sx[key], ax);
  }
}

// Correctly rounded double of (a * 2^-100).
__device__ __forceinline__ double fixed_to_double(Acc128 a) {
  const bool neg = a.hi < 0;
  unsigned __int128 x = (unsigned __int128)(unsigned long long)a.hi << 64 | a.lo;
  if (neg) x = ~x + 1;
  if (x == 0) return 0.0;
  const unsigned long long hi = (unsigned long long)(x >> 64);
  const int top = hi ? 127 - __clzll(hi) : 63 - __clzll((unsigned long long)x);
  double mag;
  if (top <= 52) {
    mag = double((unsigned long long)x);
    mag = ldexp(mag, -100);
  } else {
    const int shift = top - 52;
    unsigned long long mant = (unsigned long long)(x >> shift);
    const unsigned __int128 rem = x & ((((unsigned __int128)1) << shift) - 1);
    const unsigned __int128 half = ((unsigned __int128)1) << (shift - 1);
    if (rem > half || (rem == half && (mant & 1ull))) ++mant;
    mag = ldexp(double(mant), shift - 100);
  }
  return neg ? -mag : mag;
}

}  // namespace rpdg
