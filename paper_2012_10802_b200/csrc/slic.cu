// slic.cu — SLIC superpixels + pooling for sm_100a.
//
// Reference: /root/reference/proj/src/segmentation.cpp:13-249.
//
//  * assign_pixels (:30-72) is pixel-centric: each pixel scans the centre
//    bucket grid for every centre whose window [lround(c) +- ceil(S)] contains
//    it and keeps the lexicographic minimum (dist, k) — identical to the
//    reference's ascending-k scan with strict `<`.  Pixels covered by no window
//    go to a warp-per-pixel nearest-centre fallback.
//  * update_centers (:74-93) and pool_superpixels (:231-249) sum per label;
//    coordinate sums are exact int64, value sums are exact signed 128-bit
//    fixed point (x * 2^100), so the atomics' order cannot change the result.
//  * enforce_connectivity (:98-166): union-find pieces, largest piece per label
//    (ties -> first piece in scan order), then a level-synchronous BFS that
//    reproduces the reference's FIFO claim order exactly: the level-(k+1) queue
//    is ordered by (claimer's queue rank, neighbour index), and an orphan is
//    claimed by its adjacent level-k pixel of lowest queue rank.
//  * compaction to 1..count by first appearance in scan order (:218-224).

#include <cub/cub.cuh>

#include "ccl.cuh"
#include "scan.cuh"

namespace rpdg {

// four pixels per thread (launched with max(1, cdiv(n, 1024)) blocks of 256)
__global__ void k_uf_flatten(int h, int w, int* parent) {
  const long long n = (long long)h * w;
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 + 3 < n) {
    int4 r = *reinterpret_cast<const int4*>(parent + p0);
    // a pixel whose parent is itself or a root keeps it
    if (r.x >= 0) r.x = uf_find(parent, r.x);
    if (r.y >= 0) r.y = uf_find(parent, r.y);
    if (r.z >= 0) r.z = uf_find(parent, r.z);
    if (r.w >= 0) r.w = uf_find(parent, r.w);
    *reinterpret_cast<int4*>(parent + p0) = r;
    return;
  }
  for (long long p = p0; p < n; ++p)
    if (parent[p] >= 0) parent[p] = uf_find(parent, int(p));
}

namespace {

constexpr int kDU[8] = {1, -1, 0, 0, 1, 1, -1, -1};  // segmentation.cpp:104-105
constexpr int kDV[8] = {0, 0, 1, -1, 1, -1, 1, -1};
__constant__ int c_du[8] = {1, -1, 0, 0, 1, 1, -1, -1};
__constant__ int c_dv[8] = {0, 0, 1, -1, 1, -1, 1, -1};

struct Centers {
  double* cu;
  double* cv;
  double* val;
  int* icu;
  int* icv;
};

struct CenterSums {
  int* n;
  long long* su;
  long long* sv;
  AccSum* sx;
};

// values_or_zero, segmentation.cpp:13-19
// Elementwise passes below take four pixels per thread (16-byte accesses;
// workspace buffers are 256-byte aligned), launched with max(1, cdiv(n, 1024)).
__global__ void k_values_or_zero(const float* __restrict__ d2, long long n, float* __restrict__ vals) {
  auto z = [](float x) { return x != kInvalid ? x : 0.0f; };
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 + 3 < n && (reinterpret_cast<uintptr_t>(d2) & 15u) == 0) {
    const float4 x = *reinterpret_cast<const float4*>(d2 + p0);
    *reinterpret_cast<float4*>(vals + p0) = make_float4(z(x.x), z(x.y), z(x.z), z(x.w));
    return;
  }
  for (long long p = p0; p < min(n, p0 + 4); ++p) vals[p] = z(d2[p]);
}

// gradient_at, segmentation.cpp:22-28 (float difference, squared in double)
__device__ __forceinline__ double gradient_at(const float* vals, int h, int w, int u, int v) {
  const float c = vals[size_t(v) * w + u];
  const double gu = double(vals[size_t(v) * w + min(u + 1, w - 1)] - c);
  const double gv = double(vals[size_t(min(v + 1, h - 1)) * w + u] - c);
  return gu * gu + gv * gv;
}

// Seeds on the nu x nv grid nudged to the lowest gradient (:182-206).
__global__ void k_seeds(const float* __restrict__ vals, int h, int w, int nu, int nv, double su,
                        double sv, Centers c) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nu * nv) return;
  const int i = k % nu, j = k / nu;
  const int cu = int((i + 0.5) * su), cv = int((j + 0.5) * sv);
  double best = __longlong_as_double(0x7FF0000000000000ll);
  int bu = cu, bv = cv;
  for (int dv = -1; dv <= 1; ++dv)
    for (int du = -1; du <= 1; ++du) {
      const int uu = min(max(cu + du, 0), w - 1), vv = min(max(cv + dv, 0), h - 1);
      const double g = gradient_at(vals, h, w, uu, vv);
      if (g < best) {
        best = g;
        bu = uu;
        bv = vv;
      }
    }
  c.cu[k] = double(bu);
  c.cv[k] = double(bv);
  c.val[k] = double(vals[size_t(bv) * w + bu]);
}

// A centre as the assignment tiles read it, stored in bucket order.
struct __align__(16) CRec {
  int4 ik;       // icu, icv, k, 0
  double2 cuv;   // cu, cv
  double2 val;   // val, 0
};

// Centre grid for the assignment: bucket (bx, by) of side B holds up to
// kBucketCap centre records in a fixed-capacity slot array, filled with one
// atomic per centre (order inside a bucket is irrelevant: the assignment keeps
// the lexicographic (dist, k) minimum).  A bucket that overflows sets the
// round's overflow flag; the assignment then falls back to a brute-force scan
// of every centre.  Counts and flags are double-buffered by round parity: the
// round-r kernel fills buffer r & 1 and clears buffer (r + 1) & 1 for the next
// round (its previous user, the round r - 1 assignment, is complete).
constexpr int kBucketCap = 8;

struct CenterGrid {
  int B, nbx, nby;
  int* count[2];  // per bucket
  int* ovf[2];    // one flag
  CRec* rec;      // nb * kBucketCap
};

// Nearest-centre fallback of one orphan pixel (segmentation.cpp:59-71), one
// warp: lane-strided scan of every centre, then the lexicographic (d, k)
// minimum across the warp; lane 0 writes the label (and the sums).
template <bool SUMS>
__device__ __forceinline__ void fallback_pixel(int p, int w, const Centers& c, int K,
                                               int32_t* __restrict__ labels,
                                               const float* __restrict__ vals, CenterSums& s,
                                               int* __restrict__ inexact) {
  const int lane = threadIdx.x & 31;
  const int u = p % w, v = p / w;
  double best = __longlong_as_double(0x7FF0000000000000ll);
  int bk = -1;
  for (int k = lane; k < K; k += 32) {
    const double du = double(u) - c.cu[k], dv = double(v) - c.cv[k];
    const double d = du * du + dv * dv;
    if (d < best) {
      best = d;
      bk = k;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
    const int ok = __shfl_xor_sync(0xFFFFFFFFu, bk, off);
    if (ok >= 0 && (bk < 0 || ob < best || (ob == best && ok < bk))) {
      best = ob;
      bk = ok;
    }
  }
  if (lane == 0 && bk >= 0) {
    labels[p] = bk + 1;
    if (SUMS) {
      int bad = 0;
      const int l = bk + 1;
      atomicAdd(&s.n[l], 1);
      red_add_acc(&s.sx[l], to_fixed(vals[p], &bad));
      if (bad) atomicOr(inexact, 1);
      atomicAdd(reinterpret_cast<unsigned long long*>(&s.su[l]), (unsigned long long)u);
      atomicAdd(reinterpret_cast<unsigned long long*>(&s.sv[l]), (unsigned long long)v);
    }
  }
}

// One SLIC round's centre step:
//  1. the previous assignment's orphans (pixels no window covers) take their
//     nearest centre and add their sums (assign_pixels' fallback,
//     segmentation.cpp:59-71), when there are any;
//  2. update_centers' tail (segmentation.cpp:88-92) of the previous
//     assignment's sums when `finalize`, the lround window centres
//     (:38-41) and the bucket insert for this round's assignment.
struct Orphans {
  const int* list;
  int* count;
  const float* vals;
  int32_t* labels;
  int w;
  int* inexact;
  unsigned* done;  // blocks done with the orphans (the last one finalises)
};

// Incremental rounds (RPD_SLIC_INCREMENTAL).  A pixel's assignment depends
// only on its value and on the centres whose window holds it, so a tile that
// no MOVED centre's window reaches — neither the window of the previous round
// nor this round's — keeps every label, and the assignment skips it.  A centre
// moved when (cu, cv, value) differ bitwise from the previous round.  The
// per-label sums then persist across rounds and the assignment applies only
// the changed pixels (- old label, + new label): all sums are exact integers,
// so the totals are those of a full pass.  Orphans (pixels no window covers)
// take the nearest of ALL centres: a round that follows one with orphans
// marks every tile.
//   flags[b][t]: tile t must be re-assigned in the round using buffer b;
//   flags[b][ntx * nty]: every tile must.  Double-buffered like the grid counts.
struct TileDirty {
  int* flags[2];
  int ntx, nty;
  int tile_u, tile_v;
  int w, h, win;
  unsigned long long* moved_dbg;  // checked build: moved-centre count
};

__device__ __forceinline__ void mark_window(const TileDirty& td, int* __restrict__ flags, int iu,
                                            int iv) {
  const int u0 = max(iu - td.win, 0), u1 = min(iu + td.win, td.w - 1);
  const int v0 = max(iv - td.win, 0), v1 = min(iv + td.win, td.h - 1);
  if (u0 > u1 || v0 > v1) return;
  for (int ty = v0 / td.tile_v; ty <= v1 / td.tile_v; ++ty)
    for (int tx = u0 / td.tile_u; tx <= u1 / td.tile_u; ++tx) flags[ty * td.ntx + tx] = 1;
}

// finalize: 0 = seeds as they are (round 0); 1 = update_centers' tail, the sums
// are kept (incremental rounds); 2 = the tail, then the sums are zeroed.
__global__ void k_centers(Centers c, int K, CenterSums s, int finalize, CenterGrid g, int cur,
                          Orphans o, TileDirty td) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  int nthreads = gridDim.x * blockDim.x;
  const int norph = *o.count;  // written by the previous round's assignment
  if (norph > 0) {
    // (rare) orphans first; the LAST block to finish them then runs the
    // whole centre step alone, so every orphan's sums are in before any
    // centre is finalised (no co-residency needed)
    __shared__ bool s_last;
    const int nwarps = nthreads >> 5;
    for (int i = tid >> 5; i < norph; i += nwarps)
      fallback_pixel<true>(o.list[i], o.w, c, K, o.labels, o.vals, s, o.inexact);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(o.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) *o.done = 0u;  // rearmed for the next round
    tid = threadIdx.x;
    nthreads = blockDim.x;
  }
  const int nb = g.nbx * g.nby;
  int* cnt_next = g.count[cur ^ 1];
  for (int b = tid; b < nb; b += nthreads) cnt_next[b] = 0;
  const int ntiles = td.ntx * td.nty;
  if (td.flags[0]) {
    int* dirty_next = td.flags[cur ^ 1];
    for (int t = tid; t <= ntiles; t += nthreads) dirty_next[t] = 0;
  }
  if (tid == 0) {
    *g.ovf[cur ^ 1] = 0;
    *o.count = 0;  // every block has read it (the count-0 path rewrites 0)
    if (td.flags[0] && norph > 0) td.flags[cur][ntiles] = 1;
  }
  for (int k = tid; k < K; k += nthreads) {
    if (finalize) {
      // L2 loads: with orphans, other blocks of this launch added to the sums
      const int l = k + 1;
      const int n = __ldcg(s.n + l);
      if (n > 0) {
        const double dn = double(n);
        const double ncu = double(__ldcg(s.su + l)) / dn;
        const double ncv = double(__ldcg(s.sv + l)) / dn;
        const AccSum sx{__ldcg(&s.sx[l].a0), __ldcg(&s.sx[l].a1), __ldcg(&s.sx[l].a2), 0ll};
        const double nval = fixed_to_double(acc_value(sx)) / dn;
        if (td.flags[0]) {
          const bool moved = __double_as_longlong(ncu) != __double_as_longlong(c.cu[k]) ||
                             __double_as_longlong(ncv) != __double_as_longlong(c.cv[k]) ||
                             __double_as_longlong(nval) != __double_as_longlong(c.val[k]);
          if (moved) {
#ifdef RPD_DEBUG_KNOBS
            if (td.moved_dbg) atomicAdd(td.moved_dbg, 1ull);
#endif
            mark_window(td, td.flags[cur], c.icu[k], c.icv[k]);  // the window it leaves
            mark_window(td, td.flags[cur], int(lround(ncu)), int(lround(ncv)));
          }
        }
        c.cu[k] = ncu;
        c.cv[k] = ncv;
        c.val[k] = nval;
      }
      if (finalize == 2) {
        s.n[l] = 0;
        s.su[l] = 0;
        s.sv[l] = 0;
        s.sx[l] = AccSum{0ull, 0ull, 0ll, 0ll};
      }
    }
    const double cu = c.cu[k], cv = c.cv[k];
    const int iu = int(lround(cu)), iv = int(lround(cv));
    c.icu[k] = iu;
    c.icv[k] = iv;
    const int bx = min(max(iu, 0) / g.B, g.nbx - 1), by = min(max(iv, 0) / g.B, g.nby - 1);
    const int b = by * g.nbx + bx;
    const int slot = atomicAdd(&g.count[cur][b], 1);
    if (slot < kBucketCap)
      g.rec[size_t(b) * kBucketCap + slot] =
          CRec{make_int4(iu, iv, k, 0), make_double2(cu, cv), make_double2(c.val[k], 0.0)};
    else
      *g.ovf[cur] = 1;
  }
}

struct AssignArgs {
  const float* vals;
  int h, w, K;
  Centers c;
  const int* bcount;  // this round's bucket counts
  const int* ovf;     // this round's bucket overflow flag
  const CRec* recs;
  int B, nbx, nby, win;
  double sw;
  int32_t* labels;
  int* orphan_list;
  int* orphan_count;
  int* inexact;
  int force_walk;  // checked build only (RPD_SLIC_FORCE_WALK): exercise the brute-force path
  uint32_t b_magic;  // floor(2^32 / B) + 1: x / B == umulhi(x, b_magic) for 0 <= x < 2^16 (0: divide)
  const int* dirty;  // this round's tile flags (TileDirty), SKIP kernels only
  unsigned long long* tiles;  // {assigned, skipped, moved centres, changed pixels} counters (rpd_stats)
};

// Bucket index of a non-negative coordinate (tile-uniform values: one
// multiply-high instead of an integer division per thread).
__device__ __forceinline__ int bucket_of(const AssignArgs& a, int x) {
  return a.b_magic ? int(__umulhi(uint32_t(x), a.b_magic)) : x / a.B;
}

// assign_pixels, segmentation.cpp:30-57 (windowed part) for one pixel by
// scanning every centre; used when a tile's candidate list or a bucket
// overflows (pathological centre pile-ups).
__device__ __forceinline__ int assign_walk(const AssignArgs& a, int u, int v, double x) {
  double best = __longlong_as_double(0x7FF0000000000000ll);
  int bk = -1;
  for (int k = 0; k < a.K; ++k) {
    if (abs(u - a.c.icu[k]) > a.win || abs(v - a.c.icv[k]) > a.win) continue;
    const double dval = x - a.c.val[k];
    const double du = double(u) - a.c.cu[k], dv = double(v) - a.c.cv[k];
    const double dist = dval * dval + (du * du + dv * dv) * a.sw;
    if (dist < best || (dist == best && k < bk)) {
      best = dist;
      bk = k;
    }
  }
  return bk;
}

// Tiled assign_pixels with the next update_centers' sums fused in.  A CTA owns
// a 32 x kTileV pixel tile; the centres of every bucket that can reach the tile are
// staged once in shared memory, each pixel keeps the lexicographic minimum
// (dist, k) of the centres whose window holds it (== ascending-k strict `<`),
// and — when SUMS — the pixel's (1, u, v, value) is added to its label's sums
// with warp run aggregation (a warp is one tile row).  Pixels without a window
// are left for the fallback kernel, which adds their sums itself.
#ifndef RPD_ASSIGN_TILEV
// tile rows of large rasters (5 per warp): the staging is shared by more
// pixels, config 5 +1.3 % frames/s over 24 rows (32 / 40 rows equal, 48 rows
// lose it again through their shared memory)
#define RPD_ASSIGN_TILEV 40
#endif
#ifndef RPD_ASSIGN_TILEV_SMALL
// tile rows of rasters with few tiles (3 per warp): config 1's 240 x 320 is
// 2.5 % faster with the extra CTAs
#define RPD_ASSIGN_TILEV_SMALL 24
#endif
#ifndef RPD_ASSIGN_ROWCAP
#define RPD_ASSIGN_ROWCAP 24
#endif
#ifndef RPD_ASSIGN_UNROLL
#define RPD_ASSIGN_UNROLL 1  // candidate loop unroll (0: the compiler's choice; 1 measured best)
#endif
constexpr int kAssignUnroll = RPD_ASSIGN_UNROLL > 0 ? RPD_ASSIGN_UNROLL : 1;
constexpr int kTileU = 32, kTileVLarge = RPD_ASSIGN_TILEV, kTileVSmall = RPD_ASSIGN_TILEV_SMALL,
              kMaxTileCenters = 192;
constexpr int kRowCap = RPD_ASSIGN_ROWCAP;  // candidate records per tile row (more: per-pixel bucket walk)
#ifndef RPD_ASSIGN_THREADS
#define RPD_ASSIGN_THREADS 256
#endif
constexpr int kAssignThreads = RPD_ASSIGN_THREADS;
constexpr int kAssignWarps = kAssignThreads / 32;
#ifndef RPD_ASSIGN_MINB
#define RPD_ASSIGN_MINB (6 * 256 / RPD_ASSIGN_THREADS)  // resident CTAs per SM the register budget targets
#endif
// a warp owns rows w, w + kAssignWarps, ...
static_assert(kTileVLarge % kAssignWarps == 0 && kTileVSmall % kAssignWarps == 0,
              "whole tile rows per warp");
static_assert(kTileVLarge <= 256 && kTileVSmall <= 256,
              "a candidate's tile-row range is packed into two bytes");

// One pixel's (1, u, v, value) added to (sign = 1) or taken from (sign = -1)
// label l's exact sums: the incremental rounds' changed pixels.
__device__ __forceinline__ void delta_pixel(const CenterSums& s, int l, int sign, int u, int v,
                                            float x, int* __restrict__ inexact) {
  int bad = 0;
  Acc128 ax = to_fixed(x, &bad);
  if (bad) atomicOr(inexact, 1);
  if (sign < 0) {
    ax.lo = ~ax.lo + 1ull;
    ax.hi = ~ax.hi + (ax.lo == 0 ? 1 : 0);
  }
  atomicAdd(&s.n[l], sign);
  atomicAdd(reinterpret_cast<unsigned long long*>(&s.su[l]), (unsigned long long)(long long)(sign * u));
  atomicAdd(reinterpret_cast<unsigned long long*>(&s.sv[l]), (unsigned long long)(long long)(sign * v));
  red_add_acc(&s.sx[l], ax);
}

// SUMS: 0 = labels only (the last round), 1 = every pixel adds to its label's
// sums (round 0, and every round of the non-incremental build), 2 = the sums
// persist: only a pixel whose label changed moves its terms (see TileDirty).
// SKIP: tiles no moved centre reaches return at once.
template <int SUMS, bool SKIP, int kTileV>
__global__ void __launch_bounds__(kAssignThreads, RPD_ASSIGN_MINB)
    k_assign_tile(const __grid_constant__ AssignArgs a, CenterSums s) {
  constexpr int kRowsPerWarp = kTileV / kAssignWarps;
  if (SKIP) {
    const int ntiles = gridDim.x * gridDim.y;
    const bool dirty = (a.dirty[blockIdx.y * gridDim.x + blockIdx.x] | a.dirty[ntiles]) != 0;
    if (threadIdx.x == 0) atomicAdd(a.tiles + (dirty ? 0 : 1), 1ull);
    if (!dirty) return;
  }
  __shared__ int s_cnt;
  __shared__ int s_rowcnt[kTileV];
  // candidate c: s_cd[2c] = (cu, cv), s_cd[2c+1] = (val, icu | k << 32)
  __shared__ double2 s_cd[2 * kMaxTileCenters];
  __shared__ int s_icv[kMaxTileCenters];  // first | last << 8 tile row of the candidate's window
  // per tile row, the candidates whose window reaches it: {cu, (v - cv)^2}, {val, icu | k << 32}
  // (+1: rows start 4 banks apart; an unpadded row pitch of 768 bytes put every row of the
  // distribution step on the same banks, 79 % of its store wavefronts were conflicts)
  __shared__ double2 s_rec[kTileV][2 * kRowCap + 1];
  const int tx = threadIdx.x % 32, wid = threadIdx.x / 32;
  const int u0 = blockIdx.x * kTileU, v0 = blockIdx.y * kTileV;
  const int u = u0 + tx;
  const int win = a.win;
  // pixel values first (their loads overlap the candidate fill); one 32-bit
  // pixel index per thread, advanced by a row stride (H * W < 2^31: the orphan
  // list holds int indices)
  const bool uin = u < a.w;
  const int p0 = (v0 + wid) * a.w + u;
  const int pstride = kAssignWarps * a.w;
  float xf[kRowsPerWarp];
#pragma unroll
  for (int q = 0; q < kRowsPerWarp; ++q)
    xf[q] = (uin && v0 + wid + kAssignWarps * q < a.h) ? a.vals[p0 + q * pstride] : 0.0f;
  int oldl[kRowsPerWarp];
  if (SUMS == 2) {
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q)
      oldl[q] = (uin && v0 + wid + kAssignWarps * q < a.h) ? a.labels[p0 + q * pstride] : 0;
  }
  for (int r = threadIdx.x; r < kTileV; r += blockDim.x) s_rowcnt[r] = 0;
  if (threadIdx.x == 0) s_cnt = 0;
  const bool walk_all = a.force_walk || *a.ovf != 0;  // a bucket overflowed this round
  // bucket range of the tile +- win
  const int bx0 = u0 - win < 0 ? 0 : bucket_of(a, u0 - win);
  const int by0 = v0 - win < 0 ? 0 : bucket_of(a, v0 - win);
  const int nbxr = min(a.nbx - 1, bucket_of(a, u0 + kTileU - 1 + win)) - bx0 + 1;
  const int nbyr = min(a.nby - 1, bucket_of(a, v0 + kTileV - 1 + win)) - by0 + 1;
  __syncthreads();
  if (!walk_all) {
    // one (bucket, slot) item per thread; keep the centres whose window
    // reaches the tile
    for (int t = threadIdx.x; t < nbxr * nbyr * kBucketCap; t += blockDim.x) {
      const int bl = t / kBucketCap, slot = t % kBucketCap;
      const int b = (by0 + bl / nbxr) * a.nbx + bx0 + bl % nbxr;
      if (slot >= a.bcount[b]) continue;
      const CRec* rec = a.recs + size_t(b) * kBucketCap + slot;
      const int4 ik = rec->ik;
      const int du = ik.x < u0 ? u0 - ik.x : (ik.x > u0 + kTileU - 1 ? ik.x - (u0 + kTileU - 1) : 0);
      const int dv = ik.y < v0 ? v0 - ik.y : (ik.y > v0 + kTileV - 1 ? ik.y - (v0 + kTileV - 1) : 0);
      if (du > win || dv > win) continue;
      const int slotc = atomicAdd(&s_cnt, 1);
      if (slotc >= kMaxTileCenters) continue;  // tile overflow: per-pixel scan below
      s_cd[2 * slotc] = rec->cuv;
      s_cd[2 * slotc + 1] = make_double2(
          rec->val.x, __longlong_as_double((long long)(uint32_t(ik.x) | (uint64_t(uint32_t(ik.z)) << 32))));
      // tile rows the centre's window reaches (dv <= win: never empty)
      s_icv[slotc] = (max(ik.y - win, v0) - v0) | ((min(ik.y + win, v0 + kTileV - 1) - v0) << 8);
    }
  }
  __syncthreads();
  int nc = walk_all ? kMaxTileCenters + 1 : s_cnt;
  if (nc <= kMaxTileCenters) {
    // distribute the candidates over the rows they reach, with the row's
    // (v - cv)^2 precomputed (the reference's dv * dv, segmentation.cpp:48)
    // one (candidate, row) item per thread, consecutive threads on
    // consecutive rows (a warp's counter atomics rarely collide); every
    // thread has work
    for (int t = threadIdx.x; t < nc * kTileV; t += blockDim.x) {
      const int i = t / kTileV, r = t - i * kTileV;
      const int rows = s_icv[i];
      if (r < (rows & 255) || r > (rows >> 8)) continue;
      const double2 cuv = s_cd[2 * i];
      const int slot = atomicAdd(&s_rowcnt[r], 1);
      if (slot < kRowCap) {
        const double dv = double(v0 + r) - cuv.y;
        s_rec[r][2 * slot] = make_double2(cuv.x, dv * dv);
        s_rec[r][2 * slot + 1] = s_cd[2 * i + 1];
      }
    }
  }
  __syncthreads();
  if (nc <= kMaxTileCenters) {  // a row list overflowed: per-pixel bucket walk for the tile
    bool ov = false;
#pragma unroll
    for (int r0 = 0; r0 < kTileV; r0 += 32) ov |= r0 + tx < kTileV && s_rowcnt[r0 + tx] > kRowCap;
    const bool over = __any_sync(0xFFFFFFFFu, ov);
    if (over) nc = kMaxTileCenters + 1;
  }
#pragma unroll
  for (int q = 0; q < kRowsPerWarp; ++q) {
    const int ty = wid + kAssignWarps * q;
    const int v = v0 + ty;  // uniform across the warp
    const bool in = uin && v < a.h;
    const int p = p0 + q * pstride;
    const double x = double(xf[q]);
    double best = __longlong_as_double(0x7FF0000000000000ll);
    int bk = -1;
    if (nc <= kMaxTileCenters) {
      const double du0 = double(u), sw = a.sw;
      const int nr = s_rowcnt[ty];
      const unsigned span = 2u * unsigned(win);
#if RPD_ASSIGN_UNROLL > 0
#pragma unroll kAssignUnroll
#endif
      for (int j = 0; j < nr; ++j) {
        const double2 cd = s_rec[ty][2 * j];      // cu, (v - cv)^2
        const double2 vk = s_rec[ty][2 * j + 1];  // val, icu | k << 32
        const unsigned long long ik = (unsigned long long)__double_as_longlong(vk.y);
        const int icu = int(uint32_t(ik)), k = int(ik >> 32);
        const double dval = x - vk.x;
        const double du = du0 - cd.x;
        const double dist = dval * dval + (du * du + cd.y) * sw;
        // |u - icu| <= win, branch-free; lexicographic (dist, k) minimum
        const bool inw = unsigned(u - icu + win) <= span;
        const bool take = inw & ((dist < best) | ((dist == best) & (k < bk)));
        best = take ? dist : best;
        bk = take ? k : bk;
      }
    }
    int label = -1;  // -1: outside the image
    if (in) {
      if (nc > kMaxTileCenters)
        bk = assign_walk(a, u, v, x);  // pathological centre pile-up: per-pixel bucket walk
      label = bk + 1;
      if (bk < 0) {
        const int slot = atomicAdd(a.orphan_count, 1);
        a.orphan_list[slot] = p;
      }
      if (SUMS == 2) {
        // persistent sums: a changed pixel leaves its old label and joins the
        // new one (an orphan joins through the fallback, like every round)
        if (label != oldl[q]) {
#ifdef RPD_DEBUG_KNOBS
          if (a.tiles) atomicAdd(a.tiles + 3, 1ull);  // changed pixels
#endif
          a.labels[p] = label;
          if (oldl[q] > 0) delta_pixel(s, oldl[q], -1, u, v, xf[q], a.inexact);
          if (label > 0) delta_pixel(s, label, 1, u, v, xf[q], a.inexact);
        }
      } else {
        a.labels[p] = label;
      }
    }
    if (SUMS == 1) {
      const int key = label > 0 ? label : -1;
      const RunInfo ri = run_info(key);
      run_add_value(s.sx, key, key > 0, xf[q], ri, a.inexact);
      // a run is a contiguous pixel segment of one row: count and coordinate
      // sums follow from its bounds
      // (32-bit: cnt <= 32 and coordinates < 2^26)
      const int cnt = ri.end - tx + 1;
      if (ri.head) {
        const unsigned su = unsigned(cnt * u + ((cnt * (cnt - 1)) >> 1));
        const unsigned sv = unsigned(cnt * v);
        atomicAdd(&s.n[key], cnt);
        atomicAdd(reinterpret_cast<unsigned long long*>(&s.su[key]), (unsigned long long)su);
        atomicAdd(reinterpret_cast<unsigned long long*>(&s.sv[key]), (unsigned long long)sv);
      }
    }
  }
}

// Nearest-centre fallback of the last round's orphans (the earlier rounds'
// run inside the next k_centers), one warp per pixel.
__global__ void k_assign_fallback(int w, Centers c, int K, int32_t* __restrict__ labels,
                                  const int* __restrict__ list, const int* __restrict__ count) {
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int n = *count;
  CenterSums none{};
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps)
    fallback_pixel<false>(list[i], w, c, K, labels, nullptr, none, nullptr);
}

// Per-label sums of (u, v, value, n) with warp run pre-aggregation.  `valid`
// restricts to valid pixels (pooling); vals may be the raw d2 then.
// nvalid != nullptr (the pipeline's final update fused with pool_superpixels):
// vals is the raw D2, an invalid value adds 0 (values_or_zero) and each
// label's valid pixels are counted into nvalid — its value sum is then also
// pool_superpixels' sum of valid D2 (segmentation.cpp:236-241).
__global__ void k_label_sums(const float* __restrict__ vals, const int32_t* __restrict__ labels,
                             int h, int w, int max_label, bool valid_only, bool coords,
                             CenterSums s, int* __restrict__ inexact,
                             int* __restrict__ nvalid = nullptr) {
  const long long n = (long long)h * w;
  const long long base = (long long)blockIdx.x * blockDim.x;
  for (long long p0 = base; p0 < n; p0 += (long long)gridDim.x * blockDim.x) {
    const long long p = p0 + threadIdx.x;
    int key = -1;
    float x = 0.0f;
    bool valid = false;
    if (p < n) {
      const int l = labels[p];
      x = vals[p];
      valid = x != kInvalid;
      if (nvalid && !valid) x = 0.0f;
      if (l >= 0 && l <= max_label && (!valid_only || valid)) key = l;
    }
    // (v, u) of this lane from one division per warp
    const long long pw = p0 + (threadIdx.x & ~31u);
    int v = int(pw / w), u = int(pw - (long long)v * w) + int(threadIdx.x & 31);
    while (u >= w) {
      u -= w;
      ++v;
    }
    const RunInfo ri = run_info_brk(key, u == 0);
    run_add_value(s.sx, key, key >= 0, x, ri, inexact);
    // runs lie in one row: count and coordinate sums from the run bounds
    const int cnt = ri.end - int(threadIdx.x & 31) + 1;
    const long long su = (long long)cnt * u + (long long)cnt * (cnt - 1) / 2;
    const long long sv = (long long)cnt * v;
    unsigned vmask = 0u;
    if (nvalid) vmask = __ballot_sync(0xFFFFFFFFu, valid && key >= 0);
    if (ri.head) {
      atomicAdd(&s.n[key], cnt);
      if (coords) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&s.su[key]), (unsigned long long)su);
        atomicAdd(reinterpret_cast<unsigned long long*>(&s.sv[key]), (unsigned long long)sv);
      }
      if (nvalid) {  // valid lanes of the run [lane, end]
        const int lane = int(threadIdx.x & 31);
        const unsigned run = (ri.end == 31 ? 0xFFFFFFFFu : ((2u << ri.end) - 1u)) & ~((1u << lane) - 1u);
        const int nv = __popc(vmask & run);
        if (nv) atomicAdd(&nvalid[key], nv);
      }
    }
  }
}

// update_centers tail (:88-92), then zero the sums for the next round.
// Label k+1 belongs to centre k.
__global__ void k_center_finalize(CenterSums s, Centers c, int K) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int l = k + 1;
  const int n = s.n[l];
  if (n > 0) {
    const double dn = double(n);
    c.cu[k] = double(s.su[l]) / dn;
    c.cv[k] = double(s.sv[l]) / dn;
    c.val[k] = fixed_to_double(acc_value(s.sx[l])) / dn;
  }
  s.n[l] = 0;
  s.su[l] = 0;
  s.sv[l] = 0;
  s.sx[l] = AccSum{0ull, 0ull, 0ll, 0ll};
}

__global__ void k_zero_sums(CenterSums s, int nlabels) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlabels) return;
  s.n[l] = 0;
  s.su[l] = 0;
  s.sv[l] = 0;
  s.sx[l] = AccSum{0ull, 0ull, 0ll, 0ll};
}

// ------------------------------------------------ enforce_connectivity ----
__global__ void k_piece_sizes(const int* __restrict__ parent, long long n, int* __restrict__ size) {
  for (long long p0 = (long long)blockIdx.x * blockDim.x; p0 < n;
       p0 += (long long)gridDim.x * blockDim.x) {
    const long long p = p0 + threadIdx.x;
    const int key = p < n ? parent[p] : -1;
    const RunInfo ri = run_info(key);
    if (ri.head) atomicAdd(&size[key], ri.end - int(threadIdx.x & 31) + 1);  // run length
  }
}

// Largest piece per label; ties go to the earlier piece (smaller root index).
__global__ void k_main_piece(const int* __restrict__ parent, const int32_t* __restrict__ labels,
                             const int* __restrict__ size, long long n,
                             unsigned long long* __restrict__ best) {
  // four pixels per thread (launched with max(1, cdiv(n, 1024)) blocks of 256)
  auto root = [&](long long p) {
    const unsigned long long key =
        ((unsigned long long)(unsigned)size[p] << 32) | (0xFFFFFFFFull - (unsigned long long)p);
    atomicMax(&best[labels[p]], key);
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

__global__ void k_orphans(const int* __restrict__ parent, int32_t* __restrict__ labels,
                          const unsigned long long* __restrict__ best, long long n,
                          int* __restrict__ claim) {
  auto keep = [&](int l, long long p, int par) {
    const long long root = (long long)(0xFFFFFFFFull - (best[l] & 0xFFFFFFFFull));
    return par == root ? l : 0;
  };
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 + 3 < n) {
    const int4 l = *reinterpret_cast<const int4*>(labels + p0);
    const int4 r = *reinterpret_cast<const int4*>(parent + p0);
    *reinterpret_cast<int4*>(labels + p0) =
        make_int4(keep(l.x, p0, r.x), keep(l.y, p0 + 1, r.y), keep(l.z, p0 + 2, r.z),
                  keep(l.w, p0 + 3, r.w));
    *reinterpret_cast<int4*>(claim + p0) = make_int4(0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF, 0x7FFFFFFF);
    return;
  }
  for (long long p = p0; p < min(n, p0 + 4); ++p) {
    labels[p] = keep(labels[p], p, parent[p]);
    claim[p] = 0x7FFFFFFF;
  }
}

// Level-0 frontier: kept pixels with an orphan neighbour, in scan order.
// Orphans are rare, so the flags (zeroed beforehand) are set from the orphan
// side: each orphan marks its kept 8-neighbours (plain stores of 1).
__global__ void k_frontier_flags(const int32_t* __restrict__ labels, int h, int w,
                                 int* __restrict__ flags) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  if (u >= w) return;
  const size_t p = size_t(v) * w + u;
  if (labels[p] != 0) return;
  for (int i = 0; i < 8; ++i) {
    const int nu = u + c_du[i], nv = v + c_dv[i];
    if (nu < 0 || nu >= w || nv < 0 || nv >= h) continue;
    const size_t q = size_t(nv) * w + nu;
    if (labels[q] != 0) flags[q] = 1;
  }
}

__global__ void k_scatter_flagged(const int* __restrict__ flags, const int* __restrict__ pos,
                                  long long n, int* __restrict__ list, int* __restrict__ total) {
  // four pixels per thread (launched with max(1, cdiv(n, 1024)) blocks of 256)
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 + 3 < n) {
    const int4 f = *reinterpret_cast<const int4*>(flags + p0);
    if (f.x | f.y | f.z | f.w) {
      const int4 q = *reinterpret_cast<const int4*>(pos + p0);
      if (f.x) list[q.x] = int(p0);
      if (f.y) list[q.y] = int(p0 + 1);
      if (f.z) list[q.z] = int(p0 + 2);
      if (f.w) list[q.w] = int(p0 + 3);
    }
  } else {
    for (long long p = p0; p < n; ++p)
      if (flags[p]) list[pos[p]] = int(p);
  }
  if (p0 <= n - 1 && n - 1 < p0 + 4) *total = pos[n - 1] + flags[n - 1];
}

// Ordered multi-source BFS (single CTA), segmentation.cpp:145-165.
constexpr int kBfsThreads = 1024;
__global__ void __launch_bounds__(kBfsThreads)
    k_bfs(int32_t* labels, int h, int w, int* claim, int* qa, int* qb, const int* n0) {
  using Scan = cub::BlockScan<int, kBfsThreads>;
  __shared__ typename Scan::TempStorage tmp;
  int na = *n0;
  int* A = qa;
  int* B = qb;
  while (na > 0) {
    for (int i = threadIdx.x; i < na; i += blockDim.x) {
      const int p = A[i];
      const int u = p % w, v = p / w;
      for (int j = 0; j < 8; ++j) {
        const int nu = u + c_du[j], nv = v + c_dv[j];
        if (nu < 0 || nu >= w || nv < 0 || nv >= h) continue;
        const int q = nv * w + nu;
        if (labels[q] == 0) atomicMin(&claim[q], i * 8 + j);
      }
    }
    __syncthreads();
    int nb = 0;
    for (int c0 = 0; c0 < na; c0 += blockDim.x) {
      const int i = c0 + threadIdx.x;
      int mine = 0;
      unsigned won = 0;
      int p = 0;
      if (i < na) {
        p = A[i];
        const int u = p % w, v = p / w;
        for (int j = 0; j < 8; ++j) {
          const int nu = u + c_du[j], nv = v + c_dv[j];
          if (nu < 0 || nu >= w || nv < 0 || nv >= h) continue;
          const int q = nv * w + nu;
          if (claim[q] == i * 8 + j) {
            won |= 1u << j;
            ++mine;
          }
        }
      }
      int off, tot;
      Scan(tmp).ExclusiveSum(mine, off, tot);
      if (won) {
        const int lab = labels[p];
        const int u = p % w, v = p / w;
        int o = nb + off;
        for (int j = 0; j < 8; ++j) {
          if (!(won >> j & 1u)) continue;
          const int q = (v + c_dv[j]) * w + (u + c_du[j]);
          labels[q] = lab;
          B[o++] = q;
        }
      }
      nb += tot;
      __syncthreads();
    }
    na = nb;
    int* t = A;
    A = B;
    B = t;
    __syncthreads();
  }
}

// First appearance of each label in scan order (:218-224).
__global__ void k_label_minidx(const int32_t* __restrict__ labels, long long n,
                               int* __restrict__ minidx) {
  for (long long p0 = (long long)blockIdx.x * blockDim.x; p0 < n;
       p0 += (long long)gridDim.x * blockDim.x) {
    const long long p = p0 + threadIdx.x;
    const int l = p < n ? labels[p] : -1;
    // lanes of a warp sharing a label: only the lowest index competes
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, l);
    if (l >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMin(&minidx[l], int(p));
  }
}

// First-appearance flag of pixel p: the label's minimum raster index is p.
struct FirstFlagIn {
  const int32_t* labels;
  const int* minidx;
  __device__ __forceinline__ void load8(long long base, long long n, int (&f)[8]) const {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      f[k] = base + k < n ? (minidx[labels[base + k]] == int(base + k) ? 1 : 0) : 0;
  }
};

__global__ void k_relabel(int32_t* __restrict__ labels, const int* __restrict__ minidx,
                          const int* __restrict__ rank, long long n) {
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 + 3 < n) {
    const int4 l = *reinterpret_cast<const int4*>(labels + p0);
    *reinterpret_cast<int4*>(labels + p0) =
        make_int4(rank[minidx[l.x]] + 1, rank[minidx[l.y]] + 1, rank[minidx[l.z]] + 1,
                  rank[minidx[l.w]] + 1);
    return;
  }
  for (long long p = p0; p < min(n, p0 + 4); ++p) labels[p] = rank[minidx[labels[p]]] + 1;
}


__global__ void k_fill_int(int* p, int v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_centers_out(Centers c, const CenterSums s, const int* __restrict__ count,
                              int K, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  if (k < *count) {
    out[3 * k] = c.cu[k];
    out[3 * k + 1] = c.cv[k];
    out[3 * k + 2] = c.val[k];
  }
}

// pool_superpixels tail: D3(p) = float(sum / n) of its label or invalid.
// Pooled value per label (pool_superpixels, segmentation.cpp:236-246), once per label.
__global__ void k_pool_values(CenterSums s, int max_label, float* __restrict__ val,
                              const int* __restrict__ nvalid = nullptr) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l > max_label) return;
  const int c = nvalid ? nvalid[l] : s.n[l];
  val[l] = c > 0 ? float(fixed_to_double(acc_value(s.sx[l])) / double(c)) : kInvalid;
}

__global__ void k_pool_write(const int32_t* __restrict__ labels, const float* __restrict__ val,
                             long long n, int max_label, float* __restrict__ d3) {
  auto pv = [&](int l) { return (l >= 0 && l <= max_label) ? val[l] : kInvalid; };
  const long long p0 = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 + 3 < n && (reinterpret_cast<uintptr_t>(d3) & 15u) == 0 &&
      (reinterpret_cast<uintptr_t>(labels) & 15u) == 0) {
    const int4 l = *reinterpret_cast<const int4*>(labels + p0);
    *reinterpret_cast<float4*>(d3 + p0) = make_float4(pv(l.x), pv(l.y), pv(l.z), pv(l.w));
    return;
  }
  for (long long p = p0; p < min(n, p0 + 4); ++p) d3[p] = pv(labels[p]);
}

}  // namespace

static void scan_flags(rpd_ctx* ctx, const int* flags, int* pos, long long n, const char*) {
  scan_exclusive_i32(ctx, flags, pos, n);
}

SlicOut slic_dev(rpd_ctx* ctx, const float* d2, int h, int w, int p, double m, int iterations,
                 float* d3) {
  if (p < 4) throw InvalidArg("slic: p must be >= 4");
  if ((long long)p > (long long)w * h) throw InvalidArg("slic: p exceeds pixel count");
  // 32-bit pixel indices, also for the rows of a ragged last tile
  if ((long long)(w + kTileU) * (h + kTileVLarge) >= (1ll << 31))
    throw InvalidArg("slic: more than 2^31 - 1 pixels");
  cudaStream_t st = ctx->stream;
  const long long n = (long long)h * w;
  const int gblocks = int(std::max<long long>(1, std::min<long long>((n + 255) / 256,
                                                                      ctx->sm_count * 16)));
  const dim3 rowgrid(cdiv(w, 128), h);
  // host-side scalars exactly as segmentation.cpp:178-186 (glibc on the host)
  const double S = std::sqrt(double(w) * h / p);
  const int nu = std::max(1, int(std::lround(std::sqrt(double(p) * w / h))));
  const int nv = std::max(1, int(std::lround(double(p) / nu)));
  const int K = nu * nv;
  const double su = double(w) / nu, sv = double(h) / nv;
  const int win = int(std::ceil(S));
  const double sw = m * m / (S * S);
  const int B = std::max(win, 1);
  const int nbx = cdiv(w, B), nby = cdiv(h, B);
  const int nb = nbx * nby;

  float* vals = ctx->ws.get<float>("slic_vals", n);
  int32_t* labels = ctx->ws.get<int32_t>("slic_labels", n);
  Centers c{ctx->ws.get<double>("slic_cu", K), ctx->ws.get<double>("slic_cv", K),
            ctx->ws.get<double>("slic_val", K), ctx->ws.get<int>("slic_icu", K),
            ctx->ws.get<int>("slic_icv", K)};
  CenterSums s{ctx->ws.get<int>("slic_n", K + 1), ctx->ws.get<long long>("slic_su", K + 1),
               ctx->ws.get<long long>("slic_sv", K + 1), ctx->ws.get<AccSum>("slic_sx", K + 1)};
  int* gridbuf = ctx->ws.get<int>("slic_grid_counts", 2 * size_t(nb) + 2);
  CenterGrid grid{B, nbx, nby, {gridbuf, gridbuf + nb}, {gridbuf + 2 * nb, gridbuf + 2 * nb + 1},
                  ctx->ws.get<CRec>("slic_recs", size_t(nb) * kBucketCap)};
  int* orphan_list = ctx->ws.get<int>("slic_orphans", n);
  int* orphan_count = ctx->ws.get<int>("slic_orphan_count", 3);
  int* inexact = orphan_count + 1;
  unsigned* orph_done = reinterpret_cast<unsigned*>(orphan_count + 2);
  const Orphans orph{orphan_list, orphan_count, vals, labels, w, inexact, orph_done};

  k_values_or_zero<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(d2, n, vals);
  RPD_LAUNCH_CHECK();
  k_seeds<<<cdiv(K, 128), 128, 0, st>>>(vals, h, w, nu, nv, su, sv, c);
  RPD_LAUNCH_CHECK();
  k_zero_sums<<<cdiv(K + 1, 256), 256, 0, st>>>(s, K + 1);
  RPD_LAUNCH_CHECK();
  RPD_CK(cudaMemsetAsync(orphan_count, 0, 3 * sizeof(int), st));
  // round 0's bucket counts and overflow flag start at zero
  RPD_CK(cudaMemsetAsync(gridbuf, 0, sizeof(int) * nb, st));
  RPD_CK(cudaMemsetAsync(grid.ovf[0], 0, sizeof(int), st));

  AssignArgs aa{vals, h, w, K, c, nullptr, nullptr, grid.rec, B, nbx, nby, win, sw, labels,
                orphan_list, orphan_count, inexact,
                debug_knob("RPD_SLIC_FORCE_WALK") != nullptr ? 1 : 0, 0u, nullptr, nullptr};
  // tile height: the large tile when it still gives every SM several CTAs
  bool large_tiles = cdiv(w, kTileU) * cdiv(h, kTileVLarge) >= 3 * ctx->sm_count;
  if (const char* e = debug_knob("RPD_SLIC_LARGE_TILES")) large_tiles = std::atoi(e) != 0;  // tests
  const int kTileV = large_tiles ? kTileVLarge : kTileVSmall;
  if (B >= 2 && w + win + kTileU < 65536 && h + win + kTileV < 65536)
    aa.b_magic = uint32_t((1ull << 32) / unsigned(B) + 1ull);
  const dim3 tgrid(cdiv(w, kTileU), cdiv(h, kTileV));
  const int cblocks = cdiv(std::max(K, nb), 256);
#ifndef RPD_SLIC_INCREMENTAL
// 0: every round assigns and sums every pixel; 1: persistent sums (changed
// pixels only) and clean-tile skipping; 2: persistent sums without skipping
#define RPD_SLIC_INCREMENTAL 2
#endif
  int inc_mode = RPD_SLIC_INCREMENTAL;
  if (const char* e = debug_knob("RPD_SLIC_INCREMENTAL")) inc_mode = std::atoi(e);
  const bool incremental = inc_mode != 0, skip = inc_mode == 1;
  TileDirty td{{nullptr, nullptr}, int(tgrid.x), int(tgrid.y), kTileU, kTileV, w, h, win, nullptr};
  if (skip) {
    const size_t ntiles = size_t(tgrid.x) * tgrid.y;
    int* dirty = ctx->ws.get<int>("slic_tile_dirty", 2 * (ntiles + 1));
    td.flags[0] = dirty;
    td.flags[1] = dirty + ntiles + 1;
    // round 1 marks buffer 1 (cleared by round 0's centre kernel); buffer 0 is
    // cleared by round 1's
    unsigned long long* tiles = ctx->ws.get<unsigned long long>("slic_tile_counts", 4);
    if (tiles != ctx->slic_tiles) {
      RPD_CK(cudaMemsetAsync(tiles, 0, 4 * sizeof(unsigned long long), st));
      ctx->slic_tiles = tiles;
    }
    aa.tiles = tiles;
    td.moved_dbg = tiles + 2;
  }
  int round = 0;
  // One round = centre grid (finalising the previous round's sums first) +
  // assignment that accumulates the sums the next round needs.
  auto assign = [&](bool finalize, bool sums) {
    const int cur = round & 1;
    const bool first = round == 0;
    ++round;
    // incremental: the sums persist until the last round's centre step
    const int fin = !finalize ? 0 : (incremental && sums ? 1 : 2);
    k_centers<<<cblocks, 256, 0, st>>>(c, K, s, fin, grid, cur, orph, td);
    RPD_LAUNCH_CHECK();
    aa.bcount = grid.count[cur];
    aa.ovf = grid.ovf[cur];
    aa.dirty = td.flags[cur];
    auto launch = [&](auto tv) {
      constexpr int TV = decltype(tv)::value;
      if (skip && !first) {
        if (sums)
          k_assign_tile<2, true, TV><<<tgrid, kAssignThreads, 0, st>>>(aa, s);
        else
          k_assign_tile<0, true, TV><<<tgrid, kAssignThreads, 0, st>>>(aa, s);
      } else if (incremental && !first && sums) {
        k_assign_tile<2, false, TV><<<tgrid, kAssignThreads, 0, st>>>(aa, s);
      } else if (sums) {
        k_assign_tile<1, false, TV><<<tgrid, kAssignThreads, 0, st>>>(aa, s);
      } else {
        k_assign_tile<0, false, TV><<<tgrid, kAssignThreads, 0, st>>>(aa, s);
      }
    };
    if (large_tiles)
      launch(std::integral_constant<int, kTileVLarge>{});
    else
      launch(std::integral_constant<int, kTileVSmall>{});
    RPD_LAUNCH_CHECK();
    if (!sums) {  // the last round: no k_centers follows to take its orphans
      k_assign_fallback<<<ctx->sm_count, 256, 0, st>>>(w, c, K, labels, orphan_list, orphan_count);
      RPD_LAUNCH_CHECK();
    }
  };
  auto update = [&]() {
    k_label_sums<<<gblocks, 256, 0, st>>>(vals, labels, h, w, K, false, true, s, inexact);
    RPD_LAUNCH_CHECK();
    k_center_finalize<<<cdiv(K, 256), 256, 0, st>>>(s, c, K);
    RPD_LAUNCH_CHECK();
  };
  assign(false, iterations > 0);
  for (int it = 0; it < iterations; ++it) assign(true, it + 1 < iterations);

  // enforce_connectivity
  int* parent = ctx->ws.get<int>("slic_parent", n);
  int* psize = ctx->ws.get<int>("slic_psize", n);
  unsigned long long* best = ctx->ws.get<unsigned long long>("slic_best", K + 1);
  int* claim = ctx->ws.get<int>("slic_claim", n);
  int* flags = ctx->ws.get<int>("slic_flags", n);
  int* pos = ctx->ws.get<int>("slic_pos", n);
  int* qa = ctx->ws.get<int>("slic_qa", n);
  int* qb = ctx->ws.get<int>("slic_qb", n);
  int* n0 = ctx->ws.get<int>("slic_n0", 1);
  uf_label(SameLabel{labels}, h, w, 1, parent, ctx->sm_count, st);
  RPD_CK(cudaMemsetAsync(psize, 0, sizeof(int) * n, st));
  RPD_CK(cudaMemsetAsync(best, 0, sizeof(unsigned long long) * (K + 1), st));
  k_piece_sizes<<<gblocks, 256, 0, st>>>(parent, n, psize);
  RPD_LAUNCH_CHECK();
  k_main_piece<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(parent, labels, psize, n, best);
  RPD_LAUNCH_CHECK();
  k_orphans<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(parent, labels, best, n, claim);
  RPD_LAUNCH_CHECK();
  RPD_CK(cudaMemsetAsync(flags, 0, sizeof(int) * n, st));
  k_frontier_flags<<<rowgrid, 128, 0, st>>>(labels, h, w, flags);
  RPD_LAUNCH_CHECK();
  scan_flags(ctx, flags, pos, n, "front");
  k_scatter_flagged<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(flags, pos, n, qa, n0);
  RPD_LAUNCH_CHECK();
  k_bfs<<<1, kBfsThreads, 0, st>>>(labels, h, w, claim, qa, qb, n0);
  RPD_LAUNCH_CHECK();

  // compaction by first appearance
  int* minidx = ctx->ws.get<int>("slic_minidx", K + 1);
  int* count = ctx->ws.get<int>("slic_count", 1);
  k_fill_int<<<cdiv(K + 1, 256), 256, 0, st>>>(minidx, 0x7FFFFFFF, K + 1);
  RPD_LAUNCH_CHECK();
  k_label_minidx<<<gblocks, 256, 0, st>>>(labels, n, minidx);
  RPD_LAUNCH_CHECK();
  // first-appearance flags evaluated inside the scan; its total is the count
  scan_exclusive(ctx, FirstFlagIn{labels, minidx}, pos, n, count);
  k_relabel<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(labels, minidx, pos, n);
  RPD_LAUNCH_CHECK();
  // final update_centers over the compacted labels (centres start at zero)
  RPD_CK(cudaMemsetAsync(c.cu, 0, sizeof(double) * K, st));
  RPD_CK(cudaMemsetAsync(c.cv, 0, sizeof(double) * K, st));
  RPD_CK(cudaMemsetAsync(c.val, 0, sizeof(double) * K, st));
  if (d3) {
    // one label pass for update_centers and pool_superpixels: the same value
    // sums (invalid D2 adds 0 to both), the pooled mean over the valid count
    int* nvalid = ctx->ws.get<int>("slic_nvalid", K + 1);
    RPD_CK(cudaMemsetAsync(nvalid, 0, sizeof(int) * (K + 1), st));
    k_label_sums<<<gblocks, 256, 0, st>>>(d2, labels, h, w, K, false, true, s, inexact, nvalid);
    RPD_LAUNCH_CHECK();
    float* pval = ctx->ws.get<float>("pool_val", K + 1);
    k_pool_values<<<cdiv(K + 1, 256), 256, 0, st>>>(s, K, pval, nvalid);
    RPD_LAUNCH_CHECK();
    k_pool_write<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(labels, pval, n, K, d3);
    RPD_LAUNCH_CHECK();
    k_center_finalize<<<cdiv(K, 256), 256, 0, st>>>(s, c, K);
    RPD_LAUNCH_CHECK();
  } else {
    update();
  }
  double* cout = ctx->ws.get<double>("slic_centers_out", 3 * size_t(K));
  k_centers_out<<<cdiv(K, 128), 128, 0, st>>>(c, s, count, K, cout);
  RPD_LAUNCH_CHECK();
  SlicOut out;
  out.labels = labels;
  out.centers = cout;
  out.count = count;
  out.spacing = S;
  out.k_seeds = K;
  (void)kDU;
  (void)kDV;
  return out;
}

void pool_superpixels_dev(rpd_ctx* ctx, const float* d2, const int32_t* labels, int h, int w,
                          int max_count, float* d3) {
  cudaStream_t st = ctx->stream;
  const long long n = (long long)h * w;
  const int gblocks = int(std::max<long long>(1, std::min<long long>((n + 255) / 256,
                                                                      ctx->sm_count * 16)));
  CenterSums s{ctx->ws.get<int>("pool_n", max_count + 1), nullptr, nullptr,
               ctx->ws.get<AccSum>("pool_sx", max_count + 1)};
  int* inexact = ctx->ws.get<int>("pool_inexact", 1);
  RPD_CK(cudaMemsetAsync(s.n, 0, sizeof(int) * (max_count + 1), st));
  RPD_CK(cudaMemsetAsync(s.sx, 0, sizeof(AccSum) * (max_count + 1), st));
  k_label_sums<<<gblocks, 256, 0, st>>>(d2, labels, h, w, max_count, true, false, s, inexact);
  RPD_LAUNCH_CHECK();
  float* val = ctx->ws.get<float>("pool_val", max_count + 1);
  k_pool_values<<<cdiv(max_count + 1, 256), 256, 0, st>>>(s, max_count, val);
  RPD_LAUNCH_CHECK();
  k_pool_write<<<std::max(1, cdiv(n, 1024)), 256, 0, st>>>(labels, val, n, max_count, d3);
  RPD_LAUNCH_CHECK();
}

}  // namespace rpdg
