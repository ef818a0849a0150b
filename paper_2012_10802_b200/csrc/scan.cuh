// scan.cuh — single-pass exclusive prefix sum of per-element int flags
// (ordered stream compaction: sample_observations, the SLIC frontier and
// first-appearance compaction, the CCL root numbering).  One launch per scan:
// tiles of 2048 elements take their index from a ticket in start order and
// chain their prefixes by decoupled look-back (one warp reads 32
// predecessors at a time), so no tile waits on one that has not started.
// Descriptors carry the launch's tag (an epoch the last tile advances), so
// they never need clearing between launches or graph replays.  The flags come
// from an input functor — an array, or a predicate evaluated in place — and
// the last tile can store the total.
#pragma once

#include "common.cuh"

namespace rpdg {

// An input functor fills the flags of elements base .. base+7 (0 past n):
//   __device__ void load8(long long base, long long n, int (&v)[8]) const;
// flags from an int array (16-byte vector loads when aligned)
struct ScanArrayIn {
  const int* a;
  __device__ __forceinline__ void load8(long long base, long long n, int (&v)[8]) const {
    if (base + 8 <= n && (reinterpret_cast<uintptr_t>(a + base) & 15u) == 0) {
      const int4 x = *reinterpret_cast<const int4*>(a + base);
      const int4 y = *reinterpret_cast<const int4*>(a + base + 4);
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
      v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
      return;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = base + k < n ? a[base + k] : 0;
  }
};

namespace scan_detail {

constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kAggregate = 1ull, kInclusive = 2ull;

__device__ __forceinline__ unsigned long long pack_desc(unsigned tag, unsigned long long status,
                                                        unsigned long long value) {
  return (unsigned long long)tag << 32 | status << 30 | value;
}

template <class In>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_exclusive(const In in, int* __restrict__ out, long long n,
                     unsigned long long* __restrict__ desc, unsigned* __restrict__ ctl,
                     int* __restrict__ total_out) {
  __shared__ unsigned s_tile, s_tag;
  __shared__ int s_warp[kScanThreads / 32];
  __shared__ int s_prefix;
  if (threadIdx.x == 0) {
    // the epoch is read BEFORE the ticket: the last ticket's holder advances
    // it only after every tile has taken one
    const unsigned e = *reinterpret_cast<volatile unsigned*>(ctl + 1);
    __threadfence();
    s_tile = atomicAdd(ctl, 1u);
    s_tag = e + 1u == 0u ? 1u : e + 1u;
  }
  __syncthreads();
  const unsigned tile = s_tile, tag = s_tag;
  const long long base = (long long)tile * kScanTile + (long long)threadIdx.x * kScanItems;
  int v[kScanItems];
  static_assert(kScanItems == 8, "load8");
  in.load8(base, n, v);
  int run = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int x = v[k];
    v[k] = run;  // exclusive within the thread
    run += x;
  }
  // warp inclusive scan of the thread totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = run;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xFFFFFFFFu, inc, off);
    if (lane >= off) inc += o;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  int wpre = 0, total = 0;
#pragma unroll
  for (int q = 0; q < kScanThreads / 32; ++q) {
    const int t = s_warp[q];
    wpre += q < warp ? t : 0;
    total += t;
  }
  if (warp == 0) {
    // decoupled look-back, one warp: lane k reads predecessor tile - 1 - k;
    // the nearest inclusive prefix ends the walk, aggregates before it add up
    if (lane == 0)
      atomicExch(desc + tile, pack_desc(tag, tile == 0 ? kInclusive : kAggregate,
                                        (unsigned long long)total));
    int prefix = 0;
    long long j = (long long)tile - 1 - lane;
    while (tile > 0) {
      unsigned long long d = pack_desc(tag, kInclusive, 0ull);  // before tile 0: prefix 0
      if (j >= 0) {
        do {
          d = *reinterpret_cast<volatile unsigned long long*>(desc + j);
        } while (unsigned(d >> 32) != tag);  // started earlier: publishes soon
      }
      const unsigned incl = __ballot_sync(0xFFFFFFFFu, ((d >> 30) & 3ull) == kInclusive);
      const int stop = incl ? __ffs(incl) - 1 : 31;
      int val = lane <= stop ? int(d & 0x3FFFFFFFull) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, o);
      prefix += val;
      if (incl) break;
      j -= 32;
    }
    if (lane == 0) {
      if (tile > 0) {
        __threadfence();
        atomicExch(desc + tile, pack_desc(tag, kInclusive, (unsigned long long)(prefix + total)));
      }
      s_prefix = prefix;
      if (tile == gridDim.x - 1) {  // every tile has its ticket and has read the epoch
        if (total_out) *total_out = prefix + total;
        ctl[0] = 0u;
        *reinterpret_cast<volatile unsigned*>(ctl + 1) = tag;
      }
    }
  }
  __syncthreads();
  const int off = s_prefix + wpre + inc - run;
  if (base + kScanItems <= n && (reinterpret_cast<uintptr_t>(out + base) & 15u) == 0) {
    *reinterpret_cast<int4*>(out + base) = make_int4(off + v[0], off + v[1], off + v[2], off + v[3]);
    *reinterpret_cast<int4*>(out + base + 4) =
        make_int4(off + v[4], off + v[5], off + v[6], off + v[7]);
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (base + k < n) out[base + k] = off + v[k];
  }
}

}  // namespace scan_detail

// Workspace of one scan launch (descriptors zeroed once per allocation).
struct ScanState {
  unsigned long long* desc;
  unsigned* ctl;
  unsigned tiles;
};
ScanState scan_state(rpd_ctx* ctx, long long n);

// out[i] = in(0) + ... + in(i-1) on ctx->stream in one launch; *total (device,
// optional) = the sum of all n flags.
template <class In>
void scan_exclusive(rpd_ctx* ctx, const In& in, int* out, long long n, int* total = nullptr) {
  if (n <= 0) return;
  const ScanState s = scan_state(ctx, n);
  scan_detail::k_scan_exclusive<In><<<s.tiles, scan_detail::kScanThreads, 0, ctx->stream>>>(
      in, out, n, s.desc, s.ctl, total);
  RPD_LAUNCH_CHECK();
}

}  // namespace rpdg
