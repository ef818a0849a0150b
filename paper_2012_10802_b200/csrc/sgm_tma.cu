// sgm_tma.cu — TMA-staged SGM path aggregation (aggregate_costs, sgm.cpp:70-110)
// for sm_100a.
//
// One CTA owns NC = 32 scan chains of one (volume, direction) job; each chain
// is handled by G lanes, each lane holding WPL u8-cost words (2*WPL packed
// u16x2 level pairs) of the chain's current pixel in registers.  An elected
// thread streams the raw cost tiles of the next R steps into a DEPTH-deep
// shared-memory ring with cp.async.bulk.tensor (completion on mbarriers), and
// writes the per-path u8 results back with TMA stores from an output tile
// (RPD_AGG_OUTDEPTH deep), so the compute threads only touch shared memory.
//
// Chains: horizontal = image rows, vertical = columns, diagonal = the W+H-1
// non-wrapping diagonals u = k + du*s; tiles that stick out of the image are
// zero-filled by the TMA load and dropped by the TMA store.
//
// Recurrence per step (exact integers, sgm.cpp:95-104), per u16x2 pair:
//   best = min(prev, prev[d-1]+P1, prev[d+1]+P1, min(prev)+P2)   (2x VIADDMNMX + VIMNMX)
//   cur  = raw + best - min(prev)                                   (IADD3, no carry)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "sgm.cuh"

// TileAddr::kStride is unused by the chunked layouts
#pragma nv_diag_suppress 177

namespace rpdg {

namespace {

#ifndef RPD_AGG_NC1
#define RPD_AGG_NC1 32  // chains (= threads) per CTA of the one-lane-per-chain kernels
#endif
// chains per CTA: one warp of chains; G == 1 kernels may take several warps
__host__ __device__ constexpr int nc_of(int G) { return G == 1 ? RPD_AGG_NC1 : 32; }
#ifndef RPD_AGG_DEPTH
#define RPD_AGG_DEPTH 2
#endif
constexpr int kDepth = RPD_AGG_DEPTH;  // input ring depth (stages)
#ifndef RPD_AGG_RBASE
#define RPD_AGG_RBASE 4      // steps per stage for <= 32 words per pixel
#endif
#ifndef RPD_AGG_UNROLL
#define RPD_AGG_UNROLL 2     // unrolled steps of the inner loop, multi-lane chains (code size vs ILP)
#endif
#ifndef RPD_AGG_UNROLL_G1
#define RPD_AGG_UNROLL_G1 2  // the same, one-lane chains
#endif
#ifndef RPD_AGG_REC
// recurrence form: 0 = 2x add-min + min, 1 = min3 + add-min, 2 = min3 + add + min3,
// 3 = normalised state (n = L - min L, see chain_step_norm)
#define RPD_AGG_REC 3
#endif
#ifndef RPD_AGG_OUTDEPTH
#define RPD_AGG_OUTDEPTH 1  // output tiles in flight (TMA stores not yet read); 1: less smem, +1 % concurrent
#endif
constexpr int kOutDepth = RPD_AGG_OUTDEPTH;
constexpr int kRBase = RPD_AGG_RBASE;
#ifndef RPD_AGG_RBASE_G1
#define RPD_AGG_RBASE_G1 4  // steps per stage of the one-lane-per-chain kernels
#endif
constexpr int kRBaseG1 = RPD_AGG_RBASE_G1;
constexpr int kStepUnroll = RPD_AGG_UNROLL, kStepUnrollG1 = RPD_AGG_UNROLL_G1;
constexpr uint32_t kInf2 = 0x7FFF7FFFu;

enum JobType : int { kHoriz = 0, kVert = 1, kDiag = 2 };

struct TmaJob {
  int vol;      // 0 left-reference cost, 1 right-reference cost
  int path;     // output buffer index
  int du, dv;
  int type;
  int kmin;     // diagonal: first chain index (u = k + du*s)
  int nchains;
  int block0;
  int nseg;     // H / V: CTAs (segments) per chain group along the scan (1 = unsplit)
  int slot0;    // first segment-boundary slot of this job in the exchange area
};

struct TmaArgs {
  CUtensorMap cost_h, cost_vf, cost_vl, cost_df, cost_dl;
  CUtensorMap path_h, path_vf, path_vl, path_df, path_dl;
  TmaJob job[16];
  int njobs;
  int h, w;
  uint32_t p1x2, p2x2;
  uint32_t one;  // 1 at run time: keeps `x * one + y` an IMAD (FMA pipe) instead of an ALU add
  uint8_t* path_base;  // diagonal jobs store directly
  size_t pitch, vol_bytes;
  int dbg;  // debugging early-exit level (RPD_TMA_DBG), 0 in production
  // Segmented chains (see agg_body): boundary states and flags, CTA tickets.
  uint32_t* seg_state;  // per boundary slot: true state, then the warm-up guess
  uint32_t* seg_flag;   // per boundary slot: 1 = predecessor's true state published
  unsigned* ticket;     // dynamic CTA order (start order = logical block index)
  unsigned long long* reruns;  // count of recomputed segments (rpd_stats)
  int seg_words;        // words of one state image (NPAIR * THREADS)
  int warm_stages;      // warm-up stages of a segment before its first stored stage
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_addr(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}

#ifndef RPD_AGG_L2_HINTS
// L2 eviction hints of the aggregation's bulk copies: bit 0 = cost tiles are
// loaded evict_last (each is read by all 2P jobs of the launch), bit 1 = path
// tiles are stored evict_first (written once, read once by the WTA much later),
// bit 2 = the diagonal jobs' direct stores are streaming stores
#define RPD_AGG_L2_HINTS 1
#endif

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
#if RPD_AGG_L2_HINTS & 1
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar)),
      "l"(l2_policy_evict_last())
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar))
      : "memory");
#endif
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int x, int y, int z,
                                             const void* src) {
#if RPD_AGG_L2_HINTS & 2
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(x), "r"(y), "r"(z), "r"(smem_addr(src)), "l"(l2_policy_evict_first())
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(x), "r"(y), "r"(z), "r"(smem_addr(src))
      : "memory");
#endif
}

__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;"); }
template <int N>
__device__ __forceinline__ void tma_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tma_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int NPL>
__device__ __forceinline__ uint32_t min_pairs(const uint32_t (&x)[NPL]) {
  uint32_t t[NPL];
#pragma unroll
  for (int k = 0; k < NPL; ++k) t[k] = x[k];
#pragma unroll
  for (int width = 1; width < NPL; width *= 2)
#pragma unroll
    for (int i = 0; i + width < NPL; i += 2 * width) t[i] = __vminu2(t[i], t[i + width]);
  return t[0];
}

// Compile-time tile geometry.
template <int WPL, int G>
struct Geo {
  static constexpr int WPP = WPL * G;                  // words per pixel
  static constexpr int RB = G == 1 ? kRBaseG1 : kRBase;
  static constexpr int R = WPP <= 32 ? RB : (WPP <= 64 ? (RB + 1) / 2 : 1);
  static constexpr int NC = nc_of(G);                  // chains per CTA
  static constexpr int ROW = NC * WPP;                 // words of one step (vert / diag)
  static constexpr int CWF = ROW < 256 ? ROW : 256;    // full chunk width
  static constexpr int NCH = (ROW + 255) / 256;        // chunks per row
  static constexpr int CWL = ROW - (NCH - 1) * 256;    // last chunk width
  static constexpr int STAGE = R * ROW;                // words per output stage
  // Diagonal rows start at arbitrary columns but TMA box origins must be
  // 16-byte aligned: each row is loaded from the aligned word below it with
  // 32 extra words (keeps 128-byte aligned smem rows), read with a shift.
  static constexpr int DROW = ROW + 32;
  static constexpr int DNCH = (DROW + 255) / 256;
  static constexpr int DCWL = DROW - (DNCH - 1) * 256;
  static constexpr int STAGE_IN = R * DROW;            // words per input stage
  static constexpr int THREADS = NC * G;
};

// Shared-memory word offsets of this thread's pixel words inside a tile.
// Unchunked layouts (the common case) reduce to base + q + rr*STRIDE with a
// compile-time STRIDE, so every access is an LDS/STS with an immediate offset.
template <int TYPE, int WPL, int G>
struct TileAddr {
  using GE = Geo<WPL, G>;
  static constexpr bool kChunked =
      (TYPE == kVert && GE::NCH > 1) || (TYPE == kDiag && GE::DNCH > 1);
  static constexpr int kStride = TYPE == kHoriz ? GE::WPP : (TYPE == kVert ? GE::ROW : GE::DROW);
  // word-offset shifts of diagonal rows are 0 whenever a pixel is a whole
  // number of 16-byte groups: the chunked offsets are then step-invariant
  static constexpr bool kNoShift = TYPE != kDiag || GE::WPP % 4 == 0;
  static constexpr bool kPre = kChunked && kNoShift;
  int base;
  int off[kPre ? WPL : 1], str[kPre ? WPL : 1];
  __device__ __forceinline__ void init(int t, int g) {
    base = (TYPE == kHoriz) ? t * (GE::R * GE::WPP) + g * WPL : t * GE::WPP + g * WPL;
    if constexpr (kPre) {
      const int last = TYPE == kVert ? GE::NCH - 1 : GE::DNCH - 1;
      const int cwl = TYPE == kVert ? GE::CWL : GE::DCWL;
#pragma unroll
      for (int q = 0; q < WPL; ++q) {
        const int wd = base + q, ch = wd >> 8;
        off[q] = ch * (256 * GE::R) + (wd & 255);
        str[q] = ch == last ? cwl : 256;
      }
    }
  }
  __device__ __forceinline__ int at(int q, int rr, int shift) const {
    if constexpr (!kChunked) {
      return base + shift + q + rr * kStride;
    } else if constexpr (kPre) {
      return off[q] + rr * str[q];
    } else {
      const int wd = base + shift + q;
      const int ch = wd >> 8;
      const int last = TYPE == kVert ? GE::NCH - 1 : GE::DNCH - 1;
      const int cwl = TYPE == kVert ? GE::CWL : GE::DCWL;
      return ch * (256 * GE::R) + rr * (ch == last ? cwl : 256) + (wd & 255);
    }
  }
};

template <int NP>
__device__ __forceinline__ uint32_t min_pairs3(const uint32_t (&x)[NP]) {
  // balanced tree of 3-input DPX mins
  uint32_t t[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) t[k] = x[k];
  int n = NP;
#pragma unroll
  for (int it = 0; it < 6; ++it) {
    if (n <= 1) break;
    int m = 0;
#pragma unroll
    for (int i = 0; i < NP; i += 3) {
      if (i >= n) break;
      if (i + 2 < n)
        t[m] = __vimin3_u16x2(t[i], t[i + 1], t[i + 2]);
      else if (i + 1 < n)
        t[m] = __vminu2(t[i], t[i + 1]);
      else
        t[m] = t[i];
      ++m;
    }
    n = m;
  }
  return t[0];
}

// Per-chain recurrence state.  A chain (re)starts with prev = INF and
// min = INF: then best = INF and cur = raw + INF - INF = raw exactly, so the
// "no predecessor" case needs no branch (sgm.cpp:89-92).
template <int NPAIR>
struct ChainState {
  uint32_t prev[NPAIR];
  uint32_t mnx2;
  __device__ __forceinline__ void reset() {
#if RPD_AGG_REC == 3
    // normalised state: n = 0 gives cur = raw + min(0, P1, P2) = raw exactly
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) prev[q] = 0u;
    mnx2 = 0u;
#else
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) prev[q] = kInf2;
    mnx2 = kInf2;
#endif
  }
};

__device__ __forceinline__ uint32_t imad_add(uint32_t x, uint32_t one, uint32_t y) {
  uint32_t r;  // x * one + y on the FMA pipe (one == 1 at run time)
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(y));
  return r;
}

// Normalised recurrence (RPD_AGG_REC 3).  With n(d) = L_prev(d) - min L_prev
// (>= 0, exact integers) sgm.cpp:95-104 reads
//   cur(d) = raw(d) + min(n(d), min(n(d-1), n(d+1), P2 - P1) + P1)
//   n'(d)  = cur(d) - min cur
// (= raw + min(L, L(d+-1) + P1, min L + P2) - min L).  Per u16x2 level pair:
// PRMT (n(d+1)), VIMNMX3, VIADDMNMX and the raw-byte PRMT on the ALU pipe,
// the two adds as IMADs on the FMA pipe (co-issued; tools/pipe_probe.cu).
// A chain (re)start is n = 0: cur = raw + min(0, P1, P2) = raw.  Padding
// levels (raw 0xFF) stay >= 255 - min and never win (L <= 255 - P1 + ...,
// sgm_fast_path_ok).
template <int WPL, int G, int NPAIR>
__device__ __forceinline__ void chain_step_norm(ChainState<NPAIR>& cs, const uint32_t (&w8)[WPL],
                                                uint32_t p1x2, uint32_t c21x2, uint32_t one,
                                                int g, unsigned gmask, uint32_t (&packed)[WPL]) {
  uint32_t lo_nb = kInf2, hi_nb = kInf2;
  if (G > 1) {
    const uint32_t up = __shfl_up_sync(gmask, cs.prev[NPAIR - 1], 1, G);
    const uint32_t dn = __shfl_down_sync(gmask, cs.prev[0], 1, G);
    if (g > 0) lo_nb = up;
    if (g < G - 1) hi_nb = dn;
  }
  uint32_t cur[NPAIR];
  uint32_t qprev = __byte_perm(lo_nb, cs.prev[0], 0x5432);
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    const uint32_t nxt = (q + 1 < NPAIR) ? cs.prev[q + 1] : hi_nb;
    const uint32_t qn = __byte_perm(cs.prev[q], nxt, 0x5432);  // n(d+1) of both halves
    const uint32_t a = __vimin3_u16x2(qprev, qn, c21x2);
    const uint32_t tt = __viaddmin_u16x2(a, p1x2, cs.prev[q]);
    const uint32_t raw = __byte_perm(w8[q / 2], 0u, (q & 1) ? 0x4342 : 0x4140);
    cur[q] = imad_add(tt, one, raw);
    qprev = qn;
  }
#pragma unroll
  for (int q = 0; q < WPL; ++q)
    packed[q] =
        __byte_perm(cur[2 * q], (2 * q + 1 < NPAIR) ? cur[2 * q + 1] : 0xFFFFFFFFu, 0x6420);
  const uint32_t m2 = min_pairs3<NPAIR>(cur);
  uint32_t m = min(m2 & 0xFFFFu, m2 >> 16);
  if (G > 1) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) m = min(m, __shfl_xor_sync(gmask, m, off, G));
  }
  const uint32_t negm = 0u - m * 0x10001u;  // per-half exact: cur >= m
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) cs.prev[q] = imad_add(cur[q], one, negm);
}

// One recurrence step on packed u16x2 level pairs; returns the packed u8
// words of the new costs in `packed` and updates the state.
template <int WPL, int G, int NPAIR>
__device__ __forceinline__ void chain_step(ChainState<NPAIR>& cs, const uint32_t (&w8)[WPL],
                                           uint32_t p1x2, uint32_t p2x2, int g, unsigned gmask,
                                           uint32_t (&packed)[WPL]) {
  uint32_t raw[NPAIR];
#pragma unroll
  for (int q = 0; q < WPL; ++q) {
    raw[2 * q] = __byte_perm(w8[q], 0u, 0x4140);
    if (2 * q + 1 < NPAIR) raw[2 * q + 1] = __byte_perm(w8[q], 0u, 0x4342);
  }
  uint32_t lo_nb = kInf2, hi_nb = kInf2;
  if (G > 1) {
    const uint32_t up = __shfl_up_sync(gmask, cs.prev[NPAIR - 1], 1, G);
    const uint32_t dn = __shfl_down_sync(gmask, cs.prev[0], 1, G);
    if (g > 0) lo_nb = up;
    if (g < G - 1) hi_nb = dn;
  }
  uint32_t cur[NPAIR];
  uint32_t qprev = __byte_perm(lo_nb, cs.prev[0], 0x5432);
#if RPD_AGG_REC == 0
  const uint32_t ceil2 = cs.mnx2 + p2x2;
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    const uint32_t nxt = (q + 1 < NPAIR) ? cs.prev[q + 1] : hi_nb;
    const uint32_t qn = __byte_perm(cs.prev[q], nxt, 0x5432);  // (prev[d+1] of both halves)
    uint32_t tt = __viaddmin_u16x2(qprev, p1x2, cs.prev[q]);
    tt = __viaddmin_u16x2(qn, p1x2, tt);
    tt = __vminu2(tt, ceil2);
    cur[q] = raw[q] + tt - cs.mnx2;  // per-half exact: tt >= min, no carry
    qprev = qn;
  }
#else
  // min(prev[d-1]+P1, prev[d+1]+P1, min+P2) = min(prev[d-1], prev[d+1], min+P2-P1) + P1
  // (P2 >= P1): one 3-input DPX min (half rate) instead of two fused add-mins
  // (quarter rate on sm_100, tools/dpx_probe.cu).
  const uint32_t ceilm = cs.mnx2 + (p2x2 - p1x2);
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    const uint32_t nxt = (q + 1 < NPAIR) ? cs.prev[q + 1] : hi_nb;
    const uint32_t qn = __byte_perm(cs.prev[q], nxt, 0x5432);  // (prev[d+1] of both halves)
    const uint32_t a = __vimin3_u16x2(qprev, qn, ceilm);
#if RPD_AGG_REC == 1
    const uint32_t tt = __viaddmin_u16x2(a, p1x2, cs.prev[q]);
#else
    const uint32_t ap = a + p1x2;
    const uint32_t tt = __vimin3_u16x2(ap, cs.prev[q], cs.prev[q]);
#endif
    cur[q] = raw[q] + tt - cs.mnx2;  // per-half exact: tt >= min, no carry
    qprev = qn;
  }
#endif
#pragma unroll
  for (int q = 0; q < WPL; ++q)
    packed[q] =
        __byte_perm(cur[2 * q], (2 * q + 1 < NPAIR) ? cur[2 * q + 1] : 0xFFFFFFFFu, 0x6420);
  const uint32_t m2 = min_pairs3<NPAIR>(cur);
  uint32_t m = min(m2 & 0xFFFFu, m2 >> 16);
  if (G > 1) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) m = min(m, __shfl_xor_sync(gmask, m, off, G));
  }
  cs.mnx2 = m * 0x10001u;
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) cs.prev[q] = cur[q];
}

// One job type, fully specialised.  NPAIR <= 2*WPL level pairs are computed
// per lane; a trailing all-padding pair (odd L with G == 1) is skipped.
template <int TYPE, int WPL, int G, int NPAIR>
__device__ __forceinline__ void agg_body(const TmaArgs& a, const TmaJob& J, int cta, int cta_seg,
                                         uint32_t* in_ring, uint32_t* out_ring, uint64_t* full) {
  using GE = Geo<WPL, G>;
  constexpr int R = GE::R;
  const int du = J.du, dv = J.dv;
  const int h = a.h, w = a.w;
  const int t = int(threadIdx.x) / G;  // chain within CTA
  const int g = int(threadIdx.x) % G;
  const unsigned gmask =
      G == 32 ? 0xFFFFFFFFu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));

  constexpr int kNC = GE::NC;
  const int c0 = cta * kNC;  // first chain of this CTA (row / column / diagonal offset)
  const int nsteps = TYPE == kHoriz ? w : h;
  // Steps are "virtual": horizontal / vertical tiles are aligned to multiples
  // of R from the image origin so that no TMA store box starts at a negative
  // coordinate (the hardware faults on those); a backward scan therefore
  // begins at virtual step T - N.  Diagonals use real steps.
  const bool backward = (TYPE == kHoriz) ? du < 0 : dv < 0;
  const int T = (nsteps + R - 1) / R * R;
  int s_begin = (TYPE != kDiag && backward) ? T - nsteps : 0;
  int s_end = s_begin + nsteps;
  int stage_base = 0;
  int kbase = 0;
  if (TYPE == kDiag) {
    kbase = J.kmin + c0;
    // u = k + du*s in [0, w) for some k in [kbase, kbase+NC)
    if (du > 0) {
      s_begin = max(0, -(kbase + kNC - 1));
      s_end = min(nsteps, w - kbase);
    } else {
      s_begin = max(0, kbase - (w - 1));
      s_end = min(nsteps, kbase + kNC);
    }
    stage_base = s_begin;
  }
  const int nstage = s_end > stage_base ? (s_end - stage_base + R - 1) / R : 0;
  const int zc = J.vol, zp = J.path;

  const CUtensorMap* cm_a = TYPE == kHoriz ? &a.cost_h : (TYPE == kVert ? &a.cost_vf : &a.cost_df);
  const CUtensorMap* cm_b = TYPE == kVert ? &a.cost_vl : &a.cost_dl;
  const CUtensorMap* pm_a = TYPE == kHoriz ? &a.path_h : &a.path_vf;
  const CUtensorMap* pm_b = &a.path_vl;

  // Issue the TMA loads (or, for H/V, the stores) of stage `st`.
  auto tile_ops = [&](int st, bool load, uint32_t* buf, uint64_t* bar) {
    const int s0 = stage_base + st * R;
    if (TYPE == kHoriz) {
      const int ucol = backward ? T - s0 - R : s0;  // R columns x NC rows
      if (load)
        tma_load_3d(buf, cm_a, ucol * GE::WPP, c0, zc, bar);
      else
        tma_store_3d(pm_a, ucol * GE::WPP, c0, zp, buf);
    } else if (TYPE == kVert) {
      const int vrow = backward ? T - s0 - R : s0;
#pragma unroll
      for (int ch = 0; ch < GE::NCH; ++ch) {
        const CUtensorMap* m = ch == GE::NCH - 1 ? (load ? cm_b : pm_b) : (load ? cm_a : pm_a);
        uint32_t* dst = buf + ch * (256 * R);
        const int x = c0 * GE::WPP + ch * 256;
        if (load)
          tma_load_3d(dst, m, x, vrow, zc, bar);
        else
          tma_store_3d(m, x, vrow, zp, dst);
      }
    } else if (load) {  // diagonal results are stored directly by the threads
      for (int r = 0; r < R; ++r) {
        const int s = s0 + r;
        if (s >= s_end) break;
        const int vrow = dv > 0 ? s : h - 1 - s;
        const int x0 = ((kbase + du * s) * GE::WPP) & ~3;  // floor to a 16-byte boundary
#pragma unroll
        for (int ch = 0; ch < GE::DNCH; ++ch) {
          const bool last = ch == GE::DNCH - 1;
          uint32_t* p = buf + ch * (256 * R) + r * (last ? GE::DCWL : 256);
          tma_load_3d(p, last ? cm_b : cm_a, x0 + ch * 256, vrow, zc, bar);
        }
      }
    }
  };
  auto stage_bytes = [&](int st) -> uint32_t {
    if (TYPE != kDiag) return uint32_t(GE::STAGE) * 4u;
    const int s0 = stage_base + st * R;
    const int rows = min(R, s_end - s0);
    return uint32_t(rows) * uint32_t(GE::DROW) * 4u;
  };

  TileAddr<TYPE, WPL, G> ad;
  ad.init(t, g);
  const uint32_t p1x2 = a.p1x2, p2x2 = a.p2x2, one = a.one;
  ChainState<NPAIR> cs;
  cs.reset();
  uint8_t* const pbase = a.path_base + size_t(zp) * a.vol_bytes + size_t(g * WPL) * 4;

  // Segmented chains (H / V jobs with J.nseg > 1).  The stages of a chain
  // group are cut into nseg ranges [m0, m1), one CTA each.  Segment j > 0
  // starts `warm_stages` before m0 from the restart state and stores nothing
  // there; the recurrence forgets its start state within a few dozen steps
  // on textured costs (BASELINE scenes: every chain within 64 steps at the
  // cut), so its state at m0 - 1 (the guess) normally equals the true one.
  // The outputs from m0 on depend only on that state and the raw costs, so
  // they are exact whenever the guess equals the true state, which segment
  // j - 1 publishes when it ends.  Segment j compares the two and, on any
  // difference in a valid chain, reruns [m0, m1) from the true state,
  // overwriting its outputs (uniform cost runs do not forget their start).
  int seg = 0, nseg = 1;
  if constexpr (TYPE != kDiag) {
    nseg = J.nseg;
    seg = cta_seg;
  }
  const int m0 = nseg > 1 ? int((long long)nstage * seg / nseg) : 0;
  const int m1 = nseg > 1 ? int((long long)nstage * (seg + 1) / nseg) : nstage;
  const int slot = J.slot0 + cta * (nseg - 1) + seg - 1;  // boundary (seg-1 | seg)
  const int tid = int(threadIdx.x);

  // diagonal results are stored by the threads: byte offset of this lane's
  // pixel of the current step, advanced by one (row, column) step at a time
  long long doff = 0, dstep = 0;
  if constexpr (TYPE == kDiag) {
    const int s = stage_base;
    doff = (long long)(dv > 0 ? s : h - 1 - s) * (long long)a.pitch +
           (long long)(kbase + du * s + t) * (GE::WPP * 4);
    dstep = (dv > 0 ? (long long)a.pitch : -(long long)a.pitch) + (long long)du * (GE::WPP * 4);
  }

  uint32_t seq = 0;  // stages consumed by this CTA (ring slot / mbarrier parity)
  int ra = max(0, m0 - a.warm_stages);
#pragma unroll 1
  for (int pass = 0;; ++pass) {
    const int rb = m1;
    if (threadIdx.x == 0) {
      for (int i = 0; i < kDepth && ra + i < rb; ++i) {
        const uint32_t sl = (seq + i) % kDepth;
        mbar_expect_tx(&full[sl], stage_bytes(ra + i));
        tile_ops(ra + i, true, in_ring + sl * GE::STAGE_IN, &full[sl]);
      }
    }
#pragma unroll 1
    for (int st = ra; st < rb; ++st, ++seq) {
      const uint32_t sl = seq % kDepth;
      mbar_wait(&full[sl], (seq / kDepth) & 1u);
      const uint32_t* inb = in_ring + sl * GE::STAGE_IN;
      uint32_t* outb = out_ring + (seq % kOutDepth) * GE::STAGE;
      const bool store = st >= m0;
      const int s0 = stage_base + st * R;
      // only the first tile of a backward H/V scan holds padding steps
      const bool check = TYPE != kDiag && s0 < s_begin;
#pragma unroll(G == 1 ? kStepUnrollG1 : kStepUnroll)
      for (int r = 0; r < R; ++r) {
        const int s = s0 + r;
        const int rr = (TYPE != kDiag && backward) ? R - 1 - r : r;
        int shift = 0, col = 0;
        if (TYPE == kDiag) {
          const int cbase = kbase + du * s;
          shift = (cbase * GE::WPP) & 3;
          col = cbase + t;
          const bool has_pred = s > 0 && unsigned(col - du) < unsigned(w);
          if (!has_pred) cs.reset();  // chain (re)enters the image
        }
        uint32_t w8[WPL];
#pragma unroll
        for (int q = 0; q < WPL; ++q) w8[q] = inb[ad.at(q, rr, shift)];
        uint32_t packed[WPL];
        if (check && s < s_begin) continue;  // padding step (outside the image): state stays
#if RPD_AGG_REC == 3
        chain_step_norm<WPL, G, NPAIR>(cs, w8, p1x2, p2x2 - p1x2, one, g, gmask, packed);
#else
        chain_step<WPL, G, NPAIR>(cs, w8, p1x2, p2x2, g, gmask, packed);
#endif
        if (TYPE == kDiag) {
          if (unsigned(col) < unsigned(w) && s < s_end) {
            uint32_t* dst = reinterpret_cast<uint32_t*>(pbase + doff);
#pragma unroll
            for (int q = 0; q < WPL; ++q) {
#if RPD_AGG_L2_HINTS & 4
              __stcs(dst + q, packed[q]);  // streaming: read once by the WTA, much later
#else
              dst[q] = packed[q];
#endif
            }
          }
          doff += dstep;
        } else if (store) {
#pragma unroll
          for (int q = 0; q < WPL; ++q) outb[ad.at(q, rr, 0)] = packed[q];
        }
      }
      if constexpr (TYPE != kDiag) {
        if (seg > 0 && pass == 0 && st + 1 == m0) {
          // the warm-up guess of the state after stage m0 - 1
          uint32_t* gs = a.seg_state + size_t(slot) * 2 * a.seg_words + a.seg_words;
#pragma unroll
          for (int q = 0; q < NPAIR; ++q) __stcg(gs + q * GE::THREADS + tid, cs.prev[q]);
        }
      }
      if (TYPE != kDiag && store) fence_async_smem();  // output-tile writes -> async proxy
      __syncthreads();                                  // tile consumed, output tile written
      if (threadIdx.x == 0) {
        if (TYPE != kDiag && store) {
          tile_ops(st, false, outb, nullptr);
          tma_commit();
        }
        if (st + kDepth < rb) {
          mbar_expect_tx(&full[sl], stage_bytes(st + kDepth));
          tile_ops(st + kDepth, true, in_ring + sl * GE::STAGE_IN, &full[sl]);
        }
        if (TYPE != kDiag && store) tma_wait_read<kOutDepth - 1>();  // the next output buffer is free again
      }
      __syncthreads();
    }
    if constexpr (TYPE == kDiag) break;
    if (!(seg > 0 && pass == 0)) break;
    // Wait for the predecessor's true state after stage m0 - 1 (a lower
    // logical block: it started before this one, so it makes progress).
    if (threadIdx.x == 0) {
      const uint32_t* f = a.seg_flag + slot;
      uint32_t v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v) break;
        __nanosleep(64);
      }
      a.seg_flag[slot] = 0u;  // consumed; the next launch's producer sets it again
    }
    __syncthreads();
    const uint32_t* ts = a.seg_state + size_t(slot) * 2 * a.seg_words;
    const bool valid = c0 + t < J.nchains;
    bool diff = false;
#pragma unroll
    for (int q = 0; q < NPAIR; ++q)
      diff |= __ldcg(ts + q * GE::THREADS + tid) != __ldcg(ts + a.seg_words + q * GE::THREADS + tid);
    if (!__syncthreads_or(valid && diff)) break;
    if (threadIdx.x == 0) atomicAdd(a.reruns, 1ull);
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) cs.prev[q] = __ldcg(ts + q * GE::THREADS + tid);
    if (threadIdx.x == 0) tma_wait_all();  // own stores complete before rewriting them
    __syncthreads();
    ra = m0;
  }
  if constexpr (TYPE != kDiag) {
    if (seg < nseg - 1) {
      // publish this segment's (true) final state for segment seg + 1
      uint32_t* ts = a.seg_state + size_t(slot + 1) * 2 * a.seg_words;
#pragma unroll
      for (int q = 0; q < NPAIR; ++q) __stcg(ts + q * GE::THREADS + tid, cs.prev[q]);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.seg_flag + slot + 1), "r"(1u)
                     : "memory");
    }
  }
  if (TYPE != kDiag && threadIdx.x == 0) tma_wait_all();
}

template <int WPL, int G, int NPAIR>
__global__ void __launch_bounds__(Geo<WPL, G>::THREADS)
    k_aggregate_tma(const __grid_constant__ TmaArgs a) {
  using GE = Geo<WPL, G>;
  // TMA tensor copies need 128-byte aligned shared memory: the dynamic block
  // is over-allocated by 1 KiB and aligned in the shared address space.
  extern __shared__ __align__(16) uint32_t dsm[];
  const uint32_t pad_words = ((1024u - (smem_addr(dsm) & 1023u)) & 1023u) >> 2;
  uint32_t* in_ring = dsm + pad_words;                // kDepth * STAGE_IN
  uint32_t* out_ring = in_ring + kDepth * GE::STAGE_IN;  // kOutDepth * STAGE
  __shared__ __align__(8) uint64_t full[kDepth];
  __shared__ int s_block;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kDepth; ++i) mbar_init(&full[i], 1);
    fence_async_smem();
    // Segmented chains wait on lower logical blocks: hand out logical block
    // indices in start order (the last CTA rearms the counter for the next
    // launch on this workspace).
    int b = int(blockIdx.x);
    if (a.ticket) {
      b = int(atomicAdd(a.ticket, 1u));
      if (b == int(gridDim.x) - 1) atomicExch(a.ticket, 0u);
    }
    s_block = b;
  }
  __syncthreads();
  const int blk = s_block;
  int jidx = 0;
#pragma unroll 1
  while (jidx + 1 < a.njobs && blk >= a.job[jidx + 1].block0) ++jidx;
  const TmaJob& J = a.job[jidx];
  const int cta = (blk - J.block0) / J.nseg;
  const int cta_seg = (blk - J.block0) % J.nseg;
  unsigned long long t0 = 0;
  if (a.dbg == 100 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (J.type == kHoriz)
    agg_body<kHoriz, WPL, G, NPAIR>(a, J, cta, cta_seg, in_ring, out_ring, full);
  else if (J.type == kVert)
    agg_body<kVert, WPL, G, NPAIR>(a, J, cta, cta_seg, in_ring, out_ring, full);
  else
    agg_body<kDiag, WPL, G, NPAIR>(a, J, cta, 0, in_ring, out_ring, full);
  if (a.dbg == 100 && threadIdx.x == 0) {  // RPD_TMA_DBG=100: per-CTA timeline
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("AGGTR %d %d %d %d %d %d %d %u %llu %llu\n", WPL, G, blk, jidx, J.type, cta_seg, J.nseg,
           smid, t0, t1);
  }
}

using TmaKernel = void (*)(TmaArgs);

struct KernelInfo {
  TmaKernel fn;
  int smem;
  int threads;
  int R, wpp, row, cwf, cwl, nch, dcwf, dcwl;
  int npair;
};

template <int WPL, int G, int NPAIR>
KernelInfo info() {
  using GE = Geo<WPL, G>;
  return KernelInfo{k_aggregate_tma<WPL, G, NPAIR>,
                    (kDepth * GE::STAGE_IN + kOutDepth * GE::STAGE) * 4 + 1024,
                    GE::THREADS, GE::R, GE::WPP, GE::ROW, GE::CWF, GE::CWL, GE::NCH,
                    GE::DROW < 256 ? GE::DROW : 256, GE::DCWL, NPAIR};
}

KernelInfo pick(int wpl, int G, int levels) {
  const int npair_g1 = (levels + 1) / 2;  // G == 1: skip a trailing all-padding pair
#define RPD_TMA_G1(W_)                                                       \
  if (wpl == W_ && G == 1) {                                                 \
    if (npair_g1 == 2 * W_ - 1) return info<W_, 1, (2 * W_ - 1 > 0 ? 2 * W_ - 1 : 1)>(); \
    return info<W_, 1, 2 * W_>();                                            \
  }
#define RPD_TMA_GN(W_, G_) \
  if (wpl == W_ && G == G_) return info<W_, G_, 2 * W_>();
  RPD_TMA_G1(1) RPD_TMA_G1(2) RPD_TMA_G1(3) RPD_TMA_G1(4) RPD_TMA_G1(5) RPD_TMA_G1(6)
  RPD_TMA_G1(7) RPD_TMA_G1(8) RPD_TMA_G1(9) RPD_TMA_G1(17)
  RPD_TMA_GN(2, 2) RPD_TMA_GN(3, 2) RPD_TMA_GN(4, 2)
  RPD_TMA_GN(2, 4) RPD_TMA_GN(3, 4) RPD_TMA_GN(4, 4)
  RPD_TMA_GN(2, 8) RPD_TMA_GN(3, 8) RPD_TMA_GN(4, 8)
  RPD_TMA_GN(5, 2) RPD_TMA_GN(6, 2) RPD_TMA_GN(7, 2) RPD_TMA_GN(8, 2) RPD_TMA_GN(9, 2)
  RPD_TMA_GN(5, 4) RPD_TMA_GN(6, 4) RPD_TMA_GN(7, 4) RPD_TMA_GN(8, 4) RPD_TMA_GN(9, 4)
  RPD_TMA_GN(5, 8) RPD_TMA_GN(6, 8) RPD_TMA_GN(7, 8) RPD_TMA_GN(8, 8) RPD_TMA_GN(9, 8)
#undef RPD_TMA_G1
#undef RPD_TMA_GN
  throw InvalidArg("sgm: unsupported level layout for the TMA aggregation");
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    RPD_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      throw CudaFail("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

CUtensorMap make_map(void* base, int words_per_row, int rows, int depth, size_t pitch,
                     int box_x, int box_y) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {cuuint64_t(words_per_row), cuuint64_t(rows), cuuint64_t(depth)};
  const cuuint64_t strides[2] = {cuuint64_t(pitch), cuuint64_t(pitch) * cuuint64_t(rows)};
  const cuuint32_t box[3] = {cuuint32_t(box_x), cuuint32_t(box_y), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, base, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaFail("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

}  // namespace

bool sgm_tma_supported(const SgmLayout& L) {
  if (L.G == 1 && L.wpl == kWplG1Max) return true;
  return (L.G == 1 || L.G == 2 || L.G == 4 || L.G == 8) && L.wpl >= 1 && L.wpl <= 9 &&
         (L.G == 1 || L.wpl >= 2);
}

// Launches the aggregation of all 2P (volume, direction) jobs of one pass.
void launch_aggregate_tma(rpd_ctx* ctx, const SgmLayout& L, uint8_t* vol_lr, uint8_t* paths,
                          const int32_t* dirs, int paths_n, uint32_t p1, uint32_t p2,
                          int nvols) {
  const KernelInfo ki = pick(L.wpl, L.G, L.levels);
  const int wpp = L.lw / 4;
  const int words_row = L.w * wpp;
  TmaArgs args{};
  args.h = L.h;
  args.w = L.w;
  args.p1x2 = p1 | (p1 << 16);
  args.p2x2 = p2 | (p2 << 16);
  args.one = 1u;
  args.path_base = paths;
  args.pitch = L.pitch;
  args.vol_bytes = L.vol_bytes();
  {
    const char* e = debug_knob("RPD_TMA_DBG");
    args.dbg = e ? std::atoi(e) : 0;
  }
  const int R = ki.R;
  const int kNC = nc_of(L.G);
  args.cost_h = make_map(vol_lr, words_row, L.h, 2, L.pitch, R * wpp, kNC);
  args.cost_vf = make_map(vol_lr, words_row, L.h, 2, L.pitch, ki.cwf, R);
  args.cost_vl = make_map(vol_lr, words_row, L.h, 2, L.pitch, ki.cwl, R);
  args.cost_df = make_map(vol_lr, words_row, L.h, 2, L.pitch, ki.dcwf, 1);
  args.cost_dl = make_map(vol_lr, words_row, L.h, 2, L.pitch, ki.dcwl, 1);
  args.path_h = make_map(paths, words_row, L.h, 2 * paths_n, L.pitch, R * wpp, kNC);
  args.path_vf = make_map(paths, words_row, L.h, 2 * paths_n, L.pitch, ki.cwf, R);
  args.path_vl = make_map(paths, words_row, L.h, 2 * paths_n, L.pitch, ki.cwl, R);
  args.path_df = make_map(paths, words_row, L.h, 2 * paths_n, L.pitch, ki.cwf, 1);
  args.path_dl = make_map(paths, words_row, L.h, 2 * paths_n, L.pitch, ki.cwl, 1);
#ifndef RPD_AGG_WARM
#define RPD_AGG_WARM 64  // warm-up steps of a chain segment (multiple of R)
#endif
#ifndef RPD_AGG_SPLIT
#define RPD_AGG_SPLIT 1  // 0: never segment chains
#endif
  // H / V chains longer than the longest diagonal (min(W, H) steps) are cut
  // into segments of at most that length (plus the warm-up), so no job type
  // sets the serial makespan alone.
  const int lmin = std::min(L.w, L.h);
  int split = RPD_AGG_SPLIT, warm = RPD_AGG_WARM;
  if (const char* e = debug_knob("RPD_AGG_SPLIT")) split = std::atoi(e);  // checked build only
  if (const char* e = debug_knob("RPD_AGG_WARM")) warm = std::atoi(e);
  auto nseg_for = [&](int len) {
    // multi-lane chains (G > 1) already fill the SMs: segmenting them measured slower
    if (!split || lmin <= 0 || (L.G > 1 && split == 1)) return 1;
    // split > 1: force that many segments (A/B experiments, checked build)
    const int n = split > 1 ? split : std::min({8, cdiv(len, lmin), len / (3 * warm)});
    return std::max(n, 1);
  };
  args.warm_stages = warm / R;
  args.seg_words = ki.npair * ki.threads;
  int nslots = 0;
  int blocks = 0, nonseg_blocks = 0;
  const char* dbg = debug_knob("RPD_TMA_TYPES");  // debugging: bitmask of job types to run
  const int type_mask = dbg ? std::atoi(dbg) : 7;
#ifndef RPD_AGG_ORDER
#define RPD_AGG_ORDER 1
#endif
  // Block order = dispatch order: the long horizontal chains (W steps) first,
  // so they start on empty SMs; the shorter vertical / diagonal jobs fill in.
  for (int pass = 0; pass < (RPD_AGG_ORDER ? 3 : 1); ++pass)
  for (int vol = 0; vol < nvols; ++vol)
    for (int r = 0; r < paths_n; ++r) {
      const int du = dirs[2 * r], dv = dirs[2 * r + 1];
      const int ty = dv == 0 ? kHoriz : (du == 0 ? kVert : kDiag);
      if (RPD_AGG_ORDER && ty != pass) continue;
      if (!((type_mask >> ty) & 1)) continue;
      TmaJob& J = args.job[args.njobs++];
      J.vol = vol;
      J.path = vol * paths_n + r;
      J.du = dirs[2 * r];
      J.dv = dirs[2 * r + 1];
      if (J.dv == 0) {
        J.type = kHoriz;
        J.nchains = L.h;
      } else if (J.du == 0) {
        J.type = kVert;
        J.nchains = L.w;
      } else {
        J.type = kDiag;
        J.nchains = L.w + L.h - 1;
        J.kmin = J.du > 0 ? -(L.h - 1) : 0;
      }
      J.nseg = J.type == kHoriz ? nseg_for(L.w) : (J.type == kVert ? nseg_for(L.h) : 1);
      J.slot0 = nslots;
      J.block0 = blocks;
      nslots += cdiv(J.nchains, kNC) * (J.nseg - 1);
      blocks += cdiv(J.nchains, kNC) * J.nseg;
      nonseg_blocks += cdiv(J.nchains, kNC);
    }
  if (nslots > 0) {
    args.seg_state = ctx->ws.get<uint32_t>("agg_seg_state", size_t(nslots) * 2 * args.seg_words);
    unsigned* flags = ctx->ws.get<unsigned>("agg_seg_flags", size_t(nslots) + 1);
    // consumers rearm their flags and the last CTA the ticket: zero once per buffer
    if (ctx->agg_flags_zeroed != flags || ctx->agg_flags_words < nslots + 1) {
      RPD_CK(cudaMemsetAsync(flags, 0, (size_t(nslots) + 1) * sizeof(unsigned), ctx->stream));
      ctx->agg_flags_zeroed = flags;
      ctx->agg_flags_words = nslots + 1;
    }
    args.ticket = flags;
    args.seg_flag = flags + 1;
  }
  {
    unsigned long long* rr = ctx->ws.get<unsigned long long>("agg_reruns", 1);
    if (rr != ctx->agg_reruns) {
      RPD_CK(cudaMemsetAsync(rr, 0, sizeof(unsigned long long), ctx->stream));
      ctx->agg_reruns = rr;
    }
  }
  args.reruns = ctx->agg_reruns;
  ctx->agg_segmented_ctas = blocks - nonseg_blocks;
  RPD_CK(cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ki.smem));
  ki.fn<<<blocks, ki.threads, ki.smem, ctx->stream>>>(args);
  RPD_LAUNCH_CHECK();
}

}  // namespace rpdg
