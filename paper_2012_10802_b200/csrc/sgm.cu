// sgm.cu — semi-global matching for sm_100a.
//
// Reference: /root/reference/proj/src/sgm.cpp (census :13-34, cost :38-68,
// aggregation :70-110, swap :112-121, WTA :123-153, LR :155-170,
// match_pair :172-226) and include/rpd/perspective.hpp (warp :45-66,
// restore :69-80, shifts :23-35).
//
// Fast integer path.  With integral penalties every value the
// reference's float recursion produces is a small integer, so the recursion is
// evaluated on packed u16x2 lanes with the native sm_100 DPX instructions
// (VIADDMNMX.U16x2 = fused add+min, VIMNMX.U16x2) and stored as u8:
//   0 <= L_r(p,d) <= (window^2-1) + lambda2 <= 255.
// One thread (or a G-lane group) owns one scan chain and holds every disparity
// level of the chain's current pixel in registers; raw costs are prefetched D
// steps ahead.  All 2P (direction x {left,right}-reference) chains of a pass run
// in ONE launch and write per-path u8 volumes; a WTA kernel sums them (exact
// u16) and applies select_disparity's rules.  The right-reference cost volume
// C_R(v,u,d) = C_L(v,u+d,d) is generated directly from the census words.

#include <cfloat>
#include <type_traits>

#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include "sgm.cuh"

namespace rpdg {

// --------------------------------------------------------------- layout ----
namespace {
constexpr int kMaxFastLevels = 576;
}

#ifndef RPD_SGM_WIDE_G1
#define RPD_SGM_WIDE_G1 0  // 1: one lane per chain up to 68 levels (measured 1.4x slower bootstrap)
#endif
SgmLayout sgm_layout(int h, int w, int levels, int paths) {
  SgmLayout L;
  L.h = h;
  L.w = w;
  L.levels = levels;
  L.paths = paths;
  // tuning overrides "G,WPL" (RPD_SGM_LAYOUT_SMALL for <= 36 levels, _BIG otherwise)
  auto env_layout = [&](const char* name, int& G, int& wpl) {
    const char* e = debug_knob(name);
    int g = 0, wp = 0;
    if (e && std::sscanf(e, "%d,%d", &g, &wp) == 2 && g >= 1 && wp >= 1 && 4 * g * wp >= levels) {
      G = g;
      wpl = wp;
    }
  };
  if (levels <= 36) {
    L.G = 1;
    L.wpl = (levels + 3) / 4;
    env_layout("RPD_SGM_LAYOUT_SMALL", L.G, L.wpl);
  } else if (levels <= 4 * kWplG1Max && RPD_SGM_WIDE_G1) {
    // one lane per chain up to 68 levels (the D = 128 bootstrap's 65): no
    // shuffles on the step's dependency chain, 17 words per pixel instead of 20
    L.G = 1;
    L.wpl = kWplG1Max;
    env_layout("RPD_SGM_LAYOUT_BIG", L.G, L.wpl);
  } else {
    int G = 4;  // 4 lanes per chain: 2x the warps of G = 2
    while (4 * 9 * G < levels) G *= 2;
    L.G = G;
    L.wpl = std::max(5, (levels + 4 * G - 1) / (4 * G));
    env_layout("RPD_SGM_LAYOUT_BIG", L.G, L.wpl);
  }
  L.lw = 4 * L.wpl * L.G;
  L.pitch = size_t(round_up(w * L.lw, 16));  // TMA row strides must be 16-byte multiples
  return L;
}

bool sgm_fast_path_ok(float l1, float l2, int window) {
  const float maxc = float(window * window - 1);
  return l1 >= 1.0f && l2 >= l1 && l1 == std::floor(l1) && l2 == std::floor(l2) &&
         maxc + l2 <= 255.0f;
}

// ------------------------------------------------------- image kernels ----
__global__ void k_u8_to_f32(const uint8_t* __restrict__ in0, float* __restrict__ out0,
                            const uint8_t* __restrict__ in1, float* __restrict__ out1,
                            long long n) {
  const uint8_t* __restrict__ in = blockIdx.y ? in1 : in0;  // blockIdx.y: which image
  float* __restrict__ out = blockIdx.y ? out1 : out0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = float(in[i]);
}

// 16 pixels per thread: one 16-byte load, four 16-byte stores (n16 = n / 16
// groups; 16-byte aligned buffers), the remainder by the first threads.
__global__ void k_u8_to_f32_v16(const uint8_t* __restrict__ in0, float* __restrict__ out0,
                                const uint8_t* __restrict__ in1, float* __restrict__ out1,
                                int n16, int rem) {
  const uint8_t* __restrict__ in = blockIdx.y ? in1 : in0;
  float* __restrict__ out = blockIdx.y ? out1 : out0;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n16) {
    const uint4 b = reinterpret_cast<const uint4*>(in)[i];
    const uint32_t wd[4] = {b.x, b.y, b.z, b.w};
    float4* o = reinterpret_cast<float4*>(out) + 4 * size_t(i);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      o[k] = make_float4(float(wd[k] & 0xFFu), float((wd[k] >> 8) & 0xFFu),
                         float((wd[k] >> 16) & 0xFFu), float(wd[k] >> 24));
  }
  if (i < rem) out[16 * size_t(n16) + i] = float(in[16 * size_t(n16) + i]);
}

void launch_u8_to_f32(const uint8_t* in, float* out, long long n, cudaStream_t st,
                      const uint8_t* in1, float* out1) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (n < (1ll << 34) && al16(in) && al16(out) && (!in1 || (al16(in1) && al16(out1)))) {
    const int n16 = int(n / 16), rem = int(n % 16);
    const int blocks = std::max(1, cdiv(std::max(n16, rem), 256));
    k_u8_to_f32_v16<<<dim3(blocks, in1 ? 2 : 1), 256, 0, st>>>(in, out, in1, out1, n16, rem);
    RPD_LAUNCH_CHECK();
    return;
  }
  const int blocks = std::min<long long>((n + 255) / 256, 148 * 16);
  k_u8_to_f32<<<dim3(std::max(blocks, 1), in1 ? 2 : 1), 256, 0, st>>>(in, out, in1, out1, n);
  RPD_LAUNCH_CHECK();
}

// half_image, pipeline.cpp:25-34: 0.25f * (((a + b) + c) + d)
__global__ void k_half(const float* __restrict__ in0, const float* __restrict__ in1, int h, int w,
                       float* __restrict__ out0, float* __restrict__ out1) {
  const float* __restrict__ in = blockIdx.z ? in1 : in0;  // blockIdx.z: which image
  float* __restrict__ out = blockIdx.z ? out1 : out0;
  const int hh = h / 2, hw = w / 2;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  if (u >= hw || v >= hh) return;
  const float* r0 = in + size_t(2 * v) * w + 2 * u;
  const float* r1 = r0 + w;
  out[size_t(v) * hw + u] = 0.25f * (r0[0] + r0[1] + r1[0] + r1[1]);
}

void launch_half_image(const float* in, int h, int w, float* out, cudaStream_t st,
                       const float* in1, float* out1) {
  if (h / 2 == 0 || w / 2 == 0) return;
  k_half<<<dim3(cdiv(w / 2, 128), h / 2, in1 ? 2 : 1), 128, 0, st>>>(in, in1, h, w, out, out1);
  RPD_LAUNCH_CHECK();
}

// compute_row_shifts, perspective.hpp:23-35.  std::min / std::max semantics
// spelled out so signed zeros match.
__global__ void k_row_shifts(const DevModel* __restrict__ m, int h, int w, double delta,
                             double* __restrict__ shifts) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= h) return;
  const DevModel md = *m;
  const double g0 = road_at(md, 0.0, double(v));
  const double gw = road_at(md, double(w), double(v));
  const double lo = (gw < g0) ? gw : g0;
  const double x = lo - delta;
  shifts[v] = (0.0 < x) ? x : 0.0;
}

void launch_row_shifts(const DevModel* model, int h, int w, double delta_pt, double* shifts,
                       cudaStream_t st) {
  k_row_shifts<<<cdiv(h, 128), 128, 0, st>>>(model, h, w, delta_pt, shifts);
  RPD_LAUNCH_CHECK();
}

// warp_right_image, perspective.hpp:45-66
__global__ void k_warp(const float* __restrict__ right, const double* __restrict__ shifts, int h,
                       int w, float* __restrict__ out, uint8_t* __restrict__ iv) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= w) return;
  for (int v = blockIdx.y; v < h; v += gridDim.y) {  // rows strided over gridDim.y
    const size_t i = size_t(v) * w + u;
    const double s = double(u) - shifts[v];
    if (s < 0.0 || s > double(w - 1)) {
      out[i] = 0.0f;
      iv[i] = 0;
      continue;
    }
    const int s0 = int(floor(s));
    const int s1 = min(s0 + 1, w - 1);
    const double t = s - double(s0);
    const float* row = right + size_t(v) * w;
    out[i] = float((1.0 - t) * double(row[s0]) + t * double(row[s1]));
    iv[i] = 1;
  }
}

void launch_warp_right(const float* right, const double* shifts, int h, int w, float* out,
                       uint8_t* in_view, cudaStream_t st) {
  k_warp<<<dim3(cdiv(w, 128), std::max(1, cdiv(h, 4))), 128, 0, st>>>(right, shifts, h, w, out,
                                                                       in_view);
  RPD_LAUNCH_CHECK();
}

// restore_disparity, perspective.hpp:69-80
__global__ void k_restore(const float* __restrict__ d0, const double* __restrict__ shifts, int h,
                          int w, float* __restrict__ d1) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  if (u >= w) return;
  const size_t i = size_t(v) * w + u;
  const float d = d0[i];
  d1[i] = (d != kInvalid) ? d + float(shifts[v]) : d;
}

void launch_restore(const float* d0, const double* shifts, int h, int w, float* d1,
                    cudaStream_t st) {
  k_restore<<<dim3(cdiv(w, 128), h), 128, 0, st>>>(d0, shifts, h, w, d1);
  RPD_LAUNCH_CHECK();
}

// census_transform, sgm.cpp:13-34: MSB-first bits over the row-major window,
// centre skipped, coordinates clamped.  A CTA computes a 128 x kCensusRows
// block; the (rows + 2R) x (128 + 2R) window is staged once with clamped
// coordinates (== the reference's clamped reads) and each thread walks a
// column of the block.  Windows of <= 32 bits accumulate in 32-bit words.
constexpr int kCensusRows = 8;
template <int R>
__global__ void __launch_bounds__(128)
    k_census(const float* __restrict__ img0, const float* __restrict__ img1, int h, int w,
             uint64_t* __restrict__ out0, uint64_t* __restrict__ out1) {
  using Bits = typename std::conditional<((2 * R + 1) * (2 * R + 1) - 1 <= 32), uint32_t,
                                         uint64_t>::type;
  // blockIdx.z selects the image (both census transforms in one launch)
  const float* __restrict__ img = blockIdx.z ? img1 : img0;
  uint64_t* __restrict__ out = blockIdx.z ? out1 : out0;
  constexpr int TW = 128 + 2 * R;
  constexpr int TH = kCensusRows + 2 * R;
  __shared__ float tile[TH][TW];
  const int u0 = blockIdx.x * 128;
  const int v0 = blockIdx.y * kCensusRows;
  for (int r = 0; r < TH; ++r) {
    const int vv = min(max(v0 + r - R, 0), h - 1);
    const float* src = img + size_t(vv) * w;
    for (int c = threadIdx.x; c < TW; c += 128) tile[r][c] = src[min(max(u0 + c - R, 0), w - 1)];
  }
  __syncthreads();
  const int u = u0 + threadIdx.x;
  if (u >= w) return;
  const int t = threadIdx.x + R;
  // The thread's column of windows slides down the rows: each step loads one
  // new window row.  A bit is the sign of (neighbour - centre): for finite
  // floats a - b < 0 exactly when a < b (a difference of distinct floats is
  // never zero), and one funnel shift appends it.
  constexpr int K = 2 * R + 1;
  float win[K][K];
#pragma unroll
  for (int r = 0; r < K - 1; ++r)
#pragma unroll
    for (int k = 0; k < K; ++k) win[r][k] = tile[r][t - R + k];
#pragma unroll
  for (int y = 0; y < kCensusRows; ++y) {
#pragma unroll
    for (int k = 0; k < K; ++k) win[(y + K - 1) % K][k] = tile[y + K - 1][t - R + k];
    const int v = v0 + y;
    if (v >= h) break;
    const float c = win[(y + R) % K][R];
    uint32_t lo = 0, hi = 0;  // bits, most significant first (64-bit windows use both)
#pragma unroll
    for (int dv = 0; dv < K; ++dv) {
#pragma unroll
      for (int du = 0; du < K; ++du) {
        if (dv == R && du == R) continue;
        const uint32_t sg = __float_as_uint(__fsub_rn(win[(y + dv) % K][du], c));
        if (sizeof(Bits) == 8) hi = __funnelshift_l(lo, hi, 1);
        lo = __funnelshift_l(sg, lo, 1);
      }
    }
    out[size_t(v) * w + u] = sizeof(Bits) == 8 ? ((uint64_t(hi) << 32) | lo) : uint64_t(lo);
  }
}

void launch_census2(const float* img0, const float* img1, int h, int w, int window,
                    uint64_t* out0, uint64_t* out1, cudaStream_t st) {
  const dim3 grid(cdiv(w, 128), cdiv(h, kCensusRows), img1 ? 2 : 1);
  switch (window) {
    case 3: k_census<1><<<grid, 128, 0, st>>>(img0, img1, h, w, out0, out1); break;
    case 5: k_census<2><<<grid, 128, 0, st>>>(img0, img1, h, w, out0, out1); break;
    case 7: k_census<3><<<grid, 128, 0, st>>>(img0, img1, h, w, out0, out1); break;
    default: throw InvalidArg("census_cost_volume: window must be odd");
  }
  RPD_LAUNCH_CHECK();
}

void launch_census(const float* img, int h, int w, int window, uint64_t* out, cudaStream_t st) {
  launch_census2(img, nullptr, h, w, window, out, nullptr, st);
}

// census_cost_volume, sgm.cpp:38-68, float output in the reference layout.
__global__ void k_cost_f32(const uint64_t* __restrict__ cl, const uint64_t* __restrict__ cr,
                           const uint8_t* __restrict__ iv, int h, int w, int levels, float maxc,
                           float* __restrict__ costs) {
  const long long n = (long long)h * w * levels;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = int(i % levels);
    const long long p = i / levels;
    const int u = int(p % w);
    const int ur = u - d;
    float c;
    if (ur < 0 || (iv && !iv[p - d]))
      c = maxc;
    else
      c = float(__popcll(cl[p] ^ cr[p - d]));
    costs[i] = c;
  }
}

void launch_cost_f32(const uint64_t* cl, const uint64_t* cr, const uint8_t* in_view, int h, int w,
                     int levels, int window, float* costs, cudaStream_t st) {
  const long long n = (long long)h * w * levels;
  const int blocks = int(std::min<long long>((n + 255) / 256, 148 * 32));
  k_cost_f32<<<std::max(blocks, 1), 256, 0, st>>>(cl, cr, in_view, h, w, levels,
                                                  float(window * window - 1), costs);
  RPD_LAUNCH_CHECK();
}

// --------------------------------------------------- fast u8 cost volumes --
// One thread per (pixel, 4-level word).  Levels >= L are padded with 0xFF.
// C_L(v,u,d) = popc(cl(u) ^ cr(u-d))  if u-d >= 0 and in_view(u-d), else maxc
// C_R(v,u,d) = popc(cl(u+d) ^ cr(u))  if u+d <  W and in_view(u),   else maxc
// One CTA per image row: the row's census words are staged in shared memory
// with `levels` padding entries on both sides, and an override byte per entry
// (0xFF for an invalid or out-of-row pixel, else 0), so every cost is
// branch-free: min(popc(a ^ b) | ov, maxc) == maxc exactly when the reference
// substitutes maxc (sgm.cpp:40-60; a valid popcount never exceeds maxc).
// Volume words are produced in storage order (coalesced stores).
template <typename CW>  // staged census word: uint32_t when the window has <= 32 bits
__global__ void __launch_bounds__(256)
    k_cost_u8(const uint64_t* __restrict__ cl, const uint64_t* __restrict__ cr,
              const uint8_t* __restrict__ iv, int h, int w, int levels, int nw,
              size_t pitch_words, uint32_t maxc, uint32_t* __restrict__ vol_l,
              uint32_t* __restrict__ vol_r) {
  extern __shared__ uint64_t csm[];  // cl[W] | cr[W] | ov[W] bytes, W = w + 2*levels
  const int W = w + 2 * levels;
  CW* s_cl = reinterpret_cast<CW*>(csm) + levels;  // s_cl[u], u in [-levels, w + levels)
  CW* s_cr = reinterpret_cast<CW*>(csm) + W + levels;
  uint8_t* s_ov = reinterpret_cast<uint8_t*>(reinterpret_cast<CW*>(csm) + 2 * W) + levels;
  const int v = blockIdx.y;
  const long long row = (long long)v * w;
  for (int u = int(threadIdx.x) - levels; u < w + levels; u += blockDim.x) {
    const bool in = u >= 0 && u < w;
    s_cl[u] = in ? CW(cl[row + u]) : CW(0);
    s_cr[u] = in ? CW(cr[row + u]) : CW(0);
    s_ov[u] = (in && iv[row + u]) ? 0 : 0xFF;
  }
  __syncthreads();
  uint32_t* ol = vol_l + size_t(v) * pitch_words;
  uint32_t* orr = vol_r + size_t(v) * pitch_words;
  const int total = w * nw;
  const float inv_nw = 1.0f / float(nw);
  auto popc = [](CW x) -> uint32_t {
    if constexpr (sizeof(CW) == 8)
      return uint32_t(__popcll(x));
    else
      return uint32_t(__popc(x));
  };
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    // i / nw exactly: (i + 0.5) / nw is >= 1/(2 nw) away from an integer
    const int u = int(__fmul_rn(float(i) + 0.5f, inv_nw));
    const int j = i - u * nw;
    const CW a = s_cl[u];
    const CW b = s_cr[u];
    const uint32_t ovu = s_ov[u];
    const int d0 = 4 * j;
    const CW* crd = s_cr + (u - d0);
    const uint8_t* ovd = s_ov + (u - d0);
    const CW* cld = s_cl + (u + d0);
    uint32_t wl, wr;
    if (d0 >= levels) {  // padding word
      wl = 0xFFFFFFFFu;
      wr = 0xFFFFFFFFu;
    } else if (d0 + 3 < levels) {  // full word
      uint32_t cL[4], cR[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        cL[q] = min(popc(a ^ crd[-q]) | ovd[-q], maxc);
        cR[q] = min(popc(cld[q] ^ b) | ovu | (u + d0 + q >= w ? 0xFFu : 0u), maxc);
      }
      wl = __byte_perm(__byte_perm(cL[0], cL[1], 0x0040), __byte_perm(cL[2], cL[3], 0x0040), 0x5410);
      wr = __byte_perm(__byte_perm(cR[0], cR[1], 0x0040), __byte_perm(cR[2], cR[3], 0x0040), 0x5410);
    } else {
      wl = 0;
      wr = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t x = 0xFF, y = 0xFF;
        if (d0 + q < levels) {
          x = min(popc(a ^ crd[-q]) | ovd[-q], maxc);
          y = min(popc(cld[q] ^ b) | ovu | (u + d0 + q >= w ? 0xFFu : 0u), maxc);
        }
        wl |= x << (8 * q);
        wr |= y << (8 * q);
      }
    }
    ol[i] = wl;
    orr[i] = wr;
  }
}

// Rows too wide to stage in shared memory.
__global__ void k_cost_u8_flat(const uint64_t* __restrict__ cl, const uint64_t* __restrict__ cr,
                          const uint8_t* __restrict__ iv, int h, int w, int levels, int nw,
                          size_t pitch_words, uint32_t maxc, uint32_t* __restrict__ vol_l,
                          uint32_t* __restrict__ vol_r) {
  const long long n = (long long)h * w * nw;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = int(i % nw);
    const long long p = i / nw;
    const int u = int(p % w);
    const size_t o = size_t(p / w) * pitch_words + size_t(u) * nw + j;
    const uint64_t a = cl[p];
    const uint64_t b = cr[p];
    const bool ivu = iv[p] != 0;
    uint32_t wl = 0, wr = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int d = 4 * j + q;
      uint32_t cL = 0xFF, cR = 0xFF;
      if (d < levels) {
        cL = (u - d < 0 || !iv[p - d]) ? maxc : uint32_t(__popcll(a ^ cr[p - d]));
        cR = (u + d >= w || !ivu) ? maxc : uint32_t(__popcll(cl[p + d] ^ b));
      }
      wl |= cL << (8 * q);
      wr |= cR << (8 * q);
    }
    vol_l[o] = wl;
    vol_r[o] = wr;
  }
}

// Pixel-major cost volumes for census windows of <= 24 bits (3x3, 5x5) and a
// compile-time word count NW.  One CTA per image row; each staged census entry
// carries its own override: {word | ov << 24, ov ? ~0 : 0} with ov set for
// out-of-row pixels (and, on the right view, out-of-view ones), so a cost is
// LDS.64 + LOP3 ((a ^ e) | m) + POPC + IMNMX: an overridden entry counts 32
// bits, clamped to maxc exactly as the reference substitutes it (a valid
// count never exceeds maxc).  A thread owns one pixel and all its levels, the
// row chunk's words are staged in shared memory and written back coalesced.
// LV > 0: compile-time level count (the pipeline's passes): words that hold
// only padding levels are stored as 0xFF bytes without computing costs.
template <int NW, int LV = 0>
__global__ void __launch_bounds__(256)
    k_cost_px(const uint64_t* __restrict__ cl, const uint64_t* __restrict__ cr,
              const uint8_t* __restrict__ iv, int w, int levels, size_t pitch_words,
              uint32_t maxc, uint32_t* __restrict__ vol_l, uint32_t* __restrict__ vol_r) {
  constexpr int TPX = 256;
  constexpr int PAD = 4 * NW;  // every stored level, padding ones included, reads in range
  constexpr int V = NW % 4 == 0 ? 4 : (NW % 2 == 0 ? 2 : 1);  // words per shared store
  extern __shared__ __align__(16) uint32_t csx[];
  const int W = w + 2 * PAD;
  uint2* s_r = reinterpret_cast<uint2*>(csx) + PAD;          // right-view entries, x in [-PAD, w+PAD)
  uint2* s_l = reinterpret_cast<uint2*>(csx) + W + PAD;      // left-view entries
  uint32_t* o_l = csx + 4 * W;                               // [TPX * NW] words per volume
  uint32_t* o_r = o_l + TPX * NW;
  const int v = blockIdx.x;
  const long long row = (long long)v * w;
  for (int x = int(threadIdx.x) - PAD; x < w + PAD; x += blockDim.x) {
    const bool in = x >= 0 && x < w;
    const uint32_t a = in ? uint32_t(cl[row + x]) : 0u;
    const uint32_t b = in ? uint32_t(cr[row + x]) : 0u;
    const bool ovr = !in || !iv[row + x];
    s_r[x] = ovr ? make_uint2(b | 0xFF000000u, 0xFFFFFFFFu) : make_uint2(b, 0u);
    s_l[x] = in ? make_uint2(a, 0u) : make_uint2(0xFF000000u, 0xFFFFFFFFu);
  }
  __syncthreads();
  uint32_t* gl = vol_l + size_t(v) * pitch_words;
  uint32_t* gr = vol_r + size_t(v) * pitch_words;
  for (int u0 = 0; u0 < w; u0 += TPX) {
    const int npx = min(TPX, w - u0);
    const int t = threadIdx.x;
    if (t < npx) {
      const int u = u0 + t;
      const uint32_t a = s_l[u].x;        // left census of u (in row: no override)
      const uint2 eb = s_r[u];
      const uint32_t b = eb.x & 0xFFFFFFu;
      const bool ovu = eb.y != 0u;        // right reference: own pixel out of view -> all maxc
      const uint2* pr = s_r + u;
      const uint2* pl = s_l + u;
#pragma unroll
      for (int j0 = 0; j0 < NW; j0 += V) {
        uint32_t bl[V], br[V];
#pragma unroll
        for (int jj = 0; jj < V; ++jj) {
          const int j = j0 + jj;
          if (LV > 0 && 4 * j >= LV) {  // padding word
            bl[jj] = br[jj] = 0xFFFFFFFFu;
            continue;
          }
          uint32_t cL[4], cR[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int d = 4 * j + q;
            const uint2 e = pr[-d];
            const uint2 f = pl[d];
            cL[q] = min(uint32_t(__popc((a ^ e.x) | e.y)), maxc);
            cR[q] = min(uint32_t(__popc((f.x ^ b) | f.y)), maxc);
          }
          uint32_t wl = __byte_perm(__byte_perm(cL[0], cL[1], 0x0040),
                                    __byte_perm(cL[2], cL[3], 0x0040), 0x5410);
          uint32_t wr = __byte_perm(__byte_perm(cR[0], cR[1], 0x0040),
                                    __byte_perm(cR[2], cR[3], 0x0040), 0x5410);
          if (ovu) wr = maxc * 0x01010101u;
          const int nlev = LV > 0 ? LV : levels;
          if (4 * j + 3 >= nlev) {  // padding levels (the last words only)
            const int k = nlev - 4 * j;  // valid bytes in this word, <= 3
            const uint32_t keep = k <= 0 ? 0u : (0xFFFFFFFFu >> (32 - 8 * k));
            wl = (wl & keep) | ~keep;
            wr = (wr & keep) | ~keep;
          }
          bl[jj] = wl;
          br[jj] = wr;
        }
        if constexpr (V == 4) {
          *reinterpret_cast<uint4*>(o_l + t * NW + j0) = make_uint4(bl[0], bl[1], bl[2], bl[3]);
          *reinterpret_cast<uint4*>(o_r + t * NW + j0) = make_uint4(br[0], br[1], br[2], br[3]);
        } else if constexpr (V == 2) {
          *reinterpret_cast<uint2*>(o_l + t * NW + j0) = make_uint2(bl[0], bl[1]);
          *reinterpret_cast<uint2*>(o_r + t * NW + j0) = make_uint2(br[0], br[1]);
        } else {
          o_l[t * NW + j0] = bl[0];
          o_r[t * NW + j0] = br[0];
        }
      }
    }
    __syncthreads();
    const int nwords = npx * NW;
    uint32_t* dl = gl + size_t(u0) * NW;
    uint32_t* dr = gr + size_t(u0) * NW;
    const int nvec = nwords >> 2;  // u0 * NW * 4 bytes and the pitch are 16-byte multiples
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
      reinterpret_cast<uint4*>(dl)[i] = reinterpret_cast<const uint4*>(o_l)[i];
      reinterpret_cast<uint4*>(dr)[i] = reinterpret_cast<const uint4*>(o_r)[i];
    }
    for (int i = 4 * nvec + threadIdx.x; i < nwords; i += blockDim.x) {
      dl[i] = o_l[i];
      dr[i] = o_r[i];
    }
    __syncthreads();
  }
}

namespace {
using CostPxKernel = void (*)(const uint64_t*, const uint64_t*, const uint8_t*, int, int, size_t,
                              uint32_t, uint32_t*, uint32_t*);
CostPxKernel cost_px_pick(int nw, int levels) {
  // compile-time level counts of the pipeline's passes (as wta_bulk_pick)
  if (nw == 5 && levels == 17) return k_cost_px<5, 17>;
  if (nw == 9 && levels == 33) return k_cost_px<9, 33>;
  if (nw == 20 && levels == 65) return k_cost_px<20, 65>;
  if (nw == 17 && levels == 65) return k_cost_px<17, 65>;
  if (nw == 36 && levels == 129) return k_cost_px<36, 129>;
  switch (nw) {
    case 1: return k_cost_px<1>;
    case 2: return k_cost_px<2>;
    case 3: return k_cost_px<3>;
    case 4: return k_cost_px<4>;
    case 5: return k_cost_px<5>;
    case 6: return k_cost_px<6>;
    case 7: return k_cost_px<7>;
    case 8: return k_cost_px<8>;
    case 9: return k_cost_px<9>;
    case 17: return k_cost_px<17>;
    case 20: return k_cost_px<20>;
    case 24: return k_cost_px<24>;
    case 28: return k_cost_px<28>;
    case 32: return k_cost_px<32>;
    case 36: return k_cost_px<36>;
    default: return nullptr;
  }
}
}  // namespace

// u8 volume (row pitch, pixel stride lw) -> float reference layout (parity dumps only).
__global__ void k_u8vol_to_f32(const uint8_t* __restrict__ vol, int w, long long npix,
                               size_t pitch, int lw, int levels, float* __restrict__ out) {
  const long long n = npix * levels;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / levels;
    const int d = int(i % levels);
    out[i] = float(vol[size_t(p / w) * pitch + size_t(p % w) * lw + d]);
  }
}

// Float reference layout -> u8 volume (row pitch, pixel stride lw), levels
// >= L padded with 0xFF like the cost kernels (aggregate_costs ABI route).
__global__ void k_f32_to_u8vol(const float* __restrict__ in, int w, long long npix, size_t pitch,
                               int lw, int levels, uint8_t* __restrict__ vol) {
  const long long n = npix * lw;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / lw;
    const int d = int(i % lw);
    vol[size_t(p / w) * pitch + size_t(p % w) * lw + d] =
        d < levels ? uint8_t(in[p * levels + d]) : uint8_t(0xFF);
  }
}

// ------------------------------------------------------ path aggregation --
struct AggJob {
  const uint8_t* cost;
  uint8_t* out;
  int du, dv;
  int nchains;
  int block0;
};
struct AggArgs {
  AggJob job[16];
  int njobs;
  int h, w, lw;
  size_t pitch;
  uint32_t p1x2, p2x2;
};

constexpr uint32_t kInf2 = 0x7FFF7FFFu;
constexpr int kAggThreads = 64;

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

// Scan-chain cursor.  Horizontal chains are rows; vertical chains columns;
// diagonal chains start at column `chain` of the first row and wrap around the
// image width — a wrap starts a new reference chain (no predecessor).
struct Cursor {
  int v, u;
};

template <int WPL, int G, int D>
__global__ void __launch_bounds__(kAggThreads)
    k_aggregate(const __grid_constant__ AggArgs a) {
  constexpr int NPL = 2 * WPL;
  constexpr int CPB = kAggThreads / G;
  int j = 0;
#pragma unroll 1
  while (j + 1 < a.njobs && int(blockIdx.x) >= a.job[j + 1].block0) ++j;
  const AggJob& J = a.job[j];
  const int g = threadIdx.x % G;
  const int chain = (int(blockIdx.x) - J.block0) * CPB + int(threadIdx.x) / G;
  if (chain >= J.nchains) return;  // whole group leaves together
  const unsigned gmask =
      G == 32 ? 0xFFFFFFFFu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));

  const int h = a.h, w = a.w, lw = a.lw;
  const int du = J.du, dv = J.dv;
  const bool horiz = dv == 0;
  const int nsteps = horiz ? w : h;
  auto start = [&]() {
    Cursor c;
    if (horiz) {
      c.v = chain;
      c.u = du > 0 ? 0 : w - 1;
    } else {
      c.v = dv > 0 ? 0 : h - 1;
      c.u = chain;
    }
    return c;
  };
  auto advance = [&](Cursor& c) {
    if (horiz) {
      c.u += du;
    } else {
      c.v += dv;
      c.u += du;
      if (c.u >= w) c.u -= w;
      if (c.u < 0) c.u += w;
    }
  };
  const uint8_t* __restrict__ cost = J.cost + g * WPL * 4;
  uint8_t* __restrict__ out = J.out + g * WPL * 4;
  auto offset = [&](const Cursor& c) { return size_t(c.v) * a.pitch + size_t(c.u) * lw; };

  uint32_t buf[D][WPL];
  Cursor pc = start();
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < nsteps) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(cost + offset(pc));
#pragma unroll
      for (int q = 0; q < WPL; ++q) buf[k][q] = __ldg(src + q);
      advance(pc);
    }
  }

  Cursor cc = start();
  uint32_t prev[NPL];
  uint32_t mnx2 = 0;
#pragma unroll
  for (int k = 0; k < NPL; ++k) prev[k] = kInf2;

  for (int s0 = 0; s0 < nsteps; s0 += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int s = s0 + k;
      if (s >= nsteps) break;
      uint32_t raw[NPL];
#pragma unroll
      for (int q = 0; q < WPL; ++q) {
        raw[2 * q] = __byte_perm(buf[k][q], 0u, 0x4140);
        raw[2 * q + 1] = __byte_perm(buf[k][q], 0u, 0x4342);
      }
      if (s + D < nsteps) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(cost + offset(pc));
#pragma unroll
        for (int q = 0; q < WPL; ++q) buf[k][q] = __ldg(src + q);
        advance(pc);
      }
      const bool has_pred =
          s > 0 && (horiz || du == 0 || unsigned(cc.u - du) < unsigned(w));
      uint32_t cur[NPL];
      if (!has_pred) {
#pragma unroll
        for (int q = 0; q < NPL; ++q) cur[q] = raw[q];
      } else {
        uint32_t lo_nb = kInf2, hi_nb = kInf2;
        if (G > 1) {
          const uint32_t up = __shfl_up_sync(gmask, prev[NPL - 1], 1, G);
          const uint32_t dn = __shfl_down_sync(gmask, prev[0], 1, G);
          if (g > 0) lo_nb = up;
          if (g < G - 1) hi_nb = dn;
        }
        const uint32_t ceil2 = mnx2 + a.p2x2;
        uint32_t qprev = __byte_perm(lo_nb, prev[0], 0x5432);  // (prev[d-1], prev[d]) of pair 0
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
          const uint32_t nxt = (q + 1 < NPL) ? prev[q + 1] : hi_nb;
          const uint32_t qn = __byte_perm(prev[q], nxt, 0x5432);  // (prev[2q+1], prev[2q+2])
          uint32_t t = __viaddmin_u16x2(qprev, a.p1x2, prev[q]);
          t = __viaddmin_u16x2(qn, a.p1x2, t);
          t = __vminu2(t, ceil2);
          cur[q] = raw[q] + t - mnx2;  // per-half exact: t >= mn, no carry
          qprev = qn;
        }
      }
      {
        uint32_t* dst = reinterpret_cast<uint32_t*>(out + offset(cc));
#pragma unroll
        for (int q = 0; q < WPL; ++q) dst[q] = __byte_perm(cur[2 * q], cur[2 * q + 1], 0x6420);
      }
      const uint32_t m2 = min_pairs<NPL>(cur);
      uint32_t m = min(m2 & 0xFFFFu, m2 >> 16);
      if (G > 1) {
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1)
          m = min(m, __shfl_xor_sync(gmask, m, off, G));
      }
      mnx2 = m * 0x10001u;
#pragma unroll
      for (int q = 0; q < NPL; ++q) prev[q] = cur[q];
      advance(cc);
    }
  }
}

using AggKernel = void (*)(AggArgs);

template <int WPL, int G>
AggKernel pick_depth() {
  if constexpr (WPL <= 5)
    return k_aggregate<WPL, G, 8>;
  else
    return k_aggregate<WPL, G, 4>;
}

AggKernel agg_kernel(int wpl, int G) {
#define RPD_AGG_CASE(W_, G_) \
  if (wpl == W_ && G == G_) return pick_depth<W_, G_>();
  RPD_AGG_CASE(1, 1) RPD_AGG_CASE(2, 1) RPD_AGG_CASE(3, 1) RPD_AGG_CASE(4, 1)
  RPD_AGG_CASE(5, 1) RPD_AGG_CASE(6, 1) RPD_AGG_CASE(7, 1) RPD_AGG_CASE(8, 1)
  RPD_AGG_CASE(9, 1)
  RPD_AGG_CASE(5, 2) RPD_AGG_CASE(6, 2) RPD_AGG_CASE(7, 2) RPD_AGG_CASE(8, 2) RPD_AGG_CASE(9, 2)
  RPD_AGG_CASE(5, 4) RPD_AGG_CASE(6, 4) RPD_AGG_CASE(7, 4) RPD_AGG_CASE(8, 4) RPD_AGG_CASE(9, 4)
  RPD_AGG_CASE(5, 8) RPD_AGG_CASE(6, 8) RPD_AGG_CASE(7, 8) RPD_AGG_CASE(8, 8) RPD_AGG_CASE(9, 8)
  RPD_AGG_CASE(5, 16) RPD_AGG_CASE(6, 16) RPD_AGG_CASE(7, 16) RPD_AGG_CASE(8, 16)
  RPD_AGG_CASE(9, 16)
#undef RPD_AGG_CASE
  throw InvalidArg("sgm: unsupported level layout");
}

// ----------------------------------------------------- WTA (select_disparity)
// Sums the P per-path u8 volumes into exact u16 costs S(d) and applies
// sgm.cpp:123-153: first argmin; invalid if S(d) <= S(best) for |d-best| > 1;
// parabola with float arithmetic in the reference's order.
struct WtaArgs {
  const uint8_t* path[8];
  int paths;
  long long npix;
  int w;
  size_t pitch;
  int lw, levels;
  float* disp;
  float* dump;  // optional S(d) in the reference float layout
};

__device__ __forceinline__ void wta_visit(uint32_t s, int d, uint32_t& minv, int& best,
                                          int& cnt, uint32_t& last, uint32_t& sbm1,
                                          uint32_t& sbp1) {
  if (d == best + 1) sbp1 = s;
  if (s < minv) {
    minv = s;
    best = d;
    cnt = 1;
    sbm1 = last;
  } else if (s == minv) {
    ++cnt;
  }
  last = s;
}

__global__ void k_wta(const __grid_constant__ WtaArgs a) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= a.npix) return;
  const int nw = a.lw / 4;
  const size_t base = size_t(p / a.w) * a.pitch + size_t(p % a.w) * a.lw;
  uint32_t minv = 0xFFFFFFFFu, last = 0, sbm1 = 0, sbp1 = 0;
  int best = -2, cnt = 0;
  for (int j = 0; j < nw; ++j) {
    if (4 * j >= a.levels) break;
    uint32_t s01 = 0, s23 = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < a.paths) {
        const uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(a.path[r] + base) + j);
        s01 += __byte_perm(x, 0u, 0x4140);
        s23 += __byte_perm(x, 0u, 0x4342);
      }
    }
    const uint32_t sv[4] = {s01 & 0xFFFFu, s01 >> 16, s23 & 0xFFFFu, s23 >> 16};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int d = 4 * j + q;
      if (d < a.levels) {
        wta_visit(sv[q], d, minv, best, cnt, last, sbm1, sbp1);
        if (a.dump) a.dump[p * a.levels + d] = float(sv[q]);
      }
    }
  }
  // occurrences of the minimum other than best and best+1 make it ambiguous
  const int near = (best + 1 < a.levels && sbp1 == minv) ? 1 : 0;
  float r;
  if (cnt - 1 - near > 0) {
    r = kInvalid;
  } else {
    r = float(best);
    if (best > 0 && best < a.levels - 1) {
      const float cm = float(sbm1), cb = float(minv), cp = float(sbp1);
      const float denom = cm + cp - 2.0f * cb;
      if (denom > 0.0f) r += (cm - cp) / (2.0f * denom);
    }
  }
  a.disp[p] = r;
}

// Tiled WTA: a CTA takes kWtaPx consecutive pixels of one image row.  Phase 1
// sums the P per-path u8 words of the tile with fully coalesced loads (thread
// i owns tile words i, i+kWtaPx, ...) into exact u16x2 pairs; phase 2 hands
// each pixel's pairs to its own thread through shared memory.
constexpr int kWtaPx = 128;
constexpr int kWtaMaxWords = 36;  // lw <= 144 bytes (L <= 144)

template <int P>  // path count (4 or 8): fully unrolled sums
__global__ void __launch_bounds__(kWtaPx) k_wta_tiled(const __grid_constant__ WtaArgs a) {
  extern __shared__ uint32_t sums[];  // [pixel][2*nw + 1] u16x2 pairs (odd stride: no conflicts)
  const int nw = a.lw / 4;
  const int row = blockIdx.y;
  const int u0 = blockIdx.x * kWtaPx;
  const int npx = min(kWtaPx, a.w - u0);
  const int tile_words = npx * nw;
  const int stride = 2 * nw + 1;
  const size_t base = size_t(row) * a.pitch + size_t(u0) * a.lw;
  // 16-byte loads: 8 paths x 16 B in flight per thread (tile bases are
  // 16-byte aligned: pitch and u0 * lw are multiples of 16)
  const int nvec = tile_words >> 2;
  const float inv_nw = 1.0f / float(nw);
  for (int i4 = threadIdx.x; i4 < nvec; i4 += kWtaPx) {
    uint4 x[P];
#pragma unroll
    for (int r = 0; r < P; ++r) x[r] = __ldg(reinterpret_cast<const uint4*>(a.path[r] + base) + i4);
    // (4 i4) / nw exactly: (4 i4 + 0.5) / nw is >= 1/(2 nw) away from an integer
    int px = int(__fmul_rn(float(4 * i4) + 0.5f, inv_nw)), j = 4 * i4 - px * nw;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t s01 = 0, s23 = 0;
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const uint32_t xe = e == 0 ? x[r].x : (e == 1 ? x[r].y : (e == 2 ? x[r].z : x[r].w));
        s01 += __byte_perm(xe, 0u, 0x4140);
        s23 += __byte_perm(xe, 0u, 0x4342);
      }
      sums[px * stride + 2 * j] = s01;
      sums[px * stride + 2 * j + 1] = s23;
      if (++j == nw) {
        j = 0;
        ++px;
      }
    }
  }
  for (int i = 4 * nvec + threadIdx.x; i < tile_words; i += kWtaPx) {
    uint32_t s01 = 0, s23 = 0;
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(a.path[r] + base) + i);
      s01 += __byte_perm(x, 0u, 0x4140);
      s23 += __byte_perm(x, 0u, 0x4342);
    }
    const int px = i / nw, j = i - px * nw;
    sums[px * stride + 2 * j] = s01;
    sums[px * stride + 2 * j + 1] = s23;
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= npx) return;
  const long long p = (long long)row * a.w + u0 + t;
  uint32_t minv = 0xFFFFFFFFu, sbm1 = 0, sbp1 = 0;
  int best = -2, cnt = 0;
  const uint32_t* my = sums + t * stride;  // my[q] = exact u16 sums of levels (2q, 2q+1)
  const int L = a.levels;
  if (a.dump) {  // parity dumps: the reference's sequential scan, level by level
    uint32_t last = 0;
    for (int j = 0; j < nw; ++j) {
      if (4 * j >= L) break;
      const uint32_t s01 = my[2 * j], s23 = my[2 * j + 1];
      const uint32_t sv[4] = {s01 & 0xFFFFu, s01 >> 16, s23 & 0xFFFFu, s23 >> 16};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int d = 4 * j + q;
        if (d < L) {
          wta_visit(sv[q], d, minv, best, cnt, last, sbm1, sbp1);
          a.dump[p * L + d] = float(sv[q]);
        }
      }
    }
  } else {
    // Same result as the sequential scan (select_disparity, sgm.cpp:123-153):
    // minv = minimum, best = its FIRST level, cnt = its multiplicity,
    // sbm1 / sbp1 = the sums at best -+ 1 (0 / irrelevant at the ends).
    const int np = (L + 1) >> 1;
    const uint32_t hpad = (L & 1) ? 0xFFFF0000u : 0u;  // invalid high half of the last pair
    uint32_t m2 = 0xFFFFFFFFu;
    for (int q = 0; q < np; q += 2) {
      const uint32_t v0 = my[q] | (q == np - 1 ? hpad : 0u);
      const uint32_t v1 = q + 1 < np ? (my[q + 1] | (q + 1 == np - 1 ? hpad : 0u)) : 0xFFFFFFFFu;
      m2 = __vimin3_u16x2(m2, v0, v1);
    }
    minv = min(m2 & 0xFFFFu, m2 >> 16);
    best = -1;
    for (int q = 0; q < np; ++q) {
      const uint32_t v = my[q] | (q == np - 1 ? hpad : 0u);
      const bool lo = (v & 0xFFFFu) == minv, hi = (v >> 16) == minv;
      cnt += int(lo) + int(hi);
      best = best >= 0 ? best : (lo ? 2 * q : (hi ? 2 * q + 1 : -1));
    }
    auto level = [&](int d) { return (my[d >> 1] >> (16 * (d & 1))) & 0xFFFFu; };
    sbm1 = best > 0 ? level(best - 1) : 0u;
    sbp1 = best + 1 < L ? level(best + 1) : 0u;
  }
  const int near = (best + 1 < a.levels && sbp1 == minv) ? 1 : 0;
  float r;
  if (cnt - 1 - near > 0) {
    r = kInvalid;
  } else {
    r = float(best);
    if (best > 0 && best < a.levels - 1) {
      const float cm = float(sbm1), cb = float(minv), cp = float(sbp1);
      const float denom = cm + cp - 2.0f * cb;
      if (denom > 0.0f) r += (cm - cp) / (2.0f * denom);
    }
  }
  a.disp[p] = r;
}

// Bulk WTA: both reference volumes of a pass in one launch (blockIdx.z), the
// words per pixel NW a compile-time constant.  An elected thread copies the P
// per-path row segments of the CTA's TP-pixel tile into shared memory with
// one-dimensional bulk async copies (cp.async.bulk, mbarrier completion: the
// whole tile is in flight at once, no load instructions), then every thread
// owns one pixel: its P x NW words are summed into 2*NW exact u16x2 level
// pairs in registers and select_disparity's rules are applied with packed
// min / compare instructions.  Identical results to k_wta_tiled (parity
// dumps keep that kernel).
namespace {

__device__ __forceinline__ uint32_t wta_smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NW>
struct WtaGeo {
#ifndef RPD_WTA_TP_SMALL
#define RPD_WTA_TP_SMALL 128  // pixels per CTA, <= 9 words per pixel
#endif
#ifndef RPD_WTA_TP_BIG
#define RPD_WTA_TP_BIG 64     // pixels per CTA, wider layouts
#endif
  static constexpr int TP = NW <= 9 ? RPD_WTA_TP_SMALL : RPD_WTA_TP_BIG;  // pixels per CTA
  static constexpr int V = NW % 4 == 0 ? 4 : (NW % 2 == 0 ? 2 : 1);  // words per LDS
  static constexpr int NP = 2 * NW;                              // u16x2 level pairs
};

}  // namespace

struct WtaBulkArgs {
  const uint8_t* path[2][8];
  float* disp[2];
  int w;
  size_t pitch;
  int lw, levels;
};

// LV > 0: the level count is a compile-time constant (the pipeline's passes),
// so the padding masks and the loops over the level pairs fold away.
template <int P, int NW, int LV>
__global__ void __launch_bounds__(WtaGeo<NW>::TP) k_wta_bulk(const __grid_constant__ WtaBulkArgs a) {
  using GE = WtaGeo<NW>;
  constexpr int TP = GE::TP, V = GE::V, NP = GE::NP;
  extern __shared__ __align__(16) uint32_t tile[];  // [P][TP * NW] words
  __shared__ __align__(8) uint64_t bar;
  const int vol = blockIdx.z;
  const int row = blockIdx.y;
  const int u0 = blockIdx.x * TP;
  const int npx = min(TP, a.w - u0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wta_smem_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // row segments start 16-byte aligned (pitch and u0 * lw are multiples of
    // 16); the size is rounded up to 16 inside the row pitch
    const uint32_t bytes = uint32_t(npx * NW * 4 + 15) & ~15u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(wta_smem_addr(&bar)),
                 "r"(bytes * P)
                 : "memory");
    const size_t off = size_t(row) * a.pitch + size_t(u0) * (NW * 4);
#ifndef RPD_WTA_L2_HINT
#define RPD_WTA_L2_HINT 1  // 1: the path tiles are loaded evict_first (read once)
#endif
#if RPD_WTA_L2_HINT
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
    for (int r = 0; r < P; ++r)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              wta_smem_addr(tile + r * (TP * NW))),
          "l"(a.path[vol][r] + off), "r"(bytes), "r"(wta_smem_addr(&bar)), "l"(pol)
          : "memory");
#else
#pragma unroll
    for (int r = 0; r < P; ++r)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              wta_smem_addr(tile + r * (TP * NW))),
          "l"(a.path[vol][r] + off), "r"(bytes), "r"(wta_smem_addr(&bar))
          : "memory");
#endif
  }
#ifndef RPD_WTA_WAIT_ONE
#define RPD_WTA_WAIT_ONE 1  // 1: one thread polls the mbarrier, the others block at the CTA barrier
#endif
  // One thread observes the completion (acquire) and the CTA barrier orders
  // every thread's reads after it; the other warps wait at the barrier
  // without issuing instructions (all threads polling cost 17 % of the
  // kernel's issued instructions).
  if (!RPD_WTA_WAIT_ONE || threadIdx.x == 0)
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WTA_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        "@!p bra WTA_WAIT_%=;\n"
        "}\n" ::"r"(wta_smem_addr(&bar))
        : "memory");
  if (RPD_WTA_WAIT_ONE) __syncthreads();
  const int t = threadIdx.x;
  if (t >= npx) return;
  // exact per-level sums over the P paths, two levels per u16x2 word
  uint32_t s[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) s[q] = 0u;
  constexpr int NPS = LV > 0 ? (LV + 1) / 2 : NP;  // pairs that can hold levels < L
#pragma unroll
  for (int r = 0; r < P; r += 2) {
    const uint32_t* pa = tile + r * (TP * NW) + t * NW;
    const uint32_t* pb = pa + TP * NW;
#pragma unroll
    for (int j = 0; j < NW; j += V) {
      if (2 * j >= NPS) break;  // words of padding levels only
      uint32_t xa[V], xb[V];
      if constexpr (V == 4) {
        const uint4 ua = *reinterpret_cast<const uint4*>(pa + j);
        const uint4 ub = *reinterpret_cast<const uint4*>(pb + j);
        xa[0] = ua.x; xa[1] = ua.y; xa[2] = ua.z; xa[3] = ua.w;
        xb[0] = ub.x; xb[1] = ub.y; xb[2] = ub.z; xb[3] = ub.w;
      } else if constexpr (V == 2) {
        const uint2 ua = *reinterpret_cast<const uint2*>(pa + j);
        const uint2 ub = *reinterpret_cast<const uint2*>(pb + j);
        xa[0] = ua.x; xa[1] = ua.y;
        xb[0] = ub.x; xb[1] = ub.y;
      } else {
        xa[0] = pa[j];
        xb[0] = pb[j];
      }
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const int q = 2 * (j + e);
        if (q < NPS)
          s[q] = s[q] + __byte_perm(xa[e], 0u, 0x4140) + __byte_perm(xb[e], 0u, 0x4140);
        if (q + 1 < NPS)
          s[q + 1] = s[q + 1] + __byte_perm(xa[e], 0u, 0x4342) + __byte_perm(xb[e], 0u, 0x4342);
      }
    }
  }
  // select_disparity (sgm.cpp:123-153): minimum, its FIRST level, its
  // multiplicity and the sums at best -+ 1, over the levels < L only
  const int L = LV > 0 ? LV : a.levels;
  const int np = (L + 1) >> 1;
  const uint32_t hpad = (L & 1) ? 0xFFFF0000u : 0u;  // invalid high half of the last pair
  constexpr int NPE = NPS;
#pragma unroll
  for (int q = 0; q < NPE; ++q) s[q] = q < np ? (s[q] | (q == np - 1 ? hpad : 0u)) : 0xFFFFFFFFu;
  uint32_t m2 = 0xFFFFFFFFu;
#pragma unroll
  for (int q = 0; q < NPE; q += 2) m2 = __vimin3_u16x2(m2, s[q], q + 1 < NPE ? s[q + 1] : 0xFFFFFFFFu);
  const uint32_t minv = min(m2 & 0xFFFFu, m2 >> 16);
  const uint32_t mx2 = minv * 0x10001u;
  // per pair: e = min(s - min, 1) per half (no borrow: s >= min in both
  // halves), i.e. 0 where a level attains the minimum, 1 elsewhere
  int ne = 0, bq = 0, bh = 0;
#pragma unroll
  for (int q = NPE - 1; q >= 0; --q) {  // descending: the last hit is the first level
    const uint32_t e = __vminu2(s[q] - mx2, 0x00010001u);
    ne += __popc(e);
    if (e != 0x00010001u) {
      bq = q;
      bh = int(e & 1u);
    }
  }
  const int cnt = 2 * NPE - ne;
  const int best = 2 * bq + bh;
  // the sums at best -+ 1 through shared memory: this thread's own words of
  // paths 0 and 1 (2 * NW = NP words, read by nobody else) take its pairs
  uint32_t* own0 = tile + t * NW;
  uint32_t* own1 = own0 + TP * NW;
#pragma unroll
  for (int q = 0; q < NP; ++q) (q < NW ? own0[q] : own1[q - NW]) = s[q];
  auto pair_at = [&](int q) { return q < NW ? own0[q] : own1[q - NW]; };
  const int qm = (best - 1) >> 1, qp = (best + 1) >> 1;
  const uint32_t sbm1 = best > 0 ? ((pair_at(qm) >> (16 * ((best - 1) & 1))) & 0xFFFFu) : 0u;
  const uint32_t sbp1 = best + 1 < L ? ((pair_at(qp) >> (16 * ((best + 1) & 1))) & 0xFFFFu) : 0u;
  const int near = (best + 1 < L && sbp1 == minv) ? 1 : 0;
  float res;
  if (cnt - 1 - near > 0) {
    res = kInvalid;
  } else {
    res = float(best);
    if (best > 0 && best < L - 1) {
      const float cm = float(sbm1), cb = float(minv), cp = float(sbp1);
      const float denom = cm + cp - 2.0f * cb;
      if (denom > 0.0f) res += (cm - cp) / (2.0f * denom);
    }
  }
  a.disp[vol][(long long)row * a.w + u0 + t] = res;
}

namespace {
using WtaBulkKernel = void (*)(WtaBulkArgs);
struct WtaBulkInfo {
  WtaBulkKernel fn = nullptr;
  int tp = 0;
  int smem = 0;
};

template <int P, int NW, int LV = 0>
WtaBulkInfo wta_bulk_info() {
  return WtaBulkInfo{k_wta_bulk<P, NW, LV>, WtaGeo<NW>::TP, P * WtaGeo<NW>::TP * NW * 4};
}

template <int P>
WtaBulkInfo wta_bulk_pick(int nw, int levels) {
  // compile-time level counts of the pipeline's passes: PT (d_max_pt = 16)
  // and the bootstrap of D = 64 / 128 / 256, in their sgm_layout word counts
  if (nw == 5 && levels == 17) return wta_bulk_info<P, 5, 17>();
  if (nw == 9 && levels == 33) return wta_bulk_info<P, 9, 33>();
  if (nw == 20 && levels == 65) return wta_bulk_info<P, 20, 65>();
  if (nw == 17 && levels == 65) return wta_bulk_info<P, 17, 65>();
  if (nw == 36 && levels == 129) return wta_bulk_info<P, 36, 129>();
  switch (nw) {
    case 1: return wta_bulk_info<P, 1>();
    case 2: return wta_bulk_info<P, 2>();
    case 3: return wta_bulk_info<P, 3>();
    case 4: return wta_bulk_info<P, 4>();
    case 5: return wta_bulk_info<P, 5>();
    case 6: return wta_bulk_info<P, 6>();
    case 7: return wta_bulk_info<P, 7>();
    case 8: return wta_bulk_info<P, 8>();
    case 9: return wta_bulk_info<P, 9>();
    case 17: return wta_bulk_info<P, 17>();
    case 20: return wta_bulk_info<P, 20>();
    case 24: return wta_bulk_info<P, 24>();
    case 28: return wta_bulk_info<P, 28>();
    case 32: return wta_bulk_info<P, 32>();
    case 36: return wta_bulk_info<P, 36>();
    default: return WtaBulkInfo{};
  }
}

// Both volumes of a pass; false when the layout has no bulk instantiation.
bool launch_wta_bulk(const WtaBulkArgs& wa, int paths, int h, int w, cudaStream_t st) {
  if (debug_knob("RPD_WTA_TILED")) return false;  // A/B: the previous two-launch WTA
  const int nw = wa.lw / 4;
  const WtaBulkInfo ki = paths == 8   ? wta_bulk_pick<8>(nw, wa.levels)
                         : paths == 4 ? wta_bulk_pick<4>(nw, wa.levels)
                                      : WtaBulkInfo{};
  if (!ki.fn) return false;
#ifndef RPD_WTA_SMEM_MIN
#define RPD_WTA_SMEM_MIN 0  // experiment: request at least this much shared memory per CTA (caps CTAs/SM)
#endif
  const int wsmem = std::max(ki.smem, RPD_WTA_SMEM_MIN);
  RPD_CK(cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, wsmem));
  ki.fn<<<dim3(cdiv(w, ki.tp), h, 2), ki.tp, wsmem, st>>>(wa);
  RPD_LAUNCH_CHECK();
  return true;
}
}  // namespace

// ------------------------------------------- LR check + post filters ----
// consistency_filter (sgm.cpp:155-170), flat raw cost curve (:200-212),
// best sample out of view (:216-222), restore_disparity (perspective.hpp:69-80).
template <typename CostT>
__global__ void k_post(const float* __restrict__ dl, const float* __restrict__ dr,
                       const CostT* __restrict__ cost, int cstride, size_t crow,
                       const uint8_t* __restrict__ iv, const double* __restrict__ shifts, int h,
                       int w, int levels, double thr, float* __restrict__ d0,
                       float* __restrict__ d1) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= w) return;
  for (int v = blockIdx.y; v < h; v += gridDim.y) {  // rows strided over gridDim.y
    const size_t i = size_t(v) * w + u;
    const size_t coff = size_t(v) * crow + size_t(u) * cstride;  // element offset of the cost curve
    const size_t row = size_t(v) * w;
    float d = dl[i];
    if (d != kInvalid) {
      const int ur = u - int(lroundf(d));
      if (ur < 0 || ur >= w) {
        d = kInvalid;
      } else {
        const float x = dr[row + ur];
        if (x == kInvalid || double(fabsf(d - x)) > thr) d = kInvalid;
      }
    }
    if (d != kInvalid) {
      float lo = FLT_MAX, hi = -FLT_MAX;
      const CostT* c = cost + coff;
      for (int k = 0; k < levels; ++k) {
        const int ur = u - k;
        if (ur < 0) break;
        if (!iv[row + ur]) continue;
        const float x = float(c[k]);
        lo = (x < lo) ? x : lo;
        hi = (hi < x) ? x : hi;
        if (lo < hi) break;
      }
      if (hi <= lo) d = kInvalid;
    }
    if (d != kInvalid) {
      const int ur = u - int(lroundf(d));
      if (ur < 0 || !iv[row + ur]) d = kInvalid;
    }
    d0[i] = d;
    d1[i] = (d != kInvalid) ? d + float(shifts[v]) : d;
  }
}

// ------------------------------------------------------ generic float path --
// One thread per chain start (pixel whose predecessor is outside the image)
// walking the chain; prev values are read back from `line`, as sgm.cpp:84-105.
__global__ void k_agg_f32_dir(const float* __restrict__ raw, float* __restrict__ line,
                              float* __restrict__ total, int h, int w, int n, int du, int dv,
                              float l1, float l2, int first) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= (long long)h * w) return;
  int v = int(p / w), u = int(p % w);
  if (!(v - dv < 0 || v - dv >= h || u - du < 0 || u - du >= w)) return;
  bool head = true;
  while (v >= 0 && v < h && u >= 0 && u < w) {
    const size_t base = (size_t(v) * w + u) * n;
    const float* c = raw + base;
    float* cur = line + base;
    float* tot = total + base;
    if (head) {
      for (int d = 0; d < n; ++d) {
        cur[d] = c[d];
        tot[d] = first ? cur[d] : tot[d] + cur[d];
      }
      head = false;
    } else {
      const float* prev = line + (size_t(v - dv) * w + (u - du)) * n;
      float mn = prev[0];
      for (int d = 1; d < n; ++d) mn = (prev[d] < mn) ? prev[d] : mn;
      const float cap = mn + l2;
      for (int d = 0; d < n; ++d) {
        float b = prev[d];
        if (d > 0) { const float x = prev[d - 1] + l1; b = (x < b) ? x : b; }
        if (d + 1 < n) { const float x = prev[d + 1] + l1; b = (x < b) ? x : b; }
        b = (cap < b) ? cap : b;
        cur[d] = c[d] + b - mn;
        tot[d] = first ? cur[d] : tot[d] + cur[d];
      }
    }
    v += dv;
    u += du;
  }
}

void aggregate_f32(rpd_ctx* ctx, const float* costs, int h, int w, int levels,
                   const int32_t* dirs, int ndirs, float l1, float l2, float* out) {
  const long long npix = (long long)h * w;
  float* line = ctx->ws.get<float>("agg_f32_line", size_t(npix) * levels);
  if (ndirs == 0) {
    RPD_CK(cudaMemsetAsync(out, 0, sizeof(float) * size_t(npix) * levels, ctx->stream));
    return;
  }
  for (int r = 0; r < ndirs; ++r) {
    const int du = dirs[2 * r], dv = dirs[2 * r + 1];
    if (du == 0 && dv == 0) throw InvalidArg("aggregate_costs: zero direction");
    k_agg_f32_dir<<<cdiv(npix, 128), 128, 0, ctx->stream>>>(costs, line, out, h, w, levels, du,
                                                            dv, l1, l2, r == 0);
    RPD_LAUNCH_CHECK();
  }
}

__global__ void k_select_f32(const float* __restrict__ agg, long long npix, int n,
                             float* __restrict__ disp) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= npix) return;
  const float* c = agg + p * n;
  int best = 0;
  for (int d = 1; d < n; ++d)
    if (c[d] < c[best]) best = d;
  bool amb = false;
  for (int d = 0; d < n; ++d)
    if (abs(d - best) > 1 && c[d] <= c[best]) amb = true;
  if (amb) {
    disp[p] = kInvalid;
    return;
  }
  float r = float(best);
  if (best > 0 && best < n - 1) {
    const float denom = c[best - 1] + c[best + 1] - 2.0f * c[best];
    if (denom > 0.0f) r += (c[best - 1] - c[best + 1]) / (2.0f * denom);
  }
  disp[p] = r;
}

void select_disparity_f32(const float* agg, int h, int w, int levels, float* disp,
                          cudaStream_t st) {
  const long long npix = (long long)h * w;
  k_select_f32<<<cdiv(npix, 128), 128, 0, st>>>(agg, npix, levels, disp);
  RPD_LAUNCH_CHECK();
}

__global__ void k_swap_f32(const float* __restrict__ in, const float* __restrict__ maxv, int h,
                           int w, int n, float* __restrict__ out) {
  const long long total = (long long)h * w * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = int(i % n);
    const long long p = i / n;
    const int u = int(p % w);
    out[i] = (u + d < w) ? in[(p + d) * n + d] : *maxv;
  }
}

void swap_reference_f32(rpd_ctx* ctx, const float* costs, int h, int w, int levels, float* out) {
  const long long total = (long long)h * w * levels;
  float* maxv = ctx->ws.get<float>("swap_max", 1);
  size_t tmp_bytes = 0;
  cub::DeviceReduce::Max(nullptr, tmp_bytes, costs, maxv, total, ctx->stream);
  void* tmp = ctx->ws.get<uint8_t>("cub_tmp_swap", tmp_bytes);
  cub::DeviceReduce::Max(tmp, tmp_bytes, costs, maxv, total, ctx->stream);
  RPD_LAUNCH_CHECK();
  const int blocks = int(std::min<long long>((total + 255) / 256, 148 * 32));
  k_swap_f32<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(costs, maxv, h, w, levels, out);
  RPD_LAUNCH_CHECK();
}

__global__ void k_lr_only(float* __restrict__ left, const float* __restrict__ right, int h, int w,
                          double thr) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  if (u >= w) return;
  const size_t i = size_t(v) * w + u;
  const float d = left[i];
  if (d == kInvalid) return;
  const int ur = u - int(lroundf(d));
  if (ur < 0 || ur >= w) {
    left[i] = kInvalid;
    return;
  }
  const float x = right[size_t(v) * w + ur];
  if (x == kInvalid || double(fabsf(d - x)) > thr) left[i] = kInvalid;
}

void consistency_filter_dev(float* left, const float* right, int h, int w, double thr,
                            cudaStream_t st) {
  k_lr_only<<<dim3(cdiv(w, 128), h), 128, 0, st>>>(left, right, h, w, thr);
  RPD_LAUNCH_CHECK();
}

// ------------------------------------------------------------ match_pair ---
void match_pair_dev(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                    const DevModel* model, const rpd_config& cfg, int d_max, float* d0,
                    float* d1, double* shifts, const MatchDump* dump) {
  if (w < 2) throw InvalidArg("compute_row_shifts: width must be >= 2");
  if (cfg.census_window % 2 == 0 || cfg.census_window < 3 || cfg.census_window > 7)
    throw InvalidArg("census_cost_volume: window must be odd");
  if (d_max >= w) throw InvalidArg("census_cost_volume: d_max >= width");
  if (d_max < 0) throw InvalidArg("census_cost_volume: d_max must be >= 0");
  cudaStream_t st = ctx->stream;
  const long long npix = (long long)h * w;
  const int levels = d_max + 1;
  const int window = cfg.census_window;
  const float l1 = float(cfg.lambda1), l2 = float(cfg.lambda2);

  launch_row_shifts(model, h, w, cfg.delta_pt, shifts, st);
  float* warped = ctx->ws.get<float>("mp_warped", npix);
  uint8_t* iv = ctx->ws.get<uint8_t>("mp_inview", npix);
  launch_warp_right(right, shifts, h, w, warped, iv, st);
  uint64_t* cl = ctx->ws.get<uint64_t>("mp_census_l", npix);
  uint64_t* cr = ctx->ws.get<uint64_t>("mp_census_r", npix);
  launch_census2(left, warped, h, w, window, cl, cr, st);
  float* dl = ctx->ws.get<float>("mp_disp_l", npix);
  float* dr = ctx->ws.get<float>("mp_disp_r", npix);
  const dim3 rowgrid(cdiv(w, 128), std::max(1, cdiv(h, 4)));  // k_post strides rows over gridDim.y
  int32_t dirs[16];
  const int paths = cfg.sgm_paths == 4 ? 4 : 8;
  const int eight[16] = {1, 0, -1, 0, 0, 1, 0, -1, 1, 1, -1, 1, 1, -1, -1, -1};
  for (int i = 0; i < 2 * paths; ++i) dirs[i] = eight[i];

  if (!sgm_fast_path_ok(l1, l2, window) || levels > kMaxFastLevels) {
    // generic float path (non-integral or very large penalties)
    ctx->last_agg_kernel = kAggF32;
    float* cost = ctx->ws.get<float>("mp_cost_f32", size_t(npix) * levels);
    float* costr = ctx->ws.get<float>("mp_costr_f32", size_t(npix) * levels);
    float* agg = ctx->ws.get<float>("mp_agg_f32", size_t(npix) * levels);
    launch_cost_f32(cl, cr, iv, h, w, levels, window, cost, st);
    aggregate_f32(ctx, cost, h, w, levels, dirs, paths, l1, l2, agg);
    if (dump && dump->agg_left)
      RPD_CK(cudaMemcpyAsync(dump->agg_left, agg, sizeof(float) * npix * levels,
                             cudaMemcpyDeviceToDevice, st));
    select_disparity_f32(agg, h, w, levels, dl, st);
    swap_reference_f32(ctx, cost, h, w, levels, costr);
    if (dump && dump->cost_right)
      RPD_CK(cudaMemcpyAsync(dump->cost_right, costr, sizeof(float) * npix * levels,
                             cudaMemcpyDeviceToDevice, st));
    aggregate_f32(ctx, costr, h, w, levels, dirs, paths, l1, l2, agg);
    if (dump && dump->agg_right)
      RPD_CK(cudaMemcpyAsync(dump->agg_right, agg, sizeof(float) * npix * levels,
                             cudaMemcpyDeviceToDevice, st));
    select_disparity_f32(agg, h, w, levels, dr, st);
    if (dump && dump->cost)
      RPD_CK(cudaMemcpyAsync(dump->cost, cost, sizeof(float) * npix * levels,
                             cudaMemcpyDeviceToDevice, st));
    k_post<float><<<rowgrid, 128, 0, st>>>(dl, dr, cost, levels, size_t(w) * levels, iv, shifts,
                                           h, w, levels, cfg.lr_threshold, d0, d1);
    RPD_LAUNCH_CHECK();
  } else {
    const SgmLayout L = sgm_layout(h, w, levels, paths);
    const int nw = L.lw / 4;
    const size_t vb = L.vol_bytes();
    uint8_t* vol_l = ctx->ws.get<uint8_t>("mp_vols", 2 * vb);
    uint8_t* vol_r = vol_l + vb;
    uint8_t* pathbuf = ctx->ws.get<uint8_t>("mp_paths", vb * 2 * paths);
    {
      const bool narrow = window * window - 1 <= 32;
      const int smem = (w + 2 * levels) * (narrow ? 9 : 17);
      const CostPxKernel pxfn = window <= 5 ? cost_px_pick(nw, levels) : nullptr;
      const int pxsmem = (w + 8 * nw) * 16 + 2 * 256 * nw * 4;
      if (pxfn && pxsmem <= 200 * 1024 && !debug_knob("RPD_COST_ROWS")) {
        if (pxsmem > 48 * 1024)
          RPD_CK(cudaFuncSetAttribute(pxfn, cudaFuncAttributeMaxDynamicSharedMemorySize, pxsmem));
        pxfn<<<h, 256, pxsmem, st>>>(cl, cr, iv, w, levels, L.pitch / 4, uint32_t(window * window - 1),
                                     reinterpret_cast<uint32_t*>(vol_l),
                                     reinterpret_cast<uint32_t*>(vol_r));
      } else if (smem <= 200 * 1024) {
        auto* kfn = narrow ? k_cost_u8<uint32_t> : k_cost_u8<uint64_t>;
        if (smem > 48 * 1024)
          RPD_CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        kfn<<<dim3(1, h), 256, smem, st>>>(
            cl, cr, iv, h, w, levels, nw, L.pitch / 4, uint32_t(window * window - 1),
            reinterpret_cast<uint32_t*>(vol_l), reinterpret_cast<uint32_t*>(vol_r));
      } else {
        const long long n = npix * nw;
        const int blocks = int(std::min<long long>((n + 255) / 256, 148 * 32));
        k_cost_u8_flat<<<std::max(blocks, 1), 256, 0, st>>>(
            cl, cr, iv, h, w, levels, nw, L.pitch / 4, uint32_t(window * window - 1),
            reinterpret_cast<uint32_t*>(vol_l), reinterpret_cast<uint32_t*>(vol_r));
      }
      RPD_LAUNCH_CHECK();
    }
    const uint32_t p1 = uint32_t(l1), p2 = uint32_t(l2);
    const int pass = ctx->agg_pass;
    const bool prof = ctx->profile && pass < 2;
    if (prof) record_event(ctx, ctx->agg_ev[pass][0]);
    if (sgm_tma_supported(L)) {
      launch_aggregate_tma(ctx, L, vol_l, pathbuf, dirs, paths, p1, p2);
      ctx->last_agg_kernel = kAggU8Tma;
    } else {
      ctx->last_agg_kernel = kAggU8;
      AggArgs args{};
      args.h = h;
      args.w = w;
      args.lw = L.lw;
      args.pitch = L.pitch;
      args.p1x2 = p1 | (p1 << 16);
      args.p2x2 = p2 | (p2 << 16);
      const int cpb = kAggThreads / L.G;
      int blocks = 0;
      for (int vol = 0; vol < 2; ++vol)
        for (int r = 0; r < paths; ++r) {
          AggJob& J = args.job[args.njobs];
          J.cost = vol == 0 ? vol_l : vol_r;
          J.out = pathbuf + size_t(vol * paths + r) * vb;
          J.du = dirs[2 * r];
          J.dv = dirs[2 * r + 1];
          J.nchains = (J.dv == 0) ? h : w;
          J.block0 = blocks;
          blocks += cdiv(J.nchains, cpb);
          ++args.njobs;
        }
      agg_kernel(L.wpl, L.G)<<<blocks, kAggThreads, 0, st>>>(args);
      RPD_LAUNCH_CHECK();
    }
    if (prof) {
      record_event(ctx, ctx->agg_ev[pass][1]);
      const double cells = double(npix) * levels;
      ctx->agg_alg_bytes[pass] = 2.0 * (5.0 * paths - 2.0) * cells;
      ctx->agg_cells[pass] = cells;
      ctx->agg_pass = pass + 1;
    }
    bool wta_done = false;
    if (!dump) {
      WtaBulkArgs wb{};
      for (int vol = 0; vol < 2; ++vol)
        for (int r = 0; r < paths; ++r) wb.path[vol][r] = pathbuf + size_t(vol * paths + r) * vb;
      wb.disp[0] = dl;
      wb.disp[1] = dr;
      wb.w = w;
      wb.pitch = L.pitch;
      wb.lw = L.lw;
      wb.levels = levels;
      wta_done = launch_wta_bulk(wb, paths, h, w, st);
    }
    for (int vol = 0; vol < 2 && !wta_done; ++vol) {
      WtaArgs wa{};
      for (int r = 0; r < paths; ++r) wa.path[r] = pathbuf + size_t(vol * paths + r) * vb;
      wa.paths = paths;
      wa.npix = npix;
      wa.w = w;
      wa.pitch = L.pitch;
      wa.lw = L.lw;
      wa.levels = levels;
      wa.disp = vol == 0 ? dl : dr;
      wa.dump = dump ? (vol == 0 ? dump->agg_left : dump->agg_right) : nullptr;
      if (L.lw / 4 <= kWtaMaxWords) {
        const int smem = kWtaPx * (2 * (L.lw / 4) + 1) * 4;
        if (wa.paths == 8)
          k_wta_tiled<8><<<dim3(cdiv(w, kWtaPx), h), kWtaPx, smem, st>>>(wa);
        else
          k_wta_tiled<4><<<dim3(cdiv(w, kWtaPx), h), kWtaPx, smem, st>>>(wa);
      } else {
        k_wta<<<cdiv(npix, 128), 128, 0, st>>>(wa);
      }
      RPD_LAUNCH_CHECK();
    }
    if (dump && (dump->cost || dump->cost_right)) {
      const long long n = npix * levels;
      const int nb = int(std::min<long long>((n + 255) / 256, 148 * 32));
      if (dump->cost)
        k_u8vol_to_f32<<<nb, 256, 0, st>>>(vol_l, w, npix, L.pitch, L.lw, levels, dump->cost);
      if (dump->cost_right)  // the right-reference volume the cost kernel generated
        k_u8vol_to_f32<<<nb, 256, 0, st>>>(vol_r, w, npix, L.pitch, L.lw, levels,
                                           dump->cost_right);
      RPD_LAUNCH_CHECK();
    }
    k_post<uint8_t><<<rowgrid, 128, 0, st>>>(dl, dr, vol_l, L.lw, L.pitch, iv, shifts, h, w,
                                             levels, cfg.lr_threshold, d0, d1);
    RPD_LAUNCH_CHECK();
  }
  if (dump && dump->disp_left)
    RPD_CK(cudaMemcpyAsync(dump->disp_left, dl, sizeof(float) * npix, cudaMemcpyDeviceToDevice,
                           st));
  if (dump && dump->disp_right)
    RPD_CK(cudaMemcpyAsync(dump->disp_right, dr, sizeof(float) * npix, cudaMemcpyDeviceToDevice,
                           st));
}


// ------------------------------------------- aggregate_costs, u8 route ----
bool aggregate_u8_eligible(const float* costs, size_t cells, int levels, const int32_t* dirs,
                           int ndirs, float l1, float l2, int* paths) {
  if (!(l1 >= 1.0f && l2 >= l1 && l1 == std::floor(l1) && l2 == std::floor(l2)))
    return false;
  if (levels > kMaxFastLevels) return false;
  // direction set = first 4 or all 8 of kEightDirections (sum order is
  // irrelevant: every partial sum is an exact integer)
  const int eight[16] = {1, 0, -1, 0, 0, 1, 0, -1, 1, 1, -1, 1, 1, -1, -1, -1};
  if (ndirs != 4 && ndirs != 8) return false;
  bool seen[8] = {};
  for (int i = 0; i < ndirs; ++i) {
    int k = 0;
    while (k < ndirs && !(eight[2 * k] == dirs[2 * i] && eight[2 * k + 1] == dirs[2 * i + 1])) ++k;
    if (k == ndirs || seen[k]) return false;
    seen[k] = true;
  }
  float mx = 0.0f;
  for (size_t i = 0; i < cells; ++i) {
    const float c = costs[i];
    if (!(c >= 0.0f) || c != std::floor(c)) return false;
    mx = std::max(mx, c);
  }
  if (mx + l2 > 255.0f) return false;  // every path value fits u8
  *paths = ndirs;
  return true;
}

void aggregate_u8_dev(rpd_ctx* ctx, const float* costs, int h, int w, int levels, int paths,
                      float l1, float l2, float* out) {
  cudaStream_t st = ctx->stream;
  const long long npix = (long long)h * w;
  const SgmLayout L = sgm_layout(h, w, levels, paths);
  const size_t vb = L.vol_bytes();
  uint8_t* vol = ctx->ws.get<uint8_t>("ag_vols", 2 * vb);  // TMA maps span two planes
  uint8_t* pathbuf = ctx->ws.get<uint8_t>("ag_paths", vb * paths);
  float* disp = ctx->ws.get<float>("ag_disp", npix);
  {
    const long long n = npix * L.lw;
    k_f32_to_u8vol<<<int(std::min<long long>((n + 255) / 256, 148 * 32)), 256, 0, st>>>(
        costs, w, npix, L.pitch, L.lw, levels, vol);
    RPD_LAUNCH_CHECK();
  }
  const int eight[16] = {1, 0, -1, 0, 0, 1, 0, -1, 1, 1, -1, 1, 1, -1, -1, -1};
  int32_t dirs[16];
  for (int i = 0; i < 2 * paths; ++i) dirs[i] = eight[i];
  const uint32_t p1 = uint32_t(l1), p2 = uint32_t(l2);
  if (sgm_tma_supported(L)) {
    launch_aggregate_tma(ctx, L, vol, pathbuf, dirs, paths, p1, p2, /*nvols=*/1);
    ctx->last_agg_kernel = kAggU8Tma;
  } else {
    AggArgs args{};
    args.h = h;
    args.w = w;
    args.lw = L.lw;
    args.pitch = L.pitch;
    args.p1x2 = p1 | (p1 << 16);
    args.p2x2 = p2 | (p2 << 16);
    const int cpb = kAggThreads / L.G;
    int blocks = 0;
    for (int r = 0; r < paths; ++r) {
      AggJob& J = args.job[args.njobs++];
      J.cost = vol;
      J.out = pathbuf + size_t(r) * vb;
      J.du = dirs[2 * r];
      J.dv = dirs[2 * r + 1];
      J.nchains = (J.dv == 0) ? h : w;
      J.block0 = blocks;
      blocks += cdiv(J.nchains, cpb);
    }
    agg_kernel(L.wpl, L.G)<<<blocks, kAggThreads, 0, st>>>(args);
    RPD_LAUNCH_CHECK();
    ctx->last_agg_kernel = kAggU8;
  }
  // exact u16 sums over the paths, written in the reference float layout
  WtaArgs wa{};
  for (int r = 0; r < paths; ++r) wa.path[r] = pathbuf + size_t(r) * vb;
  wa.paths = paths;
  wa.npix = npix;
  wa.w = w;
  wa.pitch = L.pitch;
  wa.lw = L.lw;
  wa.levels = levels;
  wa.disp = disp;
  wa.dump = out;
  if (L.lw / 4 <= kWtaMaxWords) {
    const int smem = kWtaPx * (2 * (L.lw / 4) + 1) * 4;
    if (paths == 8)
      k_wta_tiled<8><<<dim3(cdiv(w, kWtaPx), h), kWtaPx, smem, st>>>(wa);
    else
      k_wta_tiled<4><<<dim3(cdiv(w, kWtaPx), h), kWtaPx, smem, st>>>(wa);
  } else {
    k_wta<<<cdiv(npix, 128), 128, 0, st>>>(wa);
  }
  RPD_LAUNCH_CHECK();
}

}  // namespace rpdg
