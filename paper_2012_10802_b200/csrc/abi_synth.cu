// abi_synth.cu — the reference scene generator on the device (synth.cpp:16-196;
// SURVEY.md §8(f) row 4): generate_scene / scene_batch with the reference's
// random streams, so a device-generated scene equals the reference's
// bit for bit and streaming runs need no host generation.
//
// Per batch of scenes (same W x H), four launches on the context stream:
//   k_mt_streams  one CTA per (scene, stream): the texture lattice stream
//                 (std::mt19937(seed), synth.cpp:61) and the noise stream
//                 (mt19937(seed ^ 0x9e3779b9), :140) — mt19937 in rounds of
//                 620 words (synth_rng.cuh), uniform floats for the lattice,
//                 polar attempts accepted and compacted in order for the noise;
//   k_truth       plane + elliptic-paraboloid dips, mask, negativity flag (:103-121);
//   k_texture     3 value-noise octaves + separable 5x5 binomial smoothing in
//                 32 x 16 tiles with a 2-pixel halo in shared memory, block
//                 min / max for the normalisation (:16-72);
//   k_views       normalised left, fixed-point right-view warp (:126-137),
//                 additive noise clamped to [0, 255] (:139-146).
// Every expression keeps the reference's operation order (the library is
// built with --fmad=false), so no tolerance is involved; the only ulp-level
// difference is glibc's log (<= 0.52 ulp) vs the correctly rounded log_dd,
// which reaches a noise double in ~4e-4 of pixels and a float pixel
// essentially never (tests/cpp/synth_rng_check.cpp).
#include <cmath>
#include <random>
#include <vector>

#include "abi_util.hpp"
#include "synth_rng.cuh"

using namespace rpdg;
using namespace rpd_synth;

namespace {

struct DevScene {
  double a0, a1, cphi, sphi;  // cos / sin of phi_true on the host (glibc), types.hpp:40
  double sigma;
  uint32_t seed;
  int pot_off, n_pot;
};

struct DevPothole {
  double cu, cv, ru, rv, depth;
};

// Lattice geometry of the three octaves (spacings 64, 16, 4; synth.cpp:62-64).
struct Lattice {
  int nu[3], nv[3], off[3], total;
};

Lattice lattice_of(int w, int h) {
  Lattice L;
  const int sp[3] = {64, 16, 4};
  int off = 0;
  for (int o = 0; o < 3; ++o) {
    L.nu[o] = w / sp[o] + 2;
    L.nv[o] = h / sp[o] + 2;
    L.off[o] = off;
    off += L.nu[o] * L.nv[o];
  }
  L.total = off;
  return L;
}

constexpr int kMtThreads = 640;
constexpr int kRing = 2048;  // > 1078 + 620: the oldest word a round reads plus one round

// The serial part: one CTA per (scene, stream) runs mt19937 in rounds of 620
// words with a single barrier per round (t[m] = twist(x[m], x[m+1]) is
// recomputed from the ring instead of stored).  The ring is mapped twice
// (word n at n mod 2048 and n mod 2048 + 2048), so every read x[n - c] is the
// thread's slot minus a constant: no index arithmetic in the loop.
// blockIdx.y = 0: the lattice stream -> lattice[scene][0..total) as uniform
// floats; blockIdx.y = 1: the noise stream -> its first `nwords` tempered
// outputs, consumed in parallel by k_polar_count / k_polar_scatter.
__global__ void __launch_bounds__(kMtThreads) k_mt_streams(const DevScene* scenes, int total,
                                                           float* lattice, uint32_t* words,
                                                           int nwords) {
  const DevScene s = scenes[blockIdx.x];
  const bool noise = blockIdx.y == 1;
  if (noise && !(s.sigma > 0)) return;
  __shared__ uint32_t X[2 * kRing];
  const int i = threadIdx.x;
  if (i == 0) {
    uint32_t v = noise ? (s.seed ^ 0x9e3779b9u) : s.seed;
    X[0] = X[kRing] = v;
    for (uint32_t k = 1; k < 624; ++k) X[k] = X[kRing + k] = v = mt_seed_next(v, k);
  }
  __syncthreads();
  const int limit = noise ? nwords : total;
  float* lat = lattice + (size_t)blockIdx.x * total;
  uint32_t* wo = words + (size_t)blockIdx.x * nwords;
  const bool live = i < kMtRound;
  int slot = (624 + i) & (kRing - 1);  // n mod 2048 of this thread's word
  for (int base = 624;; base += kMtRound) {
    const int n = base + i;
    if (live) {
      const uint32_t* h = X + kRing + slot;  // h[-c] = x[n - c]
      auto xs = [&](int k) { return h[k - n]; };
      auto ts = [&](int k) { return mt_twist(h[k - n], h[k + 1 - n]); };
      const uint32_t xn = mt_word(n, xs, ts);
      X[slot] = xn;
      X[slot + kRing] = xn;
      const int j = n - 624;  // output index
      if (j < limit) {
        const uint32_t o = mt_temper(xn);
        if (noise)
          wo[j] = o;
        else
          lat[j] = canonical_f32(o);
      }
    }
    slot = (slot + kMtRound) & (kRing - 1);
    __syncthreads();
    if (base - 624 + kMtRound >= limit) break;
  }
}

// Noise stream, parallel part: polar attempts (4 words each) accepted in
// order; pixel k takes the k-th accepted attempt (left = y m, right = x m).
constexpr int kPolarThreads = 256, kPolarPerThread = 4;
constexpr int kPolarPerBlock = kPolarThreads * kPolarPerThread;

__device__ __forceinline__ int polar_flags(const uint32_t* w, long long a0, long long attempts,
                                           double* px, double* py) {
  int mask = 0;
#pragma unroll
  for (int q = 0; q < kPolarPerThread; ++q) {
    const long long a = a0 + q;
    if (a >= attempts) break;
    const uint4 o = reinterpret_cast<const uint4*>(w)[a];
    if (polar_attempt(o.x, o.y, o.z, o.w, px[q], py[q])) mask |= 1 << q;
  }
  return mask;
}

__global__ void __launch_bounds__(kPolarThreads) k_polar_count(const DevScene* scenes,
                                                               const uint32_t* words,
                                                               long long nwords, int* counts) {
  const int b = blockIdx.y;
  if (!(scenes[b].sigma > 0)) return;
  const long long attempts = nwords / 4;
  const long long a0 = (long long)blockIdx.x * kPolarPerBlock + threadIdx.x * kPolarPerThread;
  double px[kPolarPerThread], py[kPolarPerThread];
  int c = __popc(polar_flags(words + (size_t)b * nwords, a0, attempts, px, py));
  for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  __shared__ int wsum[kPolarThreads / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < kPolarThreads / 32; ++k) t += wsum[k];
    counts[(size_t)b * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kPolarThreads) k_polar_scatter(
    const DevScene* scenes, const uint32_t* words, long long nwords, const int* counts,
    double2* pairs, long long need, int* exhausted) {
  const int b = blockIdx.y;
  if (!(scenes[b].sigma > 0)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ long long s_red[kPolarThreads / 32];
  __shared__ int s_scan[kPolarThreads / 32];
  // accepted attempts before this block
  const int* cnt = counts + (size_t)b * gridDim.x;
  long long before = 0;
  for (int k = tid; k < (int)blockIdx.x; k += kPolarThreads) before += cnt[k];
  for (int off = 16; off; off >>= 1) before += __shfl_xor_sync(0xffffffffu, before, off);
  if (lane == 0) s_red[warp] = before;
  const long long attempts = nwords / 4;
  const long long a0 = (long long)blockIdx.x * kPolarPerBlock + tid * kPolarPerThread;
  double px[kPolarPerThread], py[kPolarPerThread];
  const int mask = polar_flags(words + (size_t)b * nwords, a0, attempts, px, py);
  const int c = __popc(mask);
  int incl = c;  // warp inclusive scan
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) s_scan[warp] = incl;
  __syncthreads();
  long long base = 0;
  int wbase = 0;
  for (int k = 0; k < kPolarThreads / 32; ++k) {
    base += s_red[k];
    wbase += k < warp ? s_scan[k] : 0;
  }
  long long k = base + wbase + incl - c;
  double2* pr = pairs + (size_t)b * need;
#pragma unroll
  for (int q = 0; q < kPolarPerThread; ++q)
    if (mask & (1 << q)) {
      if (k < need) pr[k] = make_double2(px[q], py[q]);
      ++k;
    }
  if (blockIdx.x == gridDim.x - 1 && tid == kPolarThreads - 1 && k < need)
    atomicOr(exhausted, 1);  // the drawn words held fewer than `need` accepted attempts
}

// Ground truth (synth.cpp:103-121): gt disparity, mask, negativity flag.
__global__ void k_truth(const DevScene* scenes, const DevPothole* pots, int h, int w,
                        float* gt, int32_t* mask, int* negative) {
  const long long per = (long long)h * w;
  const int b = blockIdx.y;
  const DevScene s = scenes[b];
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < per;
       p += (long long)gridDim.x * blockDim.x) {
    const int v = int(p / w), u = int(p - (long long)v * w);
    double d = s.a0 + s.a1 * (v * s.cphi - u * s.sphi);
    int m = 0;
    for (int k = 0; k < s.n_pot; ++k) {
      const DevPothole q = pots[s.pot_off + k];
      const double ru = (u - q.cu) / q.ru;
      const double rv = (v - q.cv) / q.rv;
      const double r2 = ru * ru + rv * rv;
      if (r2 < 1.0) {
        d -= q.depth * (1.0 - r2);
        m = k + 1;
      }
    }
    if (d < 0) atomicOr(negative + b, 1);
    gt[b * per + p] = static_cast<float>(d);
    mask[b * per + p] = m;
  }
}

constexpr int kTexTW = 32, kTexTH = 16, kTexHalo = 2;
constexpr int kTexSW = kTexTW + 2 * kTexHalo, kTexSH = kTexTH + 2 * kTexHalo;

struct TexArgs {
  Lattice L;
  int h, w;
  const float* lattice;
  float* smooth;          // [scene][h*w], before normalisation
  unsigned* minmax;       // [scene][2]: float bits of min, max (all values >= 0)
};

// value_noise (synth.cpp:16-38) of octave o at (v, u).
__device__ __forceinline__ float value_noise(const TexArgs& a, const float* lat, int o, int sp,
                                             int v, int u) {
  const int nu = a.L.nu[o];
  const float* L = lat + a.L.off[o];
  const double y = static_cast<double>(v) / sp;
  const int j = static_cast<int>(y);
  const double ty = y - j;
  const double x = static_cast<double>(u) / sp;
  const int i = static_cast<int>(x);
  const double tx = x - i;
  const double l00 = L[j * nu + i], l01 = L[j * nu + i + 1];
  const double l10 = L[(j + 1) * nu + i], l11 = L[(j + 1) * nu + i + 1];
  return static_cast<float>((1 - ty) * ((1 - tx) * l00 + tx * l01) +
                            ty * ((1 - tx) * l10 + tx * l11));
}

// make_texture before the normalisation (synth.cpp:40-72).
__global__ void __launch_bounds__(256) k_texture(TexArgs a) {
  __shared__ float tex[kTexSH][kTexSW];
  __shared__ float tmp[kTexSH][kTexTW];
  const int b = blockIdx.z;
  const int u0 = blockIdx.x * kTexTW, v0 = blockIdx.y * kTexTH;
  const float* lat = a.lattice + (size_t)b * a.L.total;
  const int tid = threadIdx.x;
  // 3 octaves at clamped coordinates: tex(v, clamp(u + i)) of the smoothing
  for (int k = tid; k < kTexSH * kTexSW; k += 256) {
    const int r = k / kTexSW, c = k - r * kTexSW;
    const int v = min(max(v0 + r - kTexHalo, 0), a.h - 1);
    const int u = min(max(u0 + c - kTexHalo, 0), a.w - 1);
    float t = 0.0f;  // GrayImage::Zero, then tex += amps[o] * value_noise (:65)
    t = t + 1.0f * value_noise(a, lat, 0, 64, v, u);
    t = t + 0.5f * value_noise(a, lat, 1, 16, v, u);
    t = t + 0.25f * value_noise(a, lat, 2, 4, v, u);
    tex[r][c] = t;
  }
  __syncthreads();
  // horizontal pass (:46-51) on every staged row
  for (int k = tid; k < kTexSH * kTexTW; k += 256) {
    const int r = k / kTexTW, c = k - r * kTexTW;
    double s = 0;
    s += 1.0 * tex[r][c];
    s += 4.0 * tex[r][c + 1];
    s += 6.0 * tex[r][c + 2];
    s += 4.0 * tex[r][c + 3];
    s += 1.0 * tex[r][c + 4];
    tmp[r][c] = static_cast<float>(s / 16.0);
  }
  __syncthreads();
  // vertical pass (:52-57)
  float lo = 3.0e38f, hi = 0.0f;
  for (int k = tid; k < kTexTH * kTexTW; k += 256) {
    const int r = k / kTexTW, c = k - r * kTexTW;
    const int v = v0 + r, u = u0 + c;
    if (v >= a.h || u >= a.w) continue;
    double s = 0;
    s += 1.0 * tmp[r][c];
    s += 4.0 * tmp[r + 1][c];
    s += 6.0 * tmp[r + 2][c];
    s += 4.0 * tmp[r + 3][c];
    s += 1.0 * tmp[r + 4][c];
    const float o = static_cast<float>(s / 16.0);
    a.smooth[(size_t)b * a.h * a.w + (size_t)v * a.w + u] = o;
    lo = fminf(lo, o);
    hi = fmaxf(hi, o);
  }
  for (int off = 16; off; off >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((tid & 31) == 0) {
    atomicMin(a.minmax + 2 * b, __float_as_uint(lo));  // non-negative floats order as uints
    atomicMax(a.minmax + 2 * b + 1, __float_as_uint(hi));
  }
}

struct ViewArgs {
  int h, w;
  const DevScene* scenes;
  const float* smooth;
  const unsigned* minmax;
  const float* gt;
  const double2* pairs;
  long long need;
  float* left;
  float* right;
};

// sample_disparity_row (synth.cpp:84-91).
__device__ __forceinline__ double sample_disp(const float* row, int w, double s) {
  s = fmin(fmax(s, 0.0), static_cast<double>(w - 1));
  const int s0 = static_cast<int>(s);
  const int s1 = min(s0 + 1, w - 1);
  const double t = s - s0;
  return (1 - t) * row[s0] + t * row[s1];
}

__global__ void k_views(ViewArgs a) {
  const long long per = (long long)a.h * a.w;
  const int b = blockIdx.y;
  const DevScene s = a.scenes[b];
  const float lo = __uint_as_float(a.minmax[2 * b]), hi = __uint_as_float(a.minmax[2 * b + 1]);
  const bool spread = hi > lo;
  const float scale = spread ? 190.0f / (hi - lo) : 0.0f;
  const float* sm = a.smooth + b * per;
  auto norm = [&](float t) { return spread ? 30.0f + (t - lo) * scale : 125.0f; };  // :68-70
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < per;
       p += (long long)gridDim.x * blockDim.x) {
    const int v = int(p / a.w), x = int(p - (long long)v * a.w);
    const float* grow = a.gt + b * per + (long long)v * a.w;
    const float* srow = sm + (long long)v * a.w;
    float left = norm(srow[x]);
    // right(v, x) = left(v, u*), u* = x + d(v, u*) by 8 fixed-point steps (:126-137)
    double u = x + sample_disp(grow, a.w, x);
    for (int it = 0; it < 8; ++it) u = x + sample_disp(grow, a.w, u);
    const double sc = fmin(fmax(u, 0.0), static_cast<double>(a.w - 1));  // sample_row (:74-82)
    const int s0 = static_cast<int>(sc);
    const int s1 = min(s0 + 1, a.w - 1);
    const double t = sc - s0;
    float right = static_cast<float>((1 - t) * norm(srow[s0]) + t * norm(srow[s1]));
    if (s.sigma > 0) {  // :139-146: left(v,u) takes gauss #2k, right #2k+1 of pixel k
      const double2 q = a.pairs[b * a.need + p];
      double first, second;
      polar_pair(q.x, q.y, first, second);
      const double gl = first * s.sigma + 0.0, gr = second * s.sigma + 0.0;
      left = fminf(fmaxf(left + static_cast<float>(gl), 0.0f), 255.0f);
      right = fminf(fmaxf(right + static_cast<float>(gr), 0.0f), 255.0f);
    }
    a.left[b * per + p] = left;
    a.right[b * per + p] = right;
  }
}

void check_spec(const rpd_scene_spec& s) {
  if (s.width <= 0 || s.height <= 0) throw InvalidArg("generate_scene: image dimensions must be positive");
  if (s.n_potholes < 0 || (s.n_potholes > 0 && !s.potholes))
    throw InvalidArg("generate_scene: bad pothole list");
  for (int k = 0; k < s.n_potholes; ++k) {
    const rpd_pothole_spec& p = s.potholes[k];
    if (p.depth <= 0 || p.ru < 4 || p.rv < 4)
      throw InvalidArg("generate_scene: bad pothole spec");
  }
}

// Enqueues the generation of `count` scenes of one size into device buffers.
void enqueue_scenes(rpd_ctx* ctx, int count, const rpd_scene_spec* specs, float* d_left,
                    float* d_right, float* d_gt, int32_t* d_mask, int* d_negative) {
  const int w = specs[0].width, h = specs[0].height;
  std::vector<DevScene> hs(static_cast<size_t>(count));
  std::vector<DevPothole> hp;
  bool any_noise = false;
  for (int b = 0; b < count; ++b) {
    const rpd_scene_spec& s = specs[b];
    check_spec(s);
    if (s.width != w || s.height != h) throw InvalidArg("generate_scenes: scenes differ in size");
    DevScene& d = hs[size_t(b)];
    d.a0 = s.a0;
    d.a1 = s.a1;
    d.cphi = std::cos(s.phi_true);
    d.sphi = std::sin(s.phi_true);
    d.sigma = s.noise_sigma;
    d.seed = s.texture_seed;
    d.pot_off = int(hp.size());
    d.n_pot = s.n_potholes;
    for (int k = 0; k < s.n_potholes; ++k) {
      const rpd_pothole_spec& p = s.potholes[k];
      hp.push_back(DevPothole{p.cu, p.cv, p.ru, p.rv, p.depth});
    }
    any_noise |= s.noise_sigma > 0;
  }
  const long long per = (long long)h * w;
  const Lattice L = lattice_of(w, h);
  float* lattice = ctx->ws.get<float>("syn_lattice", size_t(count) * L.total);
  const long long need = any_noise ? per : 0;
  double2* pairs = ctx->ws.get<double2>("syn_pairs", size_t(count) * std::max<long long>(need, 1));
  // attempts drawn: need / (pi/4) + 2% + 4096 (the shortfall is > 20 sigma away;
  // k_polar_scatter flags it), rounded up to whole polar blocks
  const long long attempts =
      any_noise ? ((long long)(need / 0.7853981633974483 * 1.02) + 4096 + kPolarPerBlock - 1) /
                      kPolarPerBlock * kPolarPerBlock
                : 0;
  const long long nwords = 4 * attempts;
  if (nwords + 624 + kMtRound > 0x7fffffffLL || (long long)L.total > 0x7fffffffLL)
    throw InvalidArg("generate_scene: image too large for the noise stream");
  const int polar_blocks = int(attempts / kPolarPerBlock);
  uint32_t* words = ctx->ws.get<uint32_t>("syn_words", size_t(count) * std::max<long long>(nwords, 1));
  int* pcounts = ctx->ws.get<int>("syn_pcounts", size_t(count) * std::max(polar_blocks, 1));
  float* smooth = ctx->ws.get<float>("syn_smooth", size_t(count) * per);
  // one pinned staging block: scene table | pothole list | min/max seeds
  const size_t scene_bytes = sizeof(DevScene) * hs.size();
  const size_t pot_bytes = sizeof(DevPothole) * std::max<size_t>(hp.size(), 1);
  const size_t mm_bytes = sizeof(unsigned) * 2 * size_t(count);
  const size_t bytes = scene_bytes + pot_bytes + mm_bytes;
  char* stage = static_cast<char*>(ctx->pinned.get(bytes));
  std::memcpy(stage, hs.data(), scene_bytes);
  if (!hp.empty()) std::memcpy(stage + scene_bytes, hp.data(), sizeof(DevPothole) * hp.size());
  unsigned* mm = reinterpret_cast<unsigned*>(stage + scene_bytes + pot_bytes);
  for (int b = 0; b < count; ++b) {
    mm[2 * b] = 0x7f7fffffu;  // FLT_MAX
    mm[2 * b + 1] = 0u;
  }
  char* dstage = ctx->ws.get<char>("syn_spec", bytes);
  RPD_CK(cudaMemcpyAsync(dstage, stage, bytes, cudaMemcpyHostToDevice, ctx->stream));
  const DevScene* dsc = reinterpret_cast<const DevScene*>(dstage);
  const DevPothole* dpot = reinterpret_cast<const DevPothole*>(dstage + scene_bytes);
  unsigned* minmax = reinterpret_cast<unsigned*>(dstage + scene_bytes + pot_bytes);
  RPD_CK(cudaMemsetAsync(d_negative, 0, sizeof(int) * size_t(count + 1), ctx->stream));

  k_mt_streams<<<dim3(count, any_noise ? 2 : 1), kMtThreads, 0, ctx->stream>>>(
      dsc, L.total, lattice, words, int(nwords));
  RPD_LAUNCH_CHECK();
  if (any_noise) {
    k_polar_count<<<dim3(polar_blocks, count), kPolarThreads, 0, ctx->stream>>>(dsc, words, nwords,
                                                                                pcounts);
    RPD_LAUNCH_CHECK();
    k_polar_scatter<<<dim3(polar_blocks, count), kPolarThreads, 0, ctx->stream>>>(
        dsc, words, nwords, pcounts, pairs, need, d_negative + count);
    RPD_LAUNCH_CHECK();
  }
  const int px_blocks = int(std::min<long long>((per + 255) / 256, 1024));
  k_truth<<<dim3(px_blocks, count), 256, 0, ctx->stream>>>(dsc, dpot, h, w, d_gt, d_mask,
                                                          d_negative);
  RPD_LAUNCH_CHECK();
  TexArgs ta{L, h, w, lattice, smooth, minmax};
  k_texture<<<dim3((w + kTexTW - 1) / kTexTW, (h + kTexTH - 1) / kTexTH, count), 256, 0,
              ctx->stream>>>(ta);
  RPD_LAUNCH_CHECK();
  ViewArgs va{h, w, dsc, smooth, minmax, d_gt, pairs, need, d_left, d_right};
  k_views<<<dim3(px_blocks, count), 256, 0, ctx->stream>>>(va);
  RPD_LAUNCH_CHECK();
}

}  // namespace

extern "C" {

void rpd_scene_spec_default(rpd_scene_spec* s) {
  s->width = 640;
  s->height = 480;
  s->rig = rpd_stereo_rig{700.0, 0.12, 0.0, 0.0};
  s->a0 = 5.0;
  s->a1 = 0.08;
  s->phi_true = 0.0;
  s->texture_seed = 1;
  s->noise_sigma = 0.0;
  s->n_potholes = 0;
  s->potholes = nullptr;
}

void rpd_batch_ranges_default(rpd_batch_ranges* r) {
  *r = rpd_batch_ranges{1.5, 4.0, 22.0, 48.0, 4.0, 7.0, 0.07, 0.09, 0.035, 0.0, 40};
}

rpd_status rpd_scene_batch_spec(uint32_t base_seed, int32_t index, const rpd_batch_ranges* r,
                                rpd_scene_spec* spec, rpd_pothole_spec potholes[3]) {
  if (index < 0 || !r || !spec || !potholes) return RPD_EINVAL;
  // synth.cpp:157-191: a few dozen draws per scene, on the host like the
  // reference (the pixels are generated on the device)
  const uint32_t seed = base_seed + static_cast<uint32_t>(index);
  std::mt19937 rng(seed * 2654435761u + 12345u);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  rpd_scene_spec_default(spec);
  spec->texture_seed = seed;
  spec->noise_sigma = r->noise_sigma;
  spec->a0 = r->a0_min + (r->a0_max - r->a0_min) * uni(rng);
  spec->a1 = r->a1_min + (r->a1_max - r->a1_min) * uni(rng);
  spec->phi_true = r->phi_abs_max * (2.0 * uni(rng) - 1.0);
  spec->rig.cu = spec->width / 2.0;
  spec->rig.cv = spec->height / 2.0;
  int np = 0;
  const int n_potholes = 1 + static_cast<int>(uni(rng) * 3.0) % 3;
  for (int k = 0; k < n_potholes; ++k) {
    for (int attempt = 0; attempt < 100; ++attempt) {
      rpd_pothole_spec p;
      p.ru = r->radius_min + (r->radius_max - r->radius_min) * uni(rng);
      p.rv = r->radius_min + (r->radius_max - r->radius_min) * uni(rng);
      p.depth = r->depth_min + (r->depth_max - r->depth_min) * uni(rng);
      const double mu = r->margin + p.ru;
      const double mv = r->margin + p.rv;
      p.cu = mu + (spec->width - 2 * mu) * uni(rng);
      p.cv = mv + (spec->height - 2 * mv) * uni(rng);
      bool overlaps = false;
      for (int q = 0; q < np; ++q) {
        const double dx = p.cu - potholes[q].cu, dy = p.cv - potholes[q].cv;
        const double sep = std::max(p.ru + potholes[q].ru, p.rv + potholes[q].rv) + 10.0;
        if (dx * dx + dy * dy < sep * sep) overlaps = true;
      }
      if (!overlaps) {
        potholes[np++] = p;
        break;
      }
    }
  }
  spec->n_potholes = np;
  spec->potholes = potholes;
  return RPD_OK;
}

rpd_status rpd_generate_scene(rpd_ctx* ctx, const rpd_scene_spec* spec, float* left,
                              float* right, float* gt_disparity, int32_t* gt_mask) {
  return guard(ctx, [&] {
    if (!spec) throw InvalidArg("generate_scene: null spec");
    check_spec(*spec);
    const size_t n = size_t(spec->height) * spec->width;
    float* dl = ctx->ws.get<float>("syn_left", n);
    float* dr = ctx->ws.get<float>("syn_right", n);
    float* dg = ctx->ws.get<float>("syn_gt", n);
    int32_t* dm = ctx->ws.get<int32_t>("syn_mask", n);
    int* neg = ctx->ws.get<int>("syn_neg", 2);
    enqueue_scenes(ctx, 1, spec, dl, dr, dg, dm, neg);
    int hneg[2] = {0, 0};
    download(ctx, hneg, neg, sizeof(hneg));
    if (hneg[0]) throw Degenerate("generate_scene: pothole depth drives disparity negative");
    if (hneg[1]) throw CudaFail("generate_scene: noise stream exhausted");
    if (left) download(ctx, left, dl, sizeof(float) * n);
    if (right) download(ctx, right, dr, sizeof(float) * n);
    if (gt_disparity) download(ctx, gt_disparity, dg, sizeof(float) * n);
    if (gt_mask) download(ctx, gt_mask, dm, sizeof(int32_t) * n);
  });
}

rpd_status rpd_generate_scenes_device(rpd_ctx* ctx, int count, const rpd_scene_spec* specs,
                                      float* d_left, float* d_right, float* d_gt,
                                      int32_t* d_mask) {
  return guard(ctx, [&] {
    if (count < 1 || !specs) throw InvalidArg("generate_scenes: count must be >= 1");
    if (!d_left || !d_right || !d_gt || !d_mask)
      throw InvalidArg("generate_scenes: null device buffer");
    int* neg = ctx->ws.get<int>("syn_negs", size_t(count) + 1);
    enqueue_scenes(ctx, count, specs, d_left, d_right, d_gt, d_mask, neg);
    int* hneg = static_cast<int*>(ctx->pinned.get(sizeof(int) * (size_t(count) + 1)));
    download(ctx, hneg, neg, sizeof(int) * (size_t(count) + 1));
    if (hneg[count]) throw CudaFail("generate_scene: noise stream exhausted");
    for (int b = 0; b < count; ++b)
      if (hneg[b])
        throw Degenerate("generate_scene: pothole depth drives disparity negative (scene " +
                         std::to_string(b) + ")");
  });
}

}  // extern "C"
