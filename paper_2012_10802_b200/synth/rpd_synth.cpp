// rpd_synth.cpp — seeded synthetic stereo road scenes for the BASELINE configs.
//
// Harness component (the reference's counterpart is src/synth.cpp:94-196, a
// planar road with elliptic-paraboloid potholes and a fixed-point right-view
// warp).  BASELINE.json asks for a quadratic road in the rotated row
// coordinate, uint8 images, Perlin-plus-uniform texture and (config 4) shallow
// cracks; this generator implements exactly that with a counter-based RNG
// (SplitMix64), so every frame is reproducible from (seed, frame) alone:
//   seed(config c, frame i) = 20121080 + 1000*c + i
//
//   d(u,v) = d_min + (d_max-d_min) * ((1-q) s + q s^2),  s = (v' - v'_min)/(v'_max - v'_min)
//   v' = v cos(phi) - u sin(phi)   (types.hpp:40 roll convention), q = quadratic share
//   pothole: d -= depth * (1 - r^2) inside the ellipse (synth.cpp:110-118)
//   right(x) = left(u) with u = x + d(v, u) (8 fixed-point iterations, synth.cpp:131-137)
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

extern "C" {

typedef struct rpd_scene_params {
  int32_t width, height;
  uint64_t seed;
  int32_t texture;        // 0 = iid uniform [0,255], 1 = 3-octave Perlin + uniform
  double d_min, d_max;    // road disparity range over the image
  double quad_share;      // share of the quadratic term (0.25)
  double phi;             // roll, rad
  int32_t n_potholes;
  double axis_min, axis_max;    // pothole semi-axes, px
  double depth_min, depth_max;  // pothole depth, px of disparity
  int32_t centred;        // 1: a single pothole at the image centre with axes (axis_max, axis_min)
  int32_t n_cracks;
  double crack_w_min, crack_w_max, crack_depth_min, crack_depth_max;
  double noise_sigma;
  int32_t margin;         // keep potholes away from the border
} rpd_scene_params;

}  // extern "C"

namespace {

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Counter-based uniform in [0,1): stream `tag`, counter `i`.
inline double u01(uint64_t seed, uint64_t tag, uint64_t i) {
  const uint64_t x = mix64(mix64(seed ^ (tag * 0xD6E8FEB86659FD93ull)) + i);
  return double(x >> 11) * (1.0 / 9007199254740992.0);
}

inline double gauss(uint64_t seed, uint64_t tag, uint64_t i) {
  const double a = std::max(u01(seed, tag, 2 * i), 1e-300);
  const double b = u01(seed, tag, 2 * i + 1);
  return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
}

enum : uint64_t { kTagTex = 1, kTagPerlin = 2, kTagPot = 3, kTagNoise = 4, kTagCrack = 5 };

double fade(double t) { return t * t * t * (t * (t * 6.0 - 15.0) + 10.0); }

// One octave of 2-D gradient (Perlin) noise with lattice spacing `cell`.
void perlin_octave(int w, int h, double cell, uint64_t seed, uint64_t octave, double amp,
                   std::vector<double>& acc) {
  const int gx = int(w / cell) + 2, gy = int(h / cell) + 2;
  std::vector<double> gu(size_t(gx) * gy), gv(size_t(gx) * gy);
  for (int j = 0; j < gy; ++j)
    for (int i = 0; i < gx; ++i) {
      const double a = 6.283185307179586 *
                       u01(seed, kTagPerlin * 16 + octave, uint64_t(j) * uint64_t(gx) + i);
      gu[size_t(j) * gx + i] = std::cos(a);
      gv[size_t(j) * gx + i] = std::sin(a);
    }
  for (int v = 0; v < h; ++v) {
    const double y = v / cell;
    const int j = int(y);
    const double fy = y - j, sy = fade(fy);
    for (int u = 0; u < w; ++u) {
      const double x = u / cell;
      const int i = int(x);
      const double fx = x - i, sx = fade(fx);
      auto dot = [&](int ii, int jj, double dx, double dy) {
        const size_t k = size_t(jj) * gx + ii;
        return gu[k] * dx + gv[k] * dy;
      };
      const double n00 = dot(i, j, fx, fy), n10 = dot(i + 1, j, fx - 1, fy);
      const double n01 = dot(i, j + 1, fx, fy - 1), n11 = dot(i + 1, j + 1, fx - 1, fy - 1);
      const double nx0 = n00 + (n10 - n00) * sx, nx1 = n01 + (n11 - n01) * sx;
      acc[size_t(v) * w + u] += amp * (nx0 + (nx1 - nx0) * sy);
    }
  }
}

double sample_row(const std::vector<double>& img, int w, int v, double s) {
  s = std::clamp(s, 0.0, double(w - 1));
  const int s0 = int(s), s1 = std::min(s0 + 1, w - 1);
  const double t = s - s0;
  return (1 - t) * img[size_t(v) * w + s0] + t * img[size_t(v) * w + s1];
}

}  // namespace

extern "C" {

// Fills left/right (uint8, H*W) and optionally the ground-truth disparity
// (float, H*W) and pothole mask (int32, pothole index + 1).  Returns 0.
int rpd_synth_scene(const rpd_scene_params* p, uint8_t* left, uint8_t* right, float* gt_disp,
                    int32_t* gt_mask) {
  const int w = p->width, h = p->height;
  if (w < 8 || h < 8 || !(p->d_max > p->d_min) || p->d_min < 0) return 1;
  const size_t n = size_t(w) * h;
  const uint64_t seed = p->seed;
  // ---- texture
  std::vector<double> tex(n, 0.0);
  if (p->texture == 0) {
    for (size_t i = 0; i < n; ++i) tex[i] = std::floor(256.0 * u01(seed, kTagTex, i));
  } else {
    std::vector<double> pn(n, 0.0);
    const double cells[3] = {48.0, 12.0, 3.0}, amps[3] = {1.0, 0.5, 0.25};
    for (int o = 0; o < 3; ++o) perlin_octave(w, h, cells[o], seed, uint64_t(o), amps[o], pn);
    double lo = pn[0], hi = pn[0];
    for (double x : pn) {
      lo = std::min(lo, x);
      hi = std::max(hi, x);
    }
    const double span = hi > lo ? hi - lo : 1.0;
    for (size_t i = 0; i < n; ++i)
      tex[i] = std::floor(255.0 * (0.55 * (pn[i] - lo) / span + 0.45 * u01(seed, kTagTex, i)));
  }
  // ---- road surface
  const double c = std::cos(p->phi), s = std::sin(p->phi);
  double vlo = 1e300, vhi = -1e300;
  for (int cv = 0; cv <= 1; ++cv)
    for (int cu = 0; cu <= 1; ++cu) {
      const double vp = (cv * (h - 1)) * c - (cu * (w - 1)) * s;
      vlo = std::min(vlo, vp);
      vhi = std::max(vhi, vp);
    }
  const double q = p->quad_share;
  std::vector<double> disp(n);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const double t = ((v * c - u * s) - vlo) / (vhi - vlo);
      disp[size_t(v) * w + u] = p->d_min + (p->d_max - p->d_min) * ((1 - q) * t + q * t * t);
    }
  std::vector<int32_t> mask(n, 0);
  // ---- potholes (non-overlapping ellipses)
  struct Pot {
    double cu, cv, ru, rv, depth;
  };
  std::vector<Pot> pots;
  uint64_t ctr = 0;
  for (int k = 0; k < p->n_potholes; ++k) {
    for (int attempt = 0; attempt < 200; ++attempt) {
      Pot pt;
      if (p->centred) {
        pt = {w / 2.0, h / 2.0, p->axis_max, p->axis_min, p->depth_max};
      } else {
        pt.ru = p->axis_min + (p->axis_max - p->axis_min) * u01(seed, kTagPot, ctr++);
        pt.rv = p->axis_min + (p->axis_max - p->axis_min) * u01(seed, kTagPot, ctr++) * 0.6;
        pt.rv = std::max(pt.rv, 8.0);
        pt.depth = p->depth_min + (p->depth_max - p->depth_min) * u01(seed, kTagPot, ctr++);
        const double mu = p->margin + pt.ru, mv = p->margin + pt.rv;
        if (w - 2 * mu <= 0 || h - 2 * mv <= 0) continue;
        pt.cu = mu + (w - 2 * mu) * u01(seed, kTagPot, ctr++);
        pt.cv = mv + (h - 2 * mv) * u01(seed, kTagPot, ctr++);
      }
      bool overlap = false;
      for (const Pot& o : pots) {
        const double dx = pt.cu - o.cu, dy = pt.cv - o.cv;
        const double sep = std::max(pt.ru + o.ru, pt.rv + o.rv) + 10.0;
        if (dx * dx + dy * dy < sep * sep) overlap = true;
      }
      if (overlap) continue;
      pots.push_back(pt);
      break;
    }
  }
  for (size_t k = 0; k < pots.size(); ++k) {
    const Pot& pt = pots[k];
    const int v0 = std::max(0, int(pt.cv - pt.rv) - 1), v1 = std::min(h - 1, int(pt.cv + pt.rv) + 1);
    const int u0 = std::max(0, int(pt.cu - pt.ru) - 1), u1 = std::min(w - 1, int(pt.cu + pt.ru) + 1);
    for (int v = v0; v <= v1; ++v)
      for (int u = u0; u <= u1; ++u) {
        const double ru = (u - pt.cu) / pt.ru, rv = (v - pt.cv) / pt.rv;
        const double r2 = ru * ru + rv * rv;
        if (r2 < 1.0) {
          disp[size_t(v) * w + u] -= pt.depth * (1.0 - r2);
          mask[size_t(v) * w + u] = int32_t(k) + 1;
        }
      }
  }
  // ---- cracks: random polylines of constant depth
  for (int k = 0; k < p->n_cracks; ++k) {
    const uint64_t base = uint64_t(k) * 64;
    const double width = p->crack_w_min + (p->crack_w_max - p->crack_w_min) * u01(seed, kTagCrack, base);
    const double depth =
        p->crack_depth_min + (p->crack_depth_max - p->crack_depth_min) * u01(seed, kTagCrack, base + 1);
    double x = p->margin + (w - 2.0 * p->margin) * u01(seed, kTagCrack, base + 2);
    double y = p->margin + (h - 2.0 * p->margin) * u01(seed, kTagCrack, base + 3);
    double ang = 6.283185307179586 * u01(seed, kTagCrack, base + 4);
    const int segs = 4 + int(4 * u01(seed, kTagCrack, base + 5));
    for (int sgi = 0; sgi < segs; ++sgi) {
      ang += (u01(seed, kTagCrack, base + 6 + sgi) - 0.5) * 1.2;
      const double len = 20.0 + 40.0 * u01(seed, kTagCrack, base + 20 + sgi);
      const double x1 = x + len * std::cos(ang), y1 = y + len * std::sin(ang);
      const int ua = std::max(0, int(std::min(x, x1) - width) - 1);
      const int ub = std::min(w - 1, int(std::max(x, x1) + width) + 1);
      const int va = std::max(0, int(std::min(y, y1) - width) - 1);
      const int vb = std::min(h - 1, int(std::max(y, y1) + width) + 1);
      const double dx = x1 - x, dy = y1 - y, l2 = dx * dx + dy * dy;
      for (int v = va; v <= vb; ++v)
        for (int u = ua; u <= ub; ++u) {
          const double t = std::clamp(((u - x) * dx + (v - y) * dy) / l2, 0.0, 1.0);
          const double ex = u - (x + t * dx), ey = v - (y + t * dy);
          if (ex * ex + ey * ey <= 0.25 * width * width) {
            double& d = disp[size_t(v) * w + u];
            d = std::max(0.0, d - depth);
          }
        }
      x = x1;
      y = y1;
    }
  }
  // ---- right view by the fixed-point disparity warp
  std::vector<double> rv(n);
  for (int v = 0; v < h; ++v)
    for (int xx = 0; xx < w; ++xx) {
      double u = xx + sample_row(disp, w, v, xx);
      for (int it = 0; it < 8; ++it) u = xx + sample_row(disp, w, v, u);
      rv[size_t(v) * w + xx] = sample_row(tex, w, v, u);
    }
  // ---- sensor noise, rounding to uint8
  for (size_t i = 0; i < n; ++i) {
    double l = tex[i], r = rv[i];
    if (p->noise_sigma > 0) {
      l += p->noise_sigma * gauss(seed, kTagNoise, 2 * i);
      r += p->noise_sigma * gauss(seed, kTagNoise, 2 * i + 1);
    }
    left[i] = uint8_t(std::clamp(std::nearbyint(l), 0.0, 255.0));
    right[i] = uint8_t(std::clamp(std::nearbyint(r), 0.0, 255.0));
    if (gt_disp) gt_disp[i] = float(disp[i]);
    if (gt_mask) gt_mask[i] = mask[i];
  }
  return 0;
}

}  // extern "C"
