// rpd_oracle.cpp — CPU ORACLE (test infrastructure, NOT the product).
//
// A scalar, sequential C++20 restatement of the reference hot path
// (/root/reference/proj, cited file:line below).  It exports the same C-ABI as
// the CUDA library (include/rpd_b200.h) so the parity tests can run one set of
// ctypes bindings against both libraries.  Only tests/, __graft_entry__.smoke()
// and bench.py's CPU-baseline leg may load it.
//
// Parity pins: the known answers of the reference's own unit tests and
// acceptance oracles are ported in tests/test_oracle_*.py.
// The reference itself cannot be compiled here (Eigen3, libpng, doctest absent;
// SURVEY.md §8c) so there is no literal-reference cross-check.
//
// Deliberate, documented choices where the reference is unpinned:
//  * fit_line reductions (road_geometry.cpp:20-24, 37) are Eigen reductions
//    whose SIMD order cannot be reproduced without Eigen.  The oracle fixes one
//    order — kFitLanes strided lanes, then an adjacent-pairwise tree — which is
//    also the device kernel's order (DESIGN.md §road fit).  The normal
//    equations and the search energies come from double-double observation
//    moments (exact products); the reported e0min keeps the residual form.
//  * `sgm_paths` (4 or 8) selects the first entries of kEightDirections
//    (sgm.hpp:41-43); the reference always uses 8 (sgm.cpp:183-186).
//
// Build: g++ -O2 -std=c++20 -ffp-contract=off (no -march=native): x86-64 SSE2
// arithmetic without contraction, like the reference build.

#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "rpd_b200.h"

namespace oracle {

// ---------------------------------------------------------------- rasters --
template <typename T>
struct Raster {  // row-major (v, u), types.hpp:9-10
  int h = 0, w = 0;
  std::vector<T> a;
  Raster() = default;
  Raster(int h_, int w_, T fill = T{}) : h(h_), w(w_), a(size_t(h_) * w_, fill) {}
  T& operator()(int v, int u) { return a[size_t(v) * w + u]; }
  const T& operator()(int v, int u) const { return a[size_t(v) * w + u]; }
};
using Gray = Raster<float>;
using Disp = Raster<float>;
using Labels = Raster<int>;
constexpr float kInvalid = -1.0f;  // types.hpp:21
inline bool valid(float d) { return d != kInvalid; }

struct Model {
  double a0 = 0, a1 = 0, phi = 0;
};
// types.hpp:39-41
inline double road_at(const Model& m, double u, double v) {
  return m.a0 + m.a1 * (v * std::cos(m.phi) - u * std::sin(m.phi));
}

struct Degenerate : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------- config ----
void config_default(rpd_config* c) {  // config.hpp:11-33
  c->delta_pt = 5.0;
  c->delta_dt = 30.0;
  c->delta_pd = 2.36;
  c->d_max = 64;
  c->d_max_pt = 16;
  c->lambda1 = 8.0;
  c->lambda2 = 32.0;
  c->census_window = 5;
  c->lr_threshold = 1.0;
  c->superpixels = 1365;
  c->compactness = 8.0;
  c->slic_iterations = 10;
  c->hist_bin_width = 0.25;
  c->tau_diag = 3.0;
  c->border_margin = 5;
  c->min_superpixels = 2;
  c->connectivity = 8;
  c->roll_bracket = 0.261799;
  c->roll_tol = 1e-4;
  c->focal = 700.0;
  c->baseline = 0.12;
  c->cu = -1.0;
  c->cv = -1.0;
  c->sgm_paths = 8;
}

void config_validate(const rpd_config& c) {  // config.cpp:9-22
  auto fail = [](const char* m) { throw std::invalid_argument(std::string("config: ") + m); };
  if (c.delta_pt < 0) fail("delta_pt must be >= 0");
  if (c.delta_dt <= 0) fail("delta_dt must be > 0");
  if (c.delta_pd <= 0) fail("delta_pd must be > 0");
  if (c.d_max < 1 || c.d_max_pt < 1) fail("d_max must be >= 1");
  if (!(c.lambda1 > 0 && c.lambda1 <= c.lambda2)) fail("need 0 < lambda1 <= lambda2");
  if (c.census_window != 3 && c.census_window != 5 && c.census_window != 7)
    fail("census_window must be 3, 5 or 7");
  if (c.superpixels < 4) fail("superpixels must be >= 4");
  if (c.compactness <= 0) fail("compactness must be > 0");
  if (c.connectivity != 4 && c.connectivity != 8) fail("connectivity must be 4 or 8");
  if (c.roll_bracket <= 0 || c.roll_tol <= 0) fail("roll bracket/tol must be > 0");
  if (c.focal <= 0 || c.baseline <= 0) fail("focal and baseline must be > 0");
  if (c.sgm_paths != 4 && c.sgm_paths != 8) fail("sgm_paths must be 4 or 8");
}

// --------------------------------------------------------- perspective ----
struct Shifts {
  std::vector<double> s;
  double delta_pt = 0;
};

// perspective.hpp:23-35
Shifts row_shifts(const Model& m, int w, int h, double delta_pt) {
  if (w < 2) throw std::invalid_argument("compute_row_shifts: width must be >= 2");
  Shifts t;
  t.delta_pt = delta_pt;
  t.s.resize(size_t(h));
  for (int v = 0; v < h; ++v) {
    const double left = road_at(m, 0.0, v);
    const double right = road_at(m, double(w), v);
    t.s[size_t(v)] = std::max(0.0, std::min(left, right) - delta_pt);
  }
  return t;
}

struct Warped {
  Gray img;
  Raster<uint8_t> in_view;
};

// perspective.hpp:45-66
Warped warp(const Gray& right, const Shifts& t) {
  const int h = right.h, w = right.w;
  if (int(t.s.size()) != h)
    throw std::invalid_argument("warp_right_image: table length != image height");
  Warped out{Gray(h, w, 0.0f), Raster<uint8_t>(h, w, 0)};
  for (int v = 0; v < h; ++v) {
    const double shift = t.s[size_t(v)];
    for (int u = 0; u < w; ++u) {
      const double s = u - shift;
      if (s < 0.0 || s > w - 1) continue;
      const int s0 = int(std::floor(s));
      const int s1 = std::min(s0 + 1, w - 1);
      const double frac = s - s0;
      out.img(v, u) = float((1.0 - frac) * right(v, s0) + frac * right(v, s1));
      out.in_view(v, u) = 1;
    }
  }
  return out;
}

// perspective.hpp:69-80
Disp restore(const Disp& d0, const Shifts& t) {
  if (int(t.s.size()) != d0.h)
    throw std::invalid_argument("restore_disparity: table length != map height");
  Disp d1 = d0;
  for (int v = 0; v < d0.h; ++v) {
    const float add = float(t.s[size_t(v)]);
    for (int u = 0; u < d0.w; ++u)
      if (valid(d0(v, u))) d1(v, u) = d0(v, u) + add;
  }
  return d1;
}

// ----------------------------------------------------------------- SGM ----
struct Volume {  // sgm.hpp:15-33
  int w = 0, h = 0, d_max = 0;
  std::vector<float> c;
  Volume() = default;
  Volume(int w_, int h_, int dm) : w(w_), h(h_), d_max(dm), c(size_t(w_) * h_ * (dm + 1), 0.f) {}
  int levels() const { return d_max + 1; }
  float& at(int v, int u, int d) { return c[(size_t(v) * w + u) * levels() + d]; }
  float at(int v, int u, int d) const { return c[(size_t(v) * w + u) * levels() + d]; }
};

using Dirs = std::vector<std::array<int, 2>>;
Dirs eight_directions() {  // sgm.hpp:41-43
  return {{{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {1, 1}, {-1, 1}, {1, -1}, {-1, -1}}};
}

// sgm.cpp:13-34: bit per window sample, MSB first in row-major window order,
// centre skipped, coordinates clamped at the border.
Raster<uint64_t> census(const Gray& img, int window) {
  const int h = img.h, w = img.w, r = window / 2;
  Raster<uint64_t> out(h, w, 0);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const float c = img(v, u);
      uint64_t bits = 0;
      for (int dv = -r; dv <= r; ++dv) {
        const int vv = std::clamp(v + dv, 0, h - 1);
        for (int du = -r; du <= r; ++du) {
          if (dv == 0 && du == 0) continue;
          const int uu = std::clamp(u + du, 0, w - 1);
          bits = (bits << 1) | (img(vv, uu) < c ? 1u : 0u);
        }
      }
      out(v, u) = bits;
    }
  return out;
}

// sgm.cpp:38-68
Volume cost_volume(const Gray& left, const Gray& right, int d_max, int window,
                   const Raster<uint8_t>* in_view) {
  const int h = left.h, w = left.w;
  if (right.h != h || right.w != w)
    throw std::invalid_argument("census_cost_volume: dimension mismatch");
  if (window % 2 == 0) throw std::invalid_argument("census_cost_volume: window must be odd");
  if (d_max >= w) throw std::invalid_argument("census_cost_volume: d_max >= width");
  const float worst = float(window * window - 1);
  const auto cl = census(left, window), cr = census(right, window);
  Volume vol(w, h, d_max);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u)
      for (int d = 0; d <= d_max; ++d) {
        const int ur = u - d;
        vol.at(v, u, d) = (ur < 0 || (in_view && !(*in_view)(v, ur)))
                              ? worst
                              : float(std::popcount(cl(v, u) ^ cr(v, ur)));
      }
  return vol;
}

// sgm.cpp:70-110 — scan-line recursion per direction, summed over directions
// in direction order.
Volume aggregate(const Volume& raw, const Dirs& dirs, float l1, float l2) {
  const int w = raw.w, h = raw.h, n = raw.levels();
  Volume total(w, h, raw.d_max);
  std::vector<float> line(size_t(w) * h * n);
  for (const auto& dir : dirs) {
    const int du = dir[0], dv = dir[1];
    const int v0 = dv >= 0 ? 0 : h - 1, v1 = dv >= 0 ? h : -1, vs = dv >= 0 ? 1 : -1;
    const int u0 = du >= 0 ? 0 : w - 1, u1 = du >= 0 ? w : -1, us = du >= 0 ? 1 : -1;
    for (int v = v0; v != v1; v += vs)
      for (int u = u0; u != u1; u += us) {
        const size_t base = (size_t(v) * w + u) * n;
        float* cur = &line[base];
        const float* c = &raw.c[base];
        const int pv = v - dv, pu = u - du;
        if (pv < 0 || pv >= h || pu < 0 || pu >= w) {
          std::copy(c, c + n, cur);
          continue;
        }
        const float* prev = &line[(size_t(pv) * w + pu) * n];
        float mn = prev[0];
        for (int d = 1; d < n; ++d) mn = std::min(mn, prev[d]);
        const float cap = mn + l2;
        for (int d = 0; d < n; ++d) {
          float b = prev[d];
          if (d > 0) b = std::min(b, prev[d - 1] + l1);
          if (d + 1 < n) b = std::min(b, prev[d + 1] + l1);
          b = std::min(b, cap);
          cur[d] = c[d] + b - mn;
        }
      }
    for (size_t i = 0; i < total.c.size(); ++i) total.c[i] += line[i];
  }
  return total;
}

// sgm.cpp:112-121
Volume swap_ref(const Volume& left) {
  const float worst = *std::max_element(left.c.begin(), left.c.end());
  Volume right(left.w, left.h, left.d_max);
  for (int v = 0; v < left.h; ++v)
    for (int u = 0; u < left.w; ++u)
      for (int d = 0; d <= left.d_max; ++d)
        right.at(v, u, d) = (u + d < left.w) ? left.at(v, u + d, d) : worst;
  return right;
}

// sgm.cpp:123-153
Disp wta(const Volume& agg) {
  const int w = agg.w, h = agg.h, n = agg.levels();
  Disp out(h, w);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const float* c = &agg.c[(size_t(v) * w + u) * n];
      int best = 0;
      for (int d = 1; d < n; ++d)
        if (c[d] < c[best]) best = d;
      bool ambiguous = false;
      for (int d = 0; d < n; ++d)
        if (std::abs(d - best) > 1 && c[d] <= c[best]) ambiguous = true;
      if (ambiguous) {
        out(v, u) = kInvalid;
        continue;
      }
      float r = float(best);
      if (best > 0 && best < n - 1) {
        const float denom = c[best - 1] + c[best + 1] - 2.0f * c[best];
        if (denom > 0.0f) r += (c[best - 1] - c[best + 1]) / (2.0f * denom);
      }
      out(v, u) = r;
    }
  return out;
}

// sgm.cpp:155-170
void lr_check(Disp& left, const Disp& right, double thr) {
  for (int v = 0; v < left.h; ++v)
    for (int u = 0; u < left.w; ++u) {
      const float dl = left(v, u);
      if (!valid(dl)) continue;
      const int ur = u - int(std::lround(dl));
      if (ur < 0 || ur >= left.w || !valid(right(v, ur)) || std::abs(dl - right(v, ur)) > thr)
        left(v, u) = kInvalid;
    }
}

struct Match {
  Disp d0, d1;
  Shifts shifts;
};

Dirs config_dirs(const rpd_config& cfg) {
  Dirs all = eight_directions();
  all.resize(size_t(cfg.sgm_paths == 4 ? 4 : 8));
  return all;
}

// sgm.cpp:172-226
Match match_pair(const Gray& left, const Gray& right, const Model& m, const rpd_config& cfg,
                 int d_max) {
  if (left.h != right.h || left.w != right.w)
    throw std::invalid_argument("match_pair: dimension mismatch");
  Match res;
  res.shifts = row_shifts(m, left.w, left.h, cfg.delta_pt);
  Warped wr = warp(right, res.shifts);
  const float l1 = float(cfg.lambda1), l2 = float(cfg.lambda2);
  const Dirs dirs = config_dirs(cfg);
  Volume raw = cost_volume(left, wr.img, d_max, cfg.census_window, &wr.in_view);
  res.d0 = wta(aggregate(raw, dirs, l1, l2));
  Disp right_disp = wta(aggregate(swap_ref(raw), dirs, l1, l2));
  lr_check(res.d0, right_disp, cfg.lr_threshold);
  // flat raw cost curve (sgm.cpp:200-212)
  for (int v = 0; v < left.h; ++v)
    for (int u = 0; u < left.w; ++u) {
      if (!valid(res.d0(v, u))) continue;
      float lo = std::numeric_limits<float>::max(), hi = std::numeric_limits<float>::lowest();
      for (int d = 0; d <= d_max; ++d) {
        const int ur = u - d;
        if (ur < 0 || !wr.in_view(v, ur)) continue;
        lo = std::min(lo, raw.at(v, u, d));
        hi = std::max(hi, raw.at(v, u, d));
      }
      if (hi <= lo) res.d0(v, u) = kInvalid;
    }
  // best sample past the warped border (sgm.cpp:216-222)
  for (int v = 0; v < left.h; ++v)
    for (int u = 0; u < left.w; ++u) {
      const float d = res.d0(v, u);
      if (!valid(d)) continue;
      const int ur = u - int(std::lround(d));
      if (ur < 0 || !wr.in_view(v, ur)) res.d0(v, u) = kInvalid;
    }
  res.d1 = restore(res.d0, res.shifts);
  return res;
}

// ------------------------------------------------------- road geometry ----
struct Obs {
  std::vector<double> d, u, v;
  size_t count() const { return d.size(); }
};

// Fixed reduction order shared with the device kernel: element i goes to lane
// i mod kFitLanes (sequential within a lane, starting from +0.0), then lanes
// are combined by an adjacent-pairwise tree.  `mask` (optional) drops
// elements in place: survivors keep their lanes.
constexpr int kFitLanes = 8192;
template <typename F>
double lane_tree_sum(size_t k, F term, const std::vector<char>* mask = nullptr) {
  std::vector<double> lane(kFitLanes, 0.0);
  for (size_t i = 0; i < k; ++i)
    if (!mask || (*mask)[i]) lane[i % kFitLanes] += term(i);
  for (int width = 1; width < kFitLanes; width *= 2)
    for (int j = 0; j < kFitLanes; j += 2 * width) lane[size_t(j)] += lane[size_t(j + width)];
  return lane[0];
}

// Double-double arithmetic (Dekker, Knuth): the error-free transformations
// and the usual normalised sum / product / quotient.  Operation order is part
// of the contract with the device (road.cu), so is the non-commutative
// dd_add argument order (lower lane first).
struct DD {
  double hi = 0.0, lo = 0.0;
};
inline DD two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
inline DD quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
inline DD two_prod(double a, double b) {
  const double p = a * b;
  return {p, std::fma(a, b, -p)};
}
inline DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
inline DD dd_add_d(DD a, double b) {
  DD s = two_sum(a.hi, b);
  s.lo += a.lo;
  return quick_two_sum(s.hi, s.lo);
}
inline DD dd_sub(DD a, DD b) { return dd_add(a, DD{-b.hi, -b.lo}); }
inline DD dd_mul(DD a, DD b) {
  DD p = two_prod(a.hi, b.hi);
  p.lo = std::fma(a.hi, b.lo, p.lo);
  p.lo = std::fma(a.lo, b.hi, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
inline DD dd_mul_d(DD a, double b) {
  DD p = two_prod(a.hi, b);
  p.lo = std::fma(a.lo, b, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
inline DD dd_div(DD a, DD b) {
  const double q1 = a.hi / b.hi;
  DD r = dd_sub(a, dd_mul_d(b, q1));
  const double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul_d(b, q2));
  const double q3 = r.hi / b.hi;
  return dd_add_d(quick_two_sum(q1, q2), q3);
}
inline bool dd_lt(DD a, DD b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }

// Observation moments su, sv, sd, suu, svv, suv, sdu, sdv, sdd, n in
// double-double (exact products), summed in the lane order.
struct Moments {
  std::array<DD, 10> m;
};
Moments moments(const Obs& o, const std::vector<char>* mask = nullptr) {
  std::vector<std::array<DD, 10>> lane(kFitLanes);
  for (size_t i = 0; i < o.count(); ++i) {
    if (mask && !(*mask)[i]) continue;
    auto& a = lane[i % kFitLanes];
    const double u = o.u[i], v = o.v[i], d = o.d[i];
    a[0] = dd_add_d(a[0], u);
    a[1] = dd_add_d(a[1], v);
    a[2] = dd_add_d(a[2], d);
    a[3] = dd_add(a[3], two_prod(u, u));
    a[4] = dd_add(a[4], two_prod(v, v));
    a[5] = dd_add(a[5], two_prod(u, v));
    a[6] = dd_add(a[6], two_prod(d, u));
    a[7] = dd_add(a[7], two_prod(d, v));
    a[8] = dd_add(a[8], two_prod(d, d));
    a[9] = dd_add_d(a[9], 1.0);
  }
  for (int width = 1; width < kFitLanes; width *= 2)
    for (int j = 0; j < kFitLanes; j += 2 * width)
      for (int q = 0; q < 10; ++q)
        lane[size_t(j)][q] = dd_add(lane[size_t(j)][q], lane[size_t(j + width)][q]);
  return Moments{lane[0]};
}

// fit_line at (c, s) = (cos phi, sin phi) from the moments
// (road_geometry.cpp:16-37), in double-double: st = c Sv - s Su,
// stt = c^2 Svv - 2cs Suv + s^2 Suu, sdt = c Sdv - s Sdu, det = n stt - st^2
// (singular test as :26-29), then either the minimal energy
// E = Sdd - (stt Sd^2 - 2 st Sd sdt + n sdt^2) / det  (the search; the
// expanded form the reference's residual form avoids in double, :35-37, is
// harmless at ~106 bits) or the coefficients a0, a1 (:31-32).
struct LineSums {
  DD N, T1, T2, TD, det;
};
LineSums line_sums(const Moments& M, double c, double s) {
  LineSums o;
  o.N = M.m[9];
  const DD cc = two_prod(c, c), ss = two_prod(s, s), cs = two_prod(c, s);
  o.T1 = dd_sub(dd_mul_d(M.m[1], c), dd_mul_d(M.m[0], s));
  o.T2 = dd_add(dd_sub(dd_mul(cc, M.m[4]), dd_mul_d(dd_mul(cs, M.m[5]), 2.0)), dd_mul(ss, M.m[3]));
  o.TD = dd_sub(dd_mul_d(M.m[7], c), dd_mul_d(M.m[6], s));
  const DD nT2 = dd_mul(o.N, o.T2);
  o.det = dd_sub(nT2, dd_mul(o.T1, o.T1));
  const double scale = nT2.hi < 1.0 ? 1.0 : nT2.hi;
  if (std::abs(o.det.hi) < 1e-12 * scale)
    throw Degenerate("fit_line: degenerate observations (singular normal matrix)");
  return o;
}
DD line_energy(const Moments& M, double c, double s) {
  const LineSums L = line_sums(M, c, s);
  const DD D1 = M.m[2];
  DD q = dd_mul(L.T2, dd_mul(D1, D1));
  q = dd_sub(q, dd_mul_d(dd_mul(dd_mul(L.T1, D1), L.TD), 2.0));
  q = dd_add(q, dd_mul(L.N, dd_mul(L.TD, L.TD)));
  return dd_sub(M.m[8], dd_div(q, L.det));
}

struct LineFit {
  Model model;
  double e0min = 0;
};

// road_geometry.cpp:12-39: a0, a1 from the moments (rounded to double), e0min
// in the reference's residual form, summed in the lane order over `mask`.
LineFit fit_line_m(const Obs& o, const Moments& M, double phi,
                   const std::vector<char>* mask = nullptr) {
  const double c = std::cos(phi), s = std::sin(phi);
  const LineSums L = line_sums(M, c, s);
  const DD D1 = M.m[2];
  LineFit f;
  f.model.phi = phi;
  f.model.a0 = dd_div(dd_sub(dd_mul(L.T2, D1), dd_mul(L.T1, L.TD)), L.det).hi;
  f.model.a1 = dd_div(dd_sub(dd_mul(L.N, L.TD), dd_mul(L.T1, D1)), L.det).hi;
  f.e0min = lane_tree_sum(
      o.count(),
      [&](size_t i) {
        const double t = c * o.v[i] - s * o.u[i];
        const double r = o.d[i] - f.model.a0 - f.model.a1 * t;
        return r * r;
      },
      mask);
  return f;
}

LineFit fit_line(const Obs& o, double phi) {
  if (o.count() < 3) throw std::invalid_argument("fit_line: need at least 3 observations");
  return fit_line_m(o, moments(o), phi);
}

// road_geometry.cpp:41-68 — golden-section search on the energy; every
// probe is evaluated from the moments (same angles and branches as the
// reference's loop).  Returns the final midpoint.
double golden(const Moments& M, double lo, double hi, double tol) {
  constexpr double g = 0.6180339887498949;
  auto energy = [&](double phi) { return line_energy(M, std::cos(phi), std::sin(phi)); };
  double a = lo, b = hi;
  double x1 = b - g * (b - a), x2 = a + g * (b - a);
  DD f1 = energy(x1), f2 = energy(x2);
  while (b - a > tol) {
    if (dd_lt(f1, f2)) {
      b = x2;
      x2 = x1;
      f2 = f1;
      x1 = b - g * (b - a);
      f1 = energy(x1);
    } else {
      a = x1;
      x1 = x2;
      f1 = f2;
      x2 = a + g * (b - a);
      f2 = energy(x2);
    }
  }
  return 0.5 * (a + b);
}

Model estimate_roll(const Obs& o, double lo, double hi, double tol) {
  if (tol <= 0) throw std::invalid_argument("estimate_roll: tol must be > 0");
  if (o.count() < 3) throw std::invalid_argument("fit_line: need at least 3 observations");
  const Moments M = moments(o);
  return fit_line_m(o, M, golden(M, lo, hi, tol)).model;
}

struct RoadFit {
  Model model;
  double e0min = 0;
  int64_t used = 0;
};

// road_geometry.cpp:70-101 (trimming by an in-place mask: survivors keep
// their summation lanes)
RoadFit fit_road(const Obs& o, double bracket, double tol) {
  if (tol <= 0) throw std::invalid_argument("estimate_roll: tol must be > 0");
  const size_t k = o.count();
  if (k < 3) throw std::invalid_argument("fit_line: need at least 3 observations");
  const Moments M = moments(o);
  const LineFit first = fit_line_m(o, M, golden(M, -bracket, bracket, tol));
  const double rms = std::sqrt(first.e0min / double(k));
  RoadFit out{first.model, first.e0min, int64_t(k)};
  if (rms <= 0) return out;
  std::vector<char> keep(k, 0);
  size_t kept = 0;
  for (size_t i = 0; i < k; ++i) {
    const double r = o.d[i] - road_at(first.model, o.u[i], o.v[i]);
    if (std::abs(r) <= 3.0 * rms) {
      keep[i] = 1;
      ++kept;
    }
  }
  if (kept < 3 || kept == k) return out;
  const Moments M2 = moments(o, &keep);
  const LineFit second = fit_line_m(o, M2, golden(M2, -bracket, bracket, tol), &keep);
  return RoadFit{second.model, second.e0min, int64_t(kept)};
}

// road_geometry.cpp:103-134
Obs sample(const Disp& d1, const rpd_rect_roi* roi, int64_t cap) {
  const int h = d1.h, w = d1.w;
  rpd_rect_roi r = roi ? *roi : rpd_rect_roi{0, 0, w, h};
  r.u0 = std::clamp(r.u0, 0, w);
  r.v0 = std::clamp(r.v0, 0, h);
  r.width = std::clamp(r.width, 0, w - r.u0);
  r.height = std::clamp(r.height, 0, h - r.v0);
  std::vector<std::array<int, 2>> pts;
  for (int v = r.v0; v < r.v0 + r.height; ++v)
    for (int u = r.u0; u < r.u0 + r.width; ++u)
      if (valid(d1(v, u))) pts.push_back({u, v});
  const int64_t n = int64_t(pts.size());
  if (n < 3) throw Degenerate("sample_observations: fewer than 3 valid pixels");
  const int64_t k = std::min(n, cap);
  Obs o;
  o.d.resize(size_t(k));
  o.u.resize(size_t(k));
  o.v.resize(size_t(k));
  for (int64_t i = 0; i < k; ++i) {
    const auto& p = pts[size_t(i * n / k)];
    o.u[size_t(i)] = p[0];
    o.v[size_t(i)] = p[1];
    o.d[size_t(i)] = d1(p[1], p[0]);
  }
  return o;
}

// road_geometry.cpp:136-151
Disp transform(const Disp& d1, const Model& m, double delta_dt, int64_t* clamped) {
  Disp d2 = d1;
  int64_t n = 0;
  for (int v = 0; v < d1.h; ++v)
    for (int u = 0; u < d1.w; ++u) {
      if (!valid(d1(v, u))) continue;
      double x = d1(v, u) - road_at(m, u, v) + delta_dt;
      if (x < 0) {
        x = 0;
        ++n;
      }
      d2(v, u) = float(x);
    }
  if (clamped) *clamped = n;
  return d2;
}

// -------------------------------------------------------- segmentation ----
struct Center {
  double cu = 0, cv = 0, value = 0;
};
struct Superpixels {
  Labels labels;
  std::vector<Center> centers;
  int count = 0;
  double spacing = 0;
};

constexpr int kDU[8] = {1, -1, 0, 0, 1, 1, -1, -1};  // segmentation.cpp:104-105
constexpr int kDV[8] = {0, 0, 1, -1, 1, -1, 1, -1};

// segmentation.cpp:22-28 (float difference, then squared in double)
double gradient_at(const Gray& vals, int u, int v) {
  const double gu = vals(v, std::min(u + 1, vals.w - 1)) - vals(v, u);
  const double gv = vals(std::min(v + 1, vals.h - 1), u) - vals(v, u);
  return gu * gu + gv * gv;
}

// segmentation.cpp:30-72
void assign(const Gray& vals, const std::vector<Center>& cs, double S, double m, Labels& lab) {
  const int h = vals.h, w = vals.w;
  Raster<double> best(h, w, std::numeric_limits<double>::infinity());
  std::fill(lab.a.begin(), lab.a.end(), 0);
  const int win = int(std::ceil(S));
  const double sw = m * m / (S * S);
  for (size_t k = 0; k < cs.size(); ++k) {
    const Center& c = cs[k];
    const int cu = int(std::lround(c.cu)), cv = int(std::lround(c.cv));
    const int va = std::max(0, cv - win), vb = std::min(h - 1, cv + win);
    const int ua = std::max(0, cu - win), ub = std::min(w - 1, cu + win);
    for (int v = va; v <= vb; ++v)
      for (int u = ua; u <= ub; ++u) {
        const double dval = vals(v, u) - c.value;
        const double du = u - c.cu, dv = v - c.cv;
        const double dist = dval * dval + (du * du + dv * dv) * sw;
        if (dist < best(v, u)) {
          best(v, u) = dist;
          lab(v, u) = int(k) + 1;
        }
      }
  }
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      if (lab(v, u) != 0) continue;
      double nearest = std::numeric_limits<double>::infinity();
      for (size_t k = 0; k < cs.size(); ++k) {
        const double du = u - cs[k].cu, dv = v - cs[k].cv;
        const double dd = du * du + dv * dv;
        if (dd < nearest) {
          nearest = dd;
          lab(v, u) = int(k) + 1;
        }
      }
    }
}

// segmentation.cpp:74-93 (sums accumulate in scan order)
void update(const Gray& vals, const Labels& lab, std::vector<Center>& cs) {
  const size_t K = cs.size();
  std::vector<double> su(K, 0), sv(K, 0), sx(K, 0);
  std::vector<int64_t> n(K, 0);
  for (int v = 0; v < lab.h; ++v)
    for (int u = 0; u < lab.w; ++u) {
      const int k = lab(v, u) - 1;
      if (k < 0) continue;
      su[size_t(k)] += u;
      sv[size_t(k)] += v;
      sx[size_t(k)] += vals(v, u);
      ++n[size_t(k)];
    }
  for (size_t k = 0; k < K; ++k) {
    if (n[k] == 0) continue;
    cs[k].cu = su[k] / double(n[k]);
    cs[k].cv = sv[k] / double(n[k]);
    cs[k].value = sx[k] / double(n[k]);
  }
}

// segmentation.cpp:98-166
void connectivity(Labels& lab) {
  const int h = lab.h, w = lab.w;
  Labels piece(h, w, 0);
  std::vector<int64_t> size;
  std::vector<int> plabel;
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      if (piece(v, u) != 0) continue;
      const int id = int(size.size()) + 1;
      const int l = lab(v, u);
      int64_t sz = 0;
      std::deque<std::array<int, 2>> q{{u, v}};
      piece(v, u) = id;
      while (!q.empty()) {
        const auto [pu, pv] = q.front();
        q.pop_front();
        ++sz;
        for (int i = 0; i < 8; ++i) {
          const int nu = pu + kDU[i], nv = pv + kDV[i];
          if (nu < 0 || nu >= w || nv < 0 || nv >= h) continue;
          if (piece(nv, nu) == 0 && lab(nv, nu) == l) {
            piece(nv, nu) = id;
            q.push_back({nu, nv});
          }
        }
      }
      size.push_back(sz);
      plabel.push_back(l);
    }
  std::map<int, int> main_piece;
  for (size_t i = 0; i < size.size(); ++i) {
    auto it = main_piece.find(plabel[i]);
    if (it == main_piece.end() || size[i] > size[size_t(it->second - 1)])
      main_piece[plabel[i]] = int(i) + 1;
  }
  std::vector<char> kept(size.size(), 0);
  for (const auto& kv : main_piece) kept[size_t(kv.second - 1)] = 1;
  std::deque<std::array<int, 2>> front;
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      if (kept[size_t(piece(v, u) - 1)])
        front.push_back({u, v});
      else
        lab(v, u) = 0;
    }
  while (!front.empty()) {
    const auto [pu, pv] = front.front();
    front.pop_front();
    for (int i = 0; i < 8; ++i) {
      const int nu = pu + kDU[i], nv = pv + kDV[i];
      if (nu < 0 || nu >= w || nv < 0 || nv >= h) continue;
      if (lab(nv, nu) == 0) {
        lab(nv, nu) = lab(pv, pu);
        front.push_back({nu, nv});
      }
    }
  }
}

// segmentation.cpp:170-229
Superpixels slic(const Disp& d2, int p, double m, int iters) {
  const int h = d2.h, w = d2.w;
  if (p < 4) throw std::invalid_argument("slic: p must be >= 4");
  if (p > w * h) throw std::invalid_argument("slic: p exceeds pixel count");
  Gray vals = d2;
  for (auto& x : vals.a)
    if (!valid(x)) x = 0.0f;
  Superpixels sp;
  sp.spacing = std::sqrt(double(w) * h / p);
  const int nu = std::max(1, int(std::lround(std::sqrt(double(p) * w / h))));
  const int nv = std::max(1, int(std::lround(double(p) / nu)));
  const double su = double(w) / nu, sv = double(h) / nv;
  for (int j = 0; j < nv; ++j)
    for (int i = 0; i < nu; ++i) {
      const int cu = int((i + 0.5) * su), cv = int((j + 0.5) * sv);
      double best = std::numeric_limits<double>::infinity();
      int bu = cu, bv = cv;
      for (int dv = -1; dv <= 1; ++dv)
        for (int du = -1; du <= 1; ++du) {
          const int uu = std::clamp(cu + du, 0, w - 1), vv = std::clamp(cv + dv, 0, h - 1);
          const double g = gradient_at(vals, uu, vv);
          if (g < best) {
            best = g;
            bu = uu;
            bv = vv;
          }
        }
      sp.centers.push_back({double(bu), double(bv), double(vals(bv, bu))});
    }
  sp.labels = Labels(h, w, 0);
  assign(vals, sp.centers, sp.spacing, m, sp.labels);
  for (int it = 0; it < iters; ++it) {
    update(vals, sp.labels, sp.centers);
    assign(vals, sp.centers, sp.spacing, m, sp.labels);
  }
  connectivity(sp.labels);
  std::map<int, int> remap;
  for (auto& l : sp.labels.a) {
    auto [it, fresh] = remap.try_emplace(l, int(remap.size()) + 1);
    (void)fresh;
    l = it->second;
  }
  sp.count = int(remap.size());
  sp.centers.assign(size_t(sp.count), Center{});
  update(vals, sp.labels, sp.centers);
  return sp;
}

// segmentation.cpp:231-249
Disp pool(const Disp& d2, const Labels& lab, int count) {
  if (d2.h != lab.h || d2.w != lab.w)
    throw std::invalid_argument("pool_superpixels: dimension mismatch");
  std::vector<double> sum(size_t(count) + 1, 0.0);
  std::vector<int64_t> n(size_t(count) + 1, 0);
  for (size_t i = 0; i < d2.a.size(); ++i) {
    if (!valid(d2.a[i])) continue;
    sum[size_t(lab.a[i])] += d2.a[i];
    ++n[size_t(lab.a[i])];
  }
  Disp d3(d2.h, d2.w);
  for (size_t i = 0; i < d2.a.size(); ++i) {
    const size_t k = size_t(lab.a[i]);
    d3.a[i] = n[k] > 0 ? float(sum[k] / double(n[k])) : kInvalid;
  }
  return d3;
}

struct Hist {
  double bw = 0.25, origin = 0;
  int64_t n = 0;
  std::vector<int64_t> counts;  // n*n row-major, rows = g1 bins
  int64_t total = 0;
  double center(int64_t b) const { return origin + (b + 0.5) * bw; }
};

// segmentation.cpp:251-296
Hist histogram(const Disp& d2, double bw) {
  if (bw <= 0) throw std::invalid_argument("build_histogram: bin_width must be > 0");
  const int h = d2.h, w = d2.w;
  std::vector<std::array<double, 2>> g;
  for (int v = 1; v + 1 < h; ++v)
    for (int u = 1; u + 1 < w; ++u) {
      if (!valid(d2(v, u))) continue;
      double sum = 0.0;
      bool ok = true;
      for (int dv = -1; dv <= 1 && ok; ++dv)
        for (int du = -1; du <= 1; ++du) {
          if (du == 0 && dv == 0) continue;
          const float x = d2(v + dv, u + du);
          if (!valid(x)) {
            ok = false;
            break;
          }
          sum += x;
        }
      if (ok) g.push_back({double(d2(v, u)), sum / 8.0});
    }
  Hist hist;
  hist.bw = bw;
  if (g.empty()) return hist;
  double lo = g[0][0], hi = g[0][0];
  for (const auto& x : g) {
    lo = std::min({lo, x[0], x[1]});
    hi = std::max({hi, x[0], x[1]});
  }
  hist.origin = std::floor(lo / bw) * bw;
  auto bin = [&](double x) { return int64_t(std::floor((x - hist.origin) / bw)); };
  hist.n = bin(hi) + 1;
  hist.counts.assign(size_t(hist.n * hist.n), 0);
  for (const auto& x : g) {
    const int64_t i = std::min(bin(x[0]), hist.n - 1), j = std::min(bin(x[1]), hist.n - 1);
    ++hist.counts[size_t(i * hist.n + j)];
    ++hist.total;
  }
  return hist;
}

// segmentation.cpp:298-359
rpd_threshold threshold(const Hist& hist, double delta_pd, double tau) {
  std::map<double, int64_t> diag;
  int64_t excluded = 0;
  for (int64_t i = 0; i < hist.n; ++i)
    for (int64_t j = 0; j < hist.n; ++j) {
      const int64_t c = hist.counts[size_t(i * hist.n + j)];
      if (c == 0) continue;
      const double g1 = hist.center(i), g2 = hist.center(j);
      if (std::abs(g1 - g2) > tau) {
        excluded += c;
        continue;
      }
      diag[(g1 + g2) / 2.0] += c;
    }
  if (diag.empty()) throw Degenerate("find_road_threshold: all vectors excluded");
  rpd_threshold res{};
  res.excluded_fraction = hist.total > 0 ? double(excluded) / double(hist.total) : 0.0;
  std::vector<double> x;
  std::vector<int64_t> wt;
  for (const auto& kv : diag) {
    x.push_back(kv.first);
    wt.push_back(kv.second);
  }
  const size_t m = x.size();
  if (m < 2) {
    res.degenerate = 1;
    res.mu1 = res.mu2 = res.t_r = x[0];
    res.t_s = res.t_r - delta_pd;
    return res;
  }
  std::vector<double> pw(m + 1, 0), pwx(m + 1, 0), pwxx(m + 1, 0);
  for (size_t i = 0; i < m; ++i) {
    pw[i + 1] = pw[i] + double(wt[i]);
    pwx[i + 1] = pwx[i] + double(wt[i]) * x[i];
    pwxx[i + 1] = pwxx[i] + double(wt[i]) * x[i] * x[i];
  }
  auto sse = [&](size_t a, size_t b) {
    const double n = pw[b] - pw[a], s = pwx[b] - pwx[a], ss = pwxx[b] - pwxx[a];
    return ss - s * s / n;
  };
  size_t split = 1;
  double best = std::numeric_limits<double>::infinity();
  for (size_t s = 1; s < m; ++s) {
    const double e = sse(0, s) + sse(s, m);
    if (e < best) {
      best = e;
      split = s;
    }
  }
  res.mu1 = (pwx[split] - pwx[0]) / (pw[split] - pw[0]);
  res.mu2 = (pwx[m] - pwx[split]) / (pw[m] - pw[split]);
  res.t_r = res.mu2;
  res.t_s = res.t_r - delta_pd;
  return res;
}

// segmentation.cpp:361-390
Labels ccl(const Labels& mask, int conn) {
  const int h = mask.h, w = mask.w, nd = conn == 4 ? 4 : 8;
  Labels out(h, w, 0);
  int next = 0;
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      if (mask(v, u) == 0 || out(v, u) != 0) continue;
      ++next;
      std::deque<std::array<int, 2>> q{{u, v}};
      out(v, u) = next;
      while (!q.empty()) {
        const auto [pu, pv] = q.front();
        q.pop_front();
        for (int i = 0; i < nd; ++i) {
          const int nu = pu + kDU[i], nv = pv + kDV[i];
          if (nu < 0 || nu >= w || nv < 0 || nv >= h) continue;
          if (mask(nv, nu) != 0 && out(nv, nu) == 0) {
            out(nv, nu) = next;
            q.push_back({nu, nv});
          }
        }
      }
    }
  return out;
}

// segmentation.cpp:392-434
Labels detect(const Disp& d3, const Labels& sp_labels, double spacing, const rpd_threshold& thr,
              int margin, int min_sp, int conn) {
  const int h = d3.h, w = d3.w;
  Labels mask(h, w, 0);
  for (size_t i = 0; i < d3.a.size(); ++i)
    if (valid(d3.a[i]) && d3.a[i] < thr.t_s) mask.a[i] = 1;
  const Labels comp = ccl(mask, conn);
  const int nc = comp.a.empty() ? 0 : *std::max_element(comp.a.begin(), comp.a.end());
  std::vector<char> border(size_t(nc) + 1, 0);
  std::vector<int64_t> area(size_t(nc) + 1, 0);
  std::vector<std::map<int, char>> sps(size_t(nc) + 1);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const int c = comp(v, u);
      if (c == 0) continue;
      ++area[size_t(c)];
      sps[size_t(c)][sp_labels(v, u)] = 1;
      if (u < margin || u >= w - margin || v < margin || v >= h - margin) border[size_t(c)] = 1;
    }
  const int64_t min_area = int64_t(spacing * spacing);
  std::vector<int> relabel(size_t(nc) + 1, 0);
  Labels out(h, w, 0);
  int next = 0;
  for (size_t i = 0; i < comp.a.size(); ++i) {
    const int c = comp.a[i];
    if (c == 0) continue;
    if (border[size_t(c)] || area[size_t(c)] < min_area || int(sps[size_t(c)].size()) < min_sp)
      continue;
    if (relabel[size_t(c)] == 0) relabel[size_t(c)] = ++next;
    out.a[i] = relabel[size_t(c)];
  }
  return out;
}

// ------------------------------------------------------------ pipeline ----
// pipeline.cpp:25-34
Gray half(const Gray& img) {
  const int h = img.h / 2, w = img.w / 2;
  Gray out(h, w);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u)
      out(v, u) = 0.25f * (img(2 * v, 2 * u) + img(2 * v, 2 * u + 1) + img(2 * v + 1, 2 * u) +
                           img(2 * v + 1, 2 * u + 1));
  return out;
}

}  // namespace oracle

// ===================================================================== ABI ==
using namespace oracle;

struct rpd_ctx {
  std::string err;
};

namespace {

Gray to_gray(const float* p, int h, int w) {
  Gray g(h, w);
  std::memcpy(g.a.data(), p, sizeof(float) * g.a.size());
  return g;
}
void put(float* dst, const Raster<float>& r) {
  if (dst) std::memcpy(dst, r.a.data(), sizeof(float) * r.a.size());
}
void put(int32_t* dst, const Raster<int>& r) {
  if (dst) std::memcpy(dst, r.a.data(), sizeof(int32_t) * r.a.size());
}
Obs to_obs(const double* d, const double* u, const double* v, int64_t k) {
  Obs o;
  o.d.assign(d, d + k);
  o.u.assign(u, u + k);
  o.v.assign(v, v + k);
  return o;
}

// caller buffer too small (RPD_ECAPACITY)
struct Capacity : std::logic_error {
  using std::logic_error::logic_error;
};

template <typename F>
rpd_status guard(rpd_ctx* ctx, F&& f) {
  try {
    f();
    if (ctx) ctx->err.clear();
    return RPD_OK;
  } catch (const Capacity& e) {
    if (ctx) ctx->err = e.what();
    return RPD_ECAPACITY;
  } catch (const std::invalid_argument& e) {
    if (ctx) ctx->err = e.what();
    return RPD_EINVAL;
  } catch (const std::runtime_error& e) {
    if (ctx) ctx->err = e.what();
    return RPD_EDEGENERATE;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "out of memory";
    return RPD_ENOMEM;
  }
}

void check_dims(int h, int w) {
  if (h <= 0 || w <= 0) throw std::invalid_argument("image dimensions must be positive");
}

rpd_status detect_impl(rpd_ctx* ctx, const Gray& left, const Gray& right, const rpd_config* cfg,
                       rpd_detect_out* out) {
  return guard(ctx, [&] {
    const rpd_config& c = *cfg;
    config_validate(c);
    if (left.h != right.h || left.w != right.w)
      throw std::invalid_argument("match_pair: dimension mismatch");
    // pipeline.cpp:57-63 bootstrap at half resolution with a flat model
    const bool halve = left.h >= 64 && left.w >= 64;
    rpd_config boot = c;
    if (halve) boot.d_max = (c.d_max + 1) / 2;
    Match bootm = halve ? match_pair(half(left), half(right), Model{}, boot, boot.d_max)
                        : match_pair(left, right, Model{}, c, c.d_max);
    RoadFit coarse;
    try {
      coarse = fit_road(sample(bootm.d1, nullptr, 100000), c.roll_bracket, c.roll_tol);
    } catch (const std::runtime_error& e) {
      throw Degenerate(std::string("road fit failed: ") + e.what());
    }
    if (halve) coarse.model.a0 *= 2.0;
    Match pt = match_pair(left, right, coarse.model, c, c.d_max_pt);
    RoadFit fit;
    try {
      fit = fit_road(sample(pt.d1, nullptr, 100000), c.roll_bracket, c.roll_tol);
    } catch (const std::runtime_error& e) {
      throw Degenerate(std::string("road refit failed: ") + e.what());
    }
    int64_t clamped = 0;
    Disp d2 = transform(pt.d1, fit.model, c.delta_dt, &clamped);
    Superpixels sp = slic(d2, c.superpixels, c.compactness, c.slic_iterations);
    Disp d3 = pool(d2, sp.labels, sp.count);
    Hist hist = histogram(d2, c.hist_bin_width);
    rpd_threshold thr = threshold(hist, c.delta_pd, c.tau_diag);
    Labels lab = detect(d3, sp.labels, sp.spacing, thr, c.border_margin, c.min_superpixels,
                        c.connectivity);
    put(out->d0, pt.d0);
    put(out->d1, pt.d1);
    put(out->d2, d2);
    put(out->d3, d3);
    put(out->labels, lab);
    put(out->sp_labels, sp.labels);
    if (out->centers)
      for (int k = 0; k < std::min(out->centers_cap, sp.count); ++k)
        out->centers[k] = {sp.centers[size_t(k)].cu, sp.centers[size_t(k)].cv,
                           sp.centers[size_t(k)].value};
    out->sp_count = sp.count;
    out->sp_spacing = sp.spacing;
    out->coarse_fit = {{coarse.model.a0, coarse.model.a1, coarse.model.phi}, coarse.e0min,
                       coarse.used};
    out->fit = {{fit.model.a0, fit.model.a1, fit.model.phi}, fit.e0min, fit.used};
    out->threshold = thr;
    out->clamped = clamped;
    out->n_potholes = lab.a.empty() ? 0 : *std::max_element(lab.a.begin(), lab.a.end());
    for (double& s : out->stage_ms) s = 0.0;
    out->total_ms = 0.0;
  });
}

}  // namespace

extern "C" {

int rpd_abi_version(void) { return RPD_ABI_VERSION; }

rpd_status rpd_ctx_create(int, int, int, int, rpd_ctx** out) {
  if (!out) return RPD_EINVAL;
  *out = new rpd_ctx();
  return RPD_OK;
}
void rpd_ctx_destroy(rpd_ctx* ctx) { delete ctx; }
const char* rpd_last_error(const rpd_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }
void* rpd_ctx_stream(rpd_ctx*) { return nullptr; }

void rpd_config_default(rpd_config* cfg) { config_default(cfg); }

rpd_status rpd_config_validate(rpd_ctx* ctx, const rpd_config* cfg) {
  return guard(ctx, [&] { config_validate(*cfg); });
}

rpd_status rpd_config_set(rpd_ctx* ctx, rpd_config* c, const char* key_c, const char* val_c) {
  return guard(ctx, [&] {  // config.cpp:24-51
    const std::string key = key_c, value = val_c;
    auto d = [&] { return std::stod(value); };
    auto i = [&] { return std::stoi(value); };
    if (key == "delta_pt") c->delta_pt = d();
    else if (key == "delta_dt") c->delta_dt = d();
    else if (key == "delta_pd") c->delta_pd = d();
    else if (key == "d_max") c->d_max = i();
    else if (key == "d_max_pt") c->d_max_pt = i();
    else if (key == "lambda1") c->lambda1 = d();
    else if (key == "lambda2") c->lambda2 = d();
    else if (key == "census_window") c->census_window = i();
    else if (key == "lr_threshold") c->lr_threshold = d();
    else if (key == "superpixels") c->superpixels = i();
    else if (key == "compactness") c->compactness = d();
    else if (key == "slic_iterations") c->slic_iterations = i();
    else if (key == "hist_bin_width") c->hist_bin_width = d();
    else if (key == "tau_diag") c->tau_diag = d();
    else if (key == "border_margin") c->border_margin = i();
    else if (key == "min_superpixels") c->min_superpixels = i();
    else if (key == "connectivity") c->connectivity = i();
    else if (key == "roll_bracket") c->roll_bracket = d();
    else if (key == "roll_tol") c->roll_tol = d();
    else if (key == "focal") c->focal = d();
    else if (key == "baseline") c->baseline = d();
    else if (key == "cu") c->cu = d();
    else if (key == "cv") c->cv = d();
    else if (key == "sgm_paths") c->sgm_paths = i();
    else throw std::invalid_argument("config: unknown key '" + key + "'");
  });
}

rpd_status rpd_detect(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                      const rpd_config* cfg, rpd_detect_out* out) {
  if (h <= 0 || w <= 0) {
    if (ctx) ctx->err = "image dimensions must be positive";
    return RPD_EINVAL;
  }
  return detect_impl(ctx, to_gray(left, h, w), to_gray(right, h, w), cfg, out);
}

rpd_status rpd_detect_u8(rpd_ctx* ctx, const uint8_t* left, const uint8_t* right, int h, int w,
                         const rpd_config* cfg, rpd_detect_out* out) {
  if (h <= 0 || w <= 0) {
    if (ctx) ctx->err = "image dimensions must be positive";
    return RPD_EINVAL;
  }
  Gray l(h, w), r(h, w);
  for (size_t i = 0; i < l.a.size(); ++i) {
    l.a[i] = float(left[i]);
    r.a[i] = float(right[i]);
  }
  return detect_impl(ctx, l, r, cfg, out);
}

rpd_status rpd_compute_row_shifts(rpd_ctx* ctx, const rpd_road_model* m, int w, int h,
                                  double delta_pt, double* shifts) {
  return guard(ctx, [&] {
    const Shifts t = row_shifts({m->a0, m->a1, m->phi}, w, h, delta_pt);
    std::copy(t.s.begin(), t.s.end(), shifts);
  });
}

rpd_status rpd_warp_right_image(rpd_ctx* ctx, const float* right, int h, int w,
                                const double* shifts, float* image, uint8_t* in_view) {
  return guard(ctx, [&] {
    check_dims(h, w);
    Shifts t;
    t.s.assign(shifts, shifts + h);
    const Warped wr = warp(to_gray(right, h, w), t);
    put(image, wr.img);
    if (in_view) std::memcpy(in_view, wr.in_view.a.data(), wr.in_view.a.size());
  });
}

rpd_status rpd_restore_disparity(rpd_ctx* ctx, const float* d0, int h, int w,
                                 const double* shifts, float* d1) {
  return guard(ctx, [&] {
    check_dims(h, w);
    Shifts t;
    t.s.assign(shifts, shifts + h);
    put(d1, restore(to_gray(d0, h, w), t));
  });
}

rpd_status rpd_census_cost_volume(rpd_ctx* ctx, const float* left, const float* right, int h,
                                  int w, int d_max, int window, const uint8_t* in_view,
                                  float* costs) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (d_max < 0) throw std::invalid_argument("census_cost_volume: d_max must be >= 0");
    Raster<uint8_t> iv;
    if (in_view) {
      iv = Raster<uint8_t>(h, w);
      std::memcpy(iv.a.data(), in_view, iv.a.size());
    }
    const Volume vol =
        cost_volume(to_gray(left, h, w), to_gray(right, h, w), d_max, window, in_view ? &iv : nullptr);
    std::memcpy(costs, vol.c.data(), sizeof(float) * vol.c.size());
  });
}

static Volume to_volume(const float* costs, int h, int w, int d_max) {
  if (h <= 0 || w <= 0 || d_max < 0) throw std::invalid_argument("cost volume: bad dimensions");
  Volume v(w, h, d_max);
  std::memcpy(v.c.data(), costs, sizeof(float) * v.c.size());
  return v;
}

rpd_status rpd_aggregate_costs(rpd_ctx* ctx, const float* costs, int h, int w, int d_max,
                               const int32_t* dirs, int ndirs, float l1, float l2, float* agg) {
  return guard(ctx, [&] {
    Dirs ds;
    for (int i = 0; i < ndirs; ++i) ds.push_back({dirs[2 * i], dirs[2 * i + 1]});
    const Volume out = aggregate(to_volume(costs, h, w, d_max), ds, l1, l2);
    std::memcpy(agg, out.c.data(), sizeof(float) * out.c.size());
  });
}

rpd_status rpd_swap_reference(rpd_ctx* ctx, const float* costs, int h, int w, int d_max,
                              float* right_costs) {
  return guard(ctx, [&] {
    const Volume out = swap_ref(to_volume(costs, h, w, d_max));
    std::memcpy(right_costs, out.c.data(), sizeof(float) * out.c.size());
  });
}

rpd_status rpd_select_disparity(rpd_ctx* ctx, const float* agg, int h, int w, int d_max,
                                float* disp) {
  return guard(ctx, [&] { put(disp, wta(to_volume(agg, h, w, d_max))); });
}

rpd_status rpd_consistency_filter(rpd_ctx* ctx, float* left, const float* right, int h, int w,
                                  double thr) {
  return guard(ctx, [&] {
    check_dims(h, w);
    Disp l = to_gray(left, h, w);
    lr_check(l, to_gray(right, h, w), thr);
    put(left, l);
  });
}

rpd_status rpd_match_pair(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                          const rpd_road_model* m, const rpd_config* cfg, int d_max, float* d0,
                          float* d1, double* shifts) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (cfg->sgm_paths != 4 && cfg->sgm_paths != 8)
      throw std::invalid_argument("config: sgm_paths must be 4 or 8");
    const Match r = match_pair(to_gray(left, h, w), to_gray(right, h, w), {m->a0, m->a1, m->phi},
                               *cfg, d_max);
    put(d0, r.d0);
    put(d1, r.d1);
    if (shifts) std::copy(r.shifts.s.begin(), r.shifts.s.end(), shifts);
  });
}

rpd_status rpd_match_pair_dump(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                               const rpd_road_model* m, const rpd_config* cfg, int d_max,
                               float* cost, float* agg_left, float* agg_right, float* disp_left,
                               float* disp_right) {
  return guard(ctx, [&] {  // the intermediates of sgm.cpp:179-194
    check_dims(h, w);
    const Shifts t = row_shifts({m->a0, m->a1, m->phi}, w, h, cfg->delta_pt);
    const Warped wr = warp(to_gray(right, h, w), t);
    const Dirs dirs = config_dirs(*cfg);
    const float l1 = float(cfg->lambda1), l2 = float(cfg->lambda2);
    const Volume raw =
        cost_volume(to_gray(left, h, w), wr.img, d_max, cfg->census_window, &wr.in_view);
    const Volume al = aggregate(raw, dirs, l1, l2);
    const Volume ar = aggregate(swap_ref(raw), dirs, l1, l2);
    if (cost) std::memcpy(cost, raw.c.data(), sizeof(float) * raw.c.size());
    if (agg_left) std::memcpy(agg_left, al.c.data(), sizeof(float) * al.c.size());
    if (agg_right) std::memcpy(agg_right, ar.c.data(), sizeof(float) * ar.c.size());
    put(disp_left, wta(al));
    put(disp_right, wta(ar));
  });
}

rpd_status rpd_match_pair_dump_ex(rpd_ctx* ctx, const float* left, const float* right, int h,
                                  int w, const rpd_road_model* m, const rpd_config* cfg,
                                  int d_max, const rpd_sgm_dump* out) {
  const rpd_status st = rpd_match_pair_dump(ctx, left, right, h, w, m, cfg, d_max, out->cost,
                                            out->agg_left, out->agg_right, out->disp_left,
                                            out->disp_right);
  if (st != RPD_OK || !out->cost_right) return st;
  return guard(ctx, [&] {  // swap_reference of the same census volume (sgm.cpp:193)
    const Shifts t = row_shifts({m->a0, m->a1, m->phi}, w, h, cfg->delta_pt);
    const Warped wr = warp(to_gray(right, h, w), t);
    const Volume raw =
        cost_volume(to_gray(left, h, w), wr.img, d_max, cfg->census_window, &wr.in_view);
    const Volume cr = swap_ref(raw);
    std::memcpy(out->cost_right, cr.c.data(), sizeof(float) * cr.c.size());
  });
}

rpd_status rpd_sample_observations(rpd_ctx* ctx, const float* d1, int h, int w,
                                   const rpd_rect_roi* roi, int64_t cap, double* d, double* u,
                                   double* v, int64_t* count) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const Obs o = sample(to_gray(d1, h, w), roi, cap);
    std::copy(o.d.begin(), o.d.end(), d);
    std::copy(o.u.begin(), o.u.end(), u);
    std::copy(o.v.begin(), o.v.end(), v);
    *count = int64_t(o.count());
  });
}

rpd_status rpd_fit_line(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                        int64_t k, double phi, rpd_line_fit* out) {
  return guard(ctx, [&] {
    const LineFit f = fit_line(to_obs(d, u, v, k), phi);
    *out = {{f.model.a0, f.model.a1, f.model.phi}, f.e0min};
  });
}

rpd_status rpd_estimate_roll(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                             int64_t k, double lo, double hi, double tol, rpd_road_model* out) {
  return guard(ctx, [&] {
    const Model m = estimate_roll(to_obs(d, u, v, k), lo, hi, tol);
    *out = {m.a0, m.a1, m.phi};
  });
}

rpd_status rpd_fit_road(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                        int64_t k, double bracket, double tol, rpd_road_fit* out) {
  return guard(ctx, [&] {
    const RoadFit f = fit_road(to_obs(d, u, v, k), bracket, tol);
    *out = {{f.model.a0, f.model.a1, f.model.phi}, f.e0min, f.used};
  });
}

rpd_status rpd_transform_disparity(rpd_ctx* ctx, const float* d1, int h, int w,
                                   const rpd_road_model* m, double delta_dt, float* d2,
                                   int64_t* clamped) {
  return guard(ctx, [&] {
    check_dims(h, w);
    put(d2, transform(to_gray(d1, h, w), {m->a0, m->a1, m->phi}, delta_dt, clamped));
  });
}

rpd_status rpd_slic(rpd_ctx* ctx, const float* d2, int h, int w, int p, double m, int iters,
                    int32_t* labels, rpd_center* centers, int cap, int32_t* count,
                    double* spacing) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const Superpixels sp = slic(to_gray(d2, h, w), p, m, iters);
    put(labels, sp.labels);
    if (centers)
      for (int k = 0; k < std::min(cap, sp.count); ++k)
        centers[k] = {sp.centers[size_t(k)].cu, sp.centers[size_t(k)].cv,
                      sp.centers[size_t(k)].value};
    if (count) *count = sp.count;
    if (spacing) *spacing = sp.spacing;
  });
}

rpd_status rpd_pool_superpixels(rpd_ctx* ctx, const float* d2, const int32_t* lab, int count,
                                int h, int w, float* d3) {
  return guard(ctx, [&] {
    check_dims(h, w);
    Labels l(h, w);
    std::memcpy(l.a.data(), lab, sizeof(int32_t) * l.a.size());
    for (int x : l.a)
      if (x < 0 || x > count) throw std::invalid_argument("pool_superpixels: label out of range");
    put(d3, pool(to_gray(d2, h, w), l, count));
  });
}

rpd_status rpd_build_histogram(rpd_ctx* ctx, const float* d2, int h, int w, double bw,
                               int64_t* counts, int64_t cap_n, int64_t* n, double* origin,
                               int64_t* total) {
  rpd_status st = RPD_OK;
  const rpd_status g = guard(ctx, [&] {
    check_dims(h, w);
    const Hist hist = histogram(to_gray(d2, h, w), bw);
    *n = hist.n;
    *origin = hist.origin;
    *total = hist.total;
    if (hist.n > cap_n) {
      st = RPD_ECAPACITY;
      if (ctx) ctx->err = "build_histogram: counts buffer too small";
      return;
    }
    if (counts) std::copy(hist.counts.begin(), hist.counts.end(), counts);
  });
  return g != RPD_OK ? g : st;
}

rpd_status rpd_find_road_threshold(rpd_ctx* ctx, const int64_t* counts, int64_t n, double bw,
                                   double origin, int64_t total, double delta_pd, double tau,
                                   rpd_threshold* out) {
  return guard(ctx, [&] {
    Hist hist;
    hist.bw = bw;
    hist.origin = origin;
    hist.n = n;
    hist.total = total;
    hist.counts.assign(counts, counts + n * n);
    *out = threshold(hist, delta_pd, tau);
  });
}

rpd_status rpd_connected_components(rpd_ctx* ctx, const int32_t* mask, int h, int w, int conn,
                                    int32_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    Labels m(h, w);
    std::memcpy(m.a.data(), mask, sizeof(int32_t) * m.a.size());
    put(out, ccl(m, conn));
  });
}

rpd_status rpd_detect_potholes(rpd_ctx* ctx, const float* d3, const int32_t* sp_labels,
                               double spacing, int h, int w, const rpd_threshold* thr,
                               int margin, int min_sp, int conn, int32_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    Labels l(h, w);
    std::memcpy(l.a.data(), sp_labels, sizeof(int32_t) * l.a.size());
    put(out, detect(to_gray(d3, h, w), l, spacing, *thr, margin, min_sp, conn));
  });
}

// ---- evaluation.hpp:14-149, restated sequentially (raster order) ----------
rpd_status rpd_pep(rpd_ctx* ctx, const float* est, const float* gt, int h, int w, double eps,
                   double* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    long q = 0, bad = 0;
    for (long i = 0; i < long(h) * w; ++i) {
      if (!valid(est[i]) || !valid(gt[i])) continue;
      ++q;
      if (std::abs(static_cast<double>(est[i]) - gt[i]) > eps) ++bad;
    }
    if (q == 0) throw Degenerate("pep: no overlapping valid pixels");
    *out = 100.0 * static_cast<double>(bad) / static_cast<double>(q);
  });
}

rpd_status rpd_rmse(rpd_ctx* ctx, const float* est, const float* gt, int h, int w, double* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    long q = 0;
    double sum = 0.0;
    for (long i = 0; i < long(h) * w; ++i) {
      if (!valid(est[i]) || !valid(gt[i])) continue;
      ++q;
      const double e = static_cast<double>(est[i]) - gt[i];
      sum += e * e;
    }
    if (q == 0) throw Degenerate("rmse: no overlapping valid pixels");
    *out = std::sqrt(sum / static_cast<double>(q));
  });
}

double rpd_fscore(double precision, double recall) {
  const double s = precision + recall;
  return s > 0 ? 2.0 * precision * recall / s : 0.0;
}

rpd_status rpd_pixel_metrics(rpd_ctx* ctx, const int32_t* pred, const int32_t* gt_mask, int h,
                             int w, rpd_pixel_report* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    rpd_pixel_report m{};
    for (long i = 0; i < long(h) * w; ++i) {
      const bool p = pred[i] != 0, g = gt_mask[i] != 0;
      if (p && g) ++m.counts.n_tp;
      else if (p) ++m.counts.n_fp;
      else if (g) ++m.counts.n_fn;
      else ++m.counts.n_tn;
    }
    const rpd_confusion& c = m.counts;
    const long total = long(c.n_tp + c.n_fp + c.n_fn + c.n_tn);
    m.degenerate_precision = c.n_tp + c.n_fp == 0;
    m.degenerate_recall = c.n_tp + c.n_fn == 0;
    m.precision = m.degenerate_precision ? 0.0 : static_cast<double>(c.n_tp) / double(c.n_tp + c.n_fp);
    m.recall = m.degenerate_recall ? 0.0 : static_cast<double>(c.n_tp) / double(c.n_tp + c.n_fn);
    m.accuracy = total > 0 ? static_cast<double>(c.n_tp + c.n_tn) / double(total) : 0.0;
    m.fscore = rpd_fscore(m.precision, m.recall);
    *out = m;
  });
}

rpd_status rpd_instance_metrics(rpd_ctx* ctx, const int32_t* pred, const int32_t* gt, int h, int w,
                                double iou_min, rpd_instance_report* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const long n = long(h) * w;
    int np = 0, ng = 0;
    for (long i = 0; i < n; ++i) {
      np = std::max(np, pred[i]);
      ng = std::max(ng, gt[i]);
    }
    std::vector<long> area_p(size_t(np) + 1, 0), area_g(size_t(ng) + 1, 0);
    std::vector<std::vector<long>> inter(size_t(np) + 1, std::vector<long>(size_t(ng) + 1, 0));
    for (long i = 0; i < n; ++i) {
      const int p = pred[i], g = gt[i];
      if (p > 0) ++area_p[size_t(p)];
      if (g > 0) ++area_g[size_t(g)];
      if (p > 0 && g > 0) ++inter[size_t(p)][size_t(g)];
    }
    struct Pair {
      double iou;
      int p, g;
    };
    std::vector<Pair> pairs;
    for (int p = 1; p <= np; ++p)
      for (int g = 1; g <= ng; ++g) {
        const long i = inter[size_t(p)][size_t(g)];
        if (i == 0) continue;
        pairs.push_back({static_cast<double>(i) /
                             static_cast<double>(area_p[size_t(p)] + area_g[size_t(g)] - i),
                         p, g});
      }
    std::sort(pairs.begin(), pairs.end(), [](const Pair& a, const Pair& b) {
      if (a.iou != b.iou) return a.iou > b.iou;
      if (a.p != b.p) return a.p < b.p;
      return a.g < b.g;
    });
    std::vector<char> used_p(size_t(np) + 1, 0), used_g(size_t(ng) + 1, 0);
    rpd_instance_report rep{0, 0, 0};
    for (const auto& pr : pairs) {
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

// ---- road_geometry.cpp:153-188, restated sequentially ----------------------
static std::vector<rpd_point3> reproject_seq(const float* d1, const int32_t* labels, int label,
                                             int h, int w, const rpd_stereo_rig& rig) {
  if (rig.focal <= 0 || rig.baseline <= 0) throw std::invalid_argument("reproject: bad rig");
  std::vector<rpd_point3> cloud;
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const long i = long(v) * w + u;
      const float d = (labels && labels[i] != label) ? kInvalid : d1[i];
      if (!valid(d) || d <= 0.0f) continue;
      const double z = rig.focal * rig.baseline / d;
      cloud.push_back({static_cast<float>((u - rig.cu) * z / rig.focal),
                       static_cast<float>((v - rig.cv) * z / rig.focal), static_cast<float>(z)});
    }
  return cloud;
}

rpd_stereo_rig rpd_rig_from_config(const rpd_config* cfg, int width, int height) {
  rpd_stereo_rig r{700.0, 0.12, 0.0, 0.0};
  if (!cfg) return r;
  r.focal = cfg->focal;
  r.baseline = cfg->baseline;
  r.cu = cfg->cu >= 0 ? cfg->cu : width / 2.0;
  r.cv = cfg->cv >= 0 ? cfg->cv : height / 2.0;
  return r;
}

static void put_cloud(const std::vector<rpd_point3>& c, rpd_point3* out, int64_t cap, int64_t* n) {
  *n = int64_t(c.size());
  const size_t k = std::min<size_t>(c.size(), size_t(std::max<int64_t>(cap, 0)));
  if (k) std::memcpy(out, c.data(), sizeof(rpd_point3) * k);
  if (int64_t(c.size()) > cap) throw Capacity("reproject: more points than cap");
}

rpd_status rpd_reproject(rpd_ctx* ctx, const float* d1, int h, int w, const rpd_stereo_rig* rig,
                         rpd_point3* out, int64_t cap, int64_t* n) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (!rig) throw std::invalid_argument("reproject: null rig");
    put_cloud(reproject_seq(d1, nullptr, 0, h, w, *rig), out, cap, n);
  });
}

rpd_status rpd_reproject_masked(rpd_ctx* ctx, const float* d1, const int32_t* labels, int h,
                                int w, int label, const rpd_stereo_rig* rig, rpd_point3* out,
                                int64_t cap, int64_t* n) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (!rig) throw std::invalid_argument("reproject: null rig");
    put_cloud(reproject_seq(d1, labels, label, h, w, *rig), out, cap, n);
  });
}

rpd_status rpd_reproject_instances(rpd_ctx* ctx, const float* d1, const int32_t* labels, int h,
                                   int w, int max_label, const rpd_stereo_rig* rig,
                                   rpd_point3* out, int64_t cap, int64_t* offsets) {
  return guard(ctx, [&] {
    check_dims(h, w);
    if (!rig) throw std::invalid_argument("reproject: null rig");
    if (max_label < 0) throw std::invalid_argument("reproject_instances: max_label < 0");
    std::vector<rpd_point3> all;
    offsets[0] = 0;
    for (int k = 1; k <= max_label; ++k) {  // rpd_cli.cpp:99-104
      const auto c = reproject_seq(d1, labels, k, h, w, *rig);
      all.insert(all.end(), c.begin(), c.end());
      offsets[k] = int64_t(all.size());
    }
    int64_t n = 0;
    put_cloud(all, out, cap, &n);
  });
}

rpd_status rpd_closest_distance_error(rpd_ctx* ctx, const rpd_point3* test, int64_t n_test,
                                      const rpd_point3* truth, int64_t n_truth, double* out) {
  return guard(ctx, [&] {
    if (n_test <= 0 || n_truth <= 0)
      throw std::invalid_argument("closest_distance_error: empty cloud");
    double sum = 0.0;
    for (int64_t i = 0; i < n_test; ++i) {
      const rpd_point3& p = test[i];
      double best = std::numeric_limits<double>::infinity();
      for (int64_t j = 0; j < n_truth; ++j) {
        const rpd_point3& g = truth[j];
        const double dx = p.x - g.x, dy = p.y - g.y, dz = p.z - g.z;
        best = std::min(best, dx * dx + dy * dy + dz * dz);
      }
      sum += best;
    }
    *out = std::sqrt(sum / static_cast<double>(n_test));
  });
}

// ---- image_io.cpp:171-339 per-pixel transforms, restated --------------------
rpd_status rpd_encode_disparity_u16(rpd_ctx* ctx, const float* d, int h, int w, uint16_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    for (long i = 0; i < long(h) * w; ++i) {
      std::uint16_t s = 0;
      if (valid(d[i])) {
        const double scaled = std::round(static_cast<double>(d[i]) * 256.0);
        if (scaled < 0 || scaled > 65535) throw std::runtime_error("disparity exceeds encoding range");
        s = static_cast<std::uint16_t>(scaled);
      }
      out[i] = s;
    }
  });
}

rpd_status rpd_decode_disparity_u16(rpd_ctx* ctx, const uint16_t* s, int h, int w, float* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    for (long i = 0; i < long(h) * w; ++i)
      out[i] = s[i] == 0 ? kInvalid : static_cast<float>(s[i]) / 256.0f;
  });
}

rpd_status rpd_encode_labels_u16(rpd_ctx* ctx, const int32_t* labels, int h, int w,
                                 uint16_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    for (long i = 0; i < long(h) * w; ++i) {
      const int k = labels[i];
      if (k < 0 || k > 65535) throw std::runtime_error("label exceeds encoding range");
      out[i] = static_cast<std::uint16_t>(k);
    }
  });
}

static unsigned char round_clamp_u8(float x) {
  return static_cast<unsigned char>(std::clamp(std::round(x), 0.0f, 255.0f));
}

rpd_status rpd_encode_gray_u8(rpd_ctx* ctx, const float* img, int h, int w, uint8_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    for (long i = 0; i < long(h) * w; ++i) out[i] = round_clamp_u8(img[i]);
  });
}

rpd_status rpd_gray_from_rgb8(rpd_ctx* ctx, const uint8_t* rgb, int h, int w, float* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    for (long i = 0; i < long(h) * w; ++i) {
      const std::uint16_t r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
      out[i] = 0.299f * r + 0.587f * g + 0.114f * b;
    }
  });
}

rpd_status rpd_overlay_rgb8(rpd_ctx* ctx, const float* img, const int32_t* labels, int h, int w,
                            uint8_t* rgb) {
  static const unsigned char kPalette[12][3] = {
      {230, 25, 75},  {60, 180, 75},  {255, 225, 25}, {0, 130, 200},  {245, 130, 48},
      {145, 30, 180}, {70, 240, 240}, {240, 50, 230}, {210, 245, 60}, {250, 190, 190},
      {0, 128, 128},  {170, 110, 40}};
  return guard(ctx, [&] {
    check_dims(h, w);
    for (long i = 0; i < long(h) * w; ++i) {
      const float gray = img[i];
      const unsigned char g = round_clamp_u8(gray);
      unsigned char c[3] = {g, g, g};
      if (labels[i] > 0) {
        const unsigned char* p = kPalette[(labels[i] - 1) % 12];
        for (int ch = 0; ch < 3; ++ch) c[ch] = round_clamp_u8((gray + p[ch]) * 0.5f);
      }
      rgb[3 * i] = c[0];
      rgb[3 * i + 1] = c[1];
      rgb[3 * i + 2] = c[2];
    }
  });
}

// ---- synth.cpp:16-196 scene generator, restated sequentially -------------
// std::mt19937 with libstdc++'s uniform_real_distribution / normal_distribution
// (the streams the reference draws from); row-major float rasters.
}  // extern "C"

namespace {

// value_noise (synth.cpp:16-38): one octave, bilinear over a random lattice.
void add_value_noise(std::vector<float>& tex, int w, int h, int spacing, float amp,
                     std::mt19937& rng) {
  const int nu = w / spacing + 2, nv = h / spacing + 2;
  std::vector<float> lat(static_cast<size_t>(nu) * nv);
  std::uniform_real_distribution<float> uni(0.0f, 1.0f);
  for (auto& x : lat) x = uni(rng);  // row j outer, column i inner
  for (int v = 0; v < h; ++v) {
    const double y = static_cast<double>(v) / spacing;
    const int j = static_cast<int>(y);
    const double ty = y - j;
    for (int u = 0; u < w; ++u) {
      const double x = static_cast<double>(u) / spacing;
      const int i = static_cast<int>(x);
      const double tx = x - i;
      const double top = (1 - tx) * lat[size_t(j) * nu + i] + tx * lat[size_t(j) * nu + i + 1];
      const double bot =
          (1 - tx) * lat[size_t(j + 1) * nu + i] + tx * lat[size_t(j + 1) * nu + i + 1];
      const float n = static_cast<float>((1 - ty) * top + ty * bot);
      tex[size_t(v) * w + u] += amp * n;  // tex += amps[o] * value_noise (:65)
    }
  }
}

// binomial_smooth_5x5 (synth.cpp:40-58), clamped borders.
std::vector<float> binomial5(const std::vector<float>& img, int w, int h) {
  static const double k[5] = {1, 4, 6, 4, 1};
  std::vector<float> tmp(img.size()), out(img.size());
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      double s = 0;
      for (int i = -2; i <= 2; ++i) s += k[i + 2] * img[size_t(v) * w + std::clamp(u + i, 0, w - 1)];
      tmp[size_t(v) * w + u] = static_cast<float>(s / 16.0);
    }
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      double s = 0;
      for (int i = -2; i <= 2; ++i) s += k[i + 2] * tmp[size_t(std::clamp(v + i, 0, h - 1)) * w + u];
      out[size_t(v) * w + u] = static_cast<float>(s / 16.0);
    }
  return out;
}

// Linear interpolation along row v at column s, clamped (synth.cpp:74-91).
template <typename T>
double row_lerp(const T* row, int w, double s) {
  s = std::clamp(s, 0.0, static_cast<double>(w - 1));
  const int s0 = static_cast<int>(s);
  const int s1 = std::min(s0 + 1, w - 1);
  const double t = s - s0;
  return (1 - t) * row[s0] + t * row[s1];
}

void oracle_scene(const rpd_scene_spec& sp, float* left, float* right, float* gt, int32_t* mask) {
  const int w = sp.width, h = sp.height;
  if (w <= 0 || h <= 0) throw std::invalid_argument("generate_scene: image dimensions must be positive");
  for (int k = 0; k < sp.n_potholes; ++k) {
    const rpd_pothole_spec& p = sp.potholes[k];
    if (p.depth <= 0 || p.ru < 4 || p.rv < 4)
      throw std::invalid_argument("generate_scene: bad pothole spec");
  }
  const size_t n = size_t(h) * w;
  std::vector<float> g(n), l(n), r(n);
  std::vector<int32_t> m(n, 0);
  const double c = std::cos(sp.phi_true), s = std::sin(sp.phi_true);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      double d = sp.a0 + sp.a1 * (v * c - u * s);  // road_disparity_at (types.hpp:39-41)
      for (int k = 0; k < sp.n_potholes; ++k) {
        const rpd_pothole_spec& p = sp.potholes[k];
        const double ru = (u - p.cu) / p.ru, rv = (v - p.cv) / p.rv;
        const double r2 = ru * ru + rv * rv;
        if (r2 < 1.0) {
          d -= p.depth * (1.0 - r2);
          m[size_t(v) * w + u] = k + 1;
        }
      }
      if (d < 0) throw std::runtime_error("generate_scene: pothole depth drives disparity negative");
      g[size_t(v) * w + u] = static_cast<float>(d);
    }
  // make_texture (synth.cpp:60-72)
  std::mt19937 trng(sp.texture_seed);
  std::vector<float> tex(n, 0.0f);
  add_value_noise(tex, w, h, 64, 1.0f, trng);
  add_value_noise(tex, w, h, 16, 0.5f, trng);
  add_value_noise(tex, w, h, 4, 0.25f, trng);
  tex = binomial5(tex, w, h);
  const float lo = *std::min_element(tex.begin(), tex.end());
  const float hi = *std::max_element(tex.begin(), tex.end());
  const float scale = hi > lo ? 190.0f / (hi - lo) : 0.0f;
  for (size_t i = 0; i < n; ++i) l[i] = hi > lo ? 30.0f + (tex[i] - lo) * scale : 125.0f;
  // right view: fixed point u = x + d(v, u), 8 refinements (synth.cpp:126-137)
  for (int v = 0; v < h; ++v) {
    const float* grow = g.data() + size_t(v) * w;
    const float* lrow = l.data() + size_t(v) * w;
    for (int x = 0; x < w; ++x) {
      double u = x + row_lerp(grow, w, x);
      for (int it = 0; it < 8; ++it) u = x + row_lerp(grow, w, u);
      r[size_t(v) * w + x] = static_cast<float>(row_lerp(lrow, w, u));
    }
  }
  if (sp.noise_sigma > 0) {  // synth.cpp:139-146
    std::mt19937 nrng(sp.texture_seed ^ 0x9e3779b9u);
    std::normal_distribution<double> gauss(0.0, sp.noise_sigma);
    for (size_t i = 0; i < n; ++i) {
      l[i] = std::clamp(l[i] + static_cast<float>(gauss(nrng)), 0.0f, 255.0f);
      r[i] = std::clamp(r[i] + static_cast<float>(gauss(nrng)), 0.0f, 255.0f);
    }
  }
  if (left) std::memcpy(left, l.data(), sizeof(float) * n);
  if (right) std::memcpy(right, r.data(), sizeof(float) * n);
  if (gt) std::memcpy(gt, g.data(), sizeof(float) * n);
  if (mask) std::memcpy(mask, m.data(), sizeof(int32_t) * n);
}

}  // namespace

extern "C" {

void rpd_scene_spec_default(rpd_scene_spec* s) {  // synth.hpp:20-30
  *s = rpd_scene_spec{};
  s->width = 640;
  s->height = 480;
  s->rig = rpd_stereo_rig{700.0, 0.12, 0.0, 0.0};
  s->a0 = 5.0;
  s->a1 = 0.08;
  s->texture_seed = 1;
}

void rpd_batch_ranges_default(rpd_batch_ranges* r) {  // synth.hpp:45-53
  *r = rpd_batch_ranges{1.5, 4.0, 22.0, 48.0, 4.0, 7.0, 0.07, 0.09, 0.035, 0.0, 40};
}

rpd_status rpd_scene_batch_spec(uint32_t base_seed, int32_t index, const rpd_batch_ranges* r,
                                rpd_scene_spec* spec, rpd_pothole_spec potholes[3]) {
  if (index < 0 || !r || !spec || !potholes) return RPD_EINVAL;
  const uint32_t seed = base_seed + static_cast<uint32_t>(index);  // synth.cpp:157-191
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
  int placed = 0;
  const int wanted = 1 + static_cast<int>(uni(rng) * 3.0) % 3;
  for (int k = 0; k < wanted; ++k)
    for (int attempt = 0; attempt < 100; ++attempt) {
      rpd_pothole_spec p{};
      p.ru = r->radius_min + (r->radius_max - r->radius_min) * uni(rng);
      p.rv = r->radius_min + (r->radius_max - r->radius_min) * uni(rng);
      p.depth = r->depth_min + (r->depth_max - r->depth_min) * uni(rng);
      const double mu = r->margin + p.ru, mv = r->margin + p.rv;
      p.cu = mu + (spec->width - 2 * mu) * uni(rng);
      p.cv = mv + (spec->height - 2 * mv) * uni(rng);
      bool clash = false;
      for (int q = 0; q < placed; ++q) {
        const double dx = p.cu - potholes[q].cu, dy = p.cv - potholes[q].cv;
        const double sep = std::max(p.ru + potholes[q].ru, p.rv + potholes[q].rv) + 10.0;
        clash |= dx * dx + dy * dy < sep * sep;
      }
      if (!clash) {
        potholes[placed++] = p;
        break;
      }
    }
  spec->n_potholes = placed;
  spec->potholes = potholes;
  return RPD_OK;
}

rpd_status rpd_generate_scene(rpd_ctx* ctx, const rpd_scene_spec* spec, float* left,
                              float* right, float* gt_disparity, int32_t* gt_mask) {
  return guard(ctx, [&] {
    if (!spec) throw std::invalid_argument("generate_scene: null spec");
    oracle_scene(*spec, left, right, gt_disparity, gt_mask);
  });
}

}  // extern "C"

