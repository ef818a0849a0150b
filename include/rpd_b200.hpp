// rpd_b200.hpp — header-only C++17 drop-in for the reference `namespace rpd`
// hot path (/root/reference/proj/include/rpd/*.hpp), implemented over the
// C-ABI of include/rpd_b200.h (link with -lrpd_b200).
//
// Same function names, argument meaning, result types and exception types
// (std::invalid_argument, std::runtime_error, DegenerateFitError).  The only
// representational change: rasters are a small row-major std::vector raster
// instead of Eigen arrays (Eigen is not a dependency of this library); index
// (v, u) = v*W + u exactly like Raster<T> (types.hpp:9-10).
//
// Each calling thread gets its own device context (rpd_ctx) on the current
// device, created lazily: functions are reentrant like the reference's.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "rpd_b200.h"

namespace rpd_b200 {

// ------------------------------------------------------------------- types --
template <typename T>
struct Raster {  // types.hpp:9-10 (row-major, (v, u))
  std::vector<T> data;
  int h = 0, w = 0;
  Raster() = default;
  Raster(int rows, int cols, T fill = T{}) : data(size_t(rows) * cols, fill), h(rows), w(cols) {}
  static Raster Constant(int rows, int cols, T v) { return Raster(rows, cols, v); }
  static Raster Zero(int rows, int cols) { return Raster(rows, cols, T{}); }
  int rows() const { return h; }
  int cols() const { return w; }
  T& operator()(int v, int u) { return data[size_t(v) * w + u]; }
  const T& operator()(int v, int u) const { return data[size_t(v) * w + u]; }
  T* ptr() { return data.data(); }
  const T* ptr() const { return data.data(); }
};
using GrayImage = Raster<float>;     // types.hpp:13
using DisparityMap = Raster<float>;  // types.hpp:16
using LabelMap = Raster<int>;        // types.hpp:19
inline constexpr float kInvalidDisparity = -1.0f;  // types.hpp:21
inline bool is_valid(float d) { return d != kInvalidDisparity; }

struct RoadModel {  // types.hpp:33-37
  double a0 = 0.0, a1 = 0.0, phi = 0.0;
};
inline double road_disparity_at(const RoadModel& m, double u, double v) {  // types.hpp:39-41
  return m.a0 + m.a1 * (v * std::cos(m.phi) - u * std::sin(m.phi));
}

struct DegenerateFitError : std::runtime_error {  // pipeline.hpp:17-19
  using std::runtime_error::runtime_error;
};

// PipelineConfig (config.hpp:10-36) with the `sgm_paths` extension.
struct PipelineConfig : rpd_config {
  PipelineConfig() { rpd_config_default(this); }
  void validate() const;
};

// ----------------------------------------------------------------- context --
namespace detail {
struct CtxDeleter {
  void operator()(rpd_ctx* c) const { rpd_ctx_destroy(c); }
};
inline int& device_slot() {
  thread_local int dev = 0;
  return dev;
}
inline rpd_ctx* ctx() {
  thread_local std::unique_ptr<rpd_ctx, CtxDeleter> c;
  thread_local int bound = -1;
  if (!c || bound != device_slot()) {
    rpd_ctx* raw = nullptr;
    const rpd_status st = rpd_ctx_create(device_slot(), 0, 0, 0, &raw);
    if (st != RPD_OK) throw std::runtime_error("rpd_b200: cannot create a CUDA context");
    c.reset(raw);
    bound = device_slot();
  }
  return c.get();
}
inline void check(rpd_status st) {
  if (st == RPD_OK) return;
  const std::string msg = rpd_last_error(ctx());
  switch (st) {
    case RPD_EINVAL: throw std::invalid_argument(msg);
    case RPD_EDEGENERATE:
      if (msg.rfind("road fit failed", 0) == 0 || msg.rfind("road refit failed", 0) == 0)
        throw DegenerateFitError(msg);
      throw std::runtime_error(msg);
    default: throw std::runtime_error("rpd_b200: " + msg);
  }
}
}  // namespace detail

// Selects the CUDA device used by the calling thread.
inline void set_device(int device) { detail::device_slot() = device; }

inline void PipelineConfig::validate() const { detail::check(rpd_config_validate(detail::ctx(), this)); }

inline void apply_key_value(PipelineConfig& c, const std::string& key, const std::string& value) {
  detail::check(rpd_config_set(detail::ctx(), &c, key.c_str(), value.c_str()));
}

// ------------------------------------------------------------ perspective --
struct RowShiftTable {  // perspective.hpp:15-18
  std::vector<double> shifts;
  double delta_pt = 0.0;
};
inline RowShiftTable compute_row_shifts(const RoadModel& m, int width, int height,
                                        double delta_pt) {
  RowShiftTable t;
  t.delta_pt = delta_pt;
  t.shifts.resize(size_t(height));
  const rpd_road_model rm{m.a0, m.a1, m.phi};
  detail::check(rpd_compute_row_shifts(detail::ctx(), &rm, width, height, delta_pt,
                                       t.shifts.data()));
  return t;
}
struct WarpResult {  // perspective.hpp:37-40
  GrayImage image;
  Raster<unsigned char> in_view;
};
inline WarpResult warp_right_image(const GrayImage& right, const RowShiftTable& t) {
  if (int(t.shifts.size()) != right.rows())
    throw std::invalid_argument("warp_right_image: table length != image height");
  WarpResult r{GrayImage(right.rows(), right.cols()),
               Raster<unsigned char>(right.rows(), right.cols())};
  detail::check(rpd_warp_right_image(detail::ctx(), right.ptr(), right.rows(), right.cols(),
                                     t.shifts.data(), r.image.ptr(), r.in_view.ptr()));
  return r;
}
inline DisparityMap restore_disparity(const DisparityMap& d0, const RowShiftTable& t) {
  if (int(t.shifts.size()) != d0.rows())
    throw std::invalid_argument("restore_disparity: table length != map height");
  DisparityMap d1(d0.rows(), d0.cols());
  detail::check(rpd_restore_disparity(detail::ctx(), d0.ptr(), d0.rows(), d0.cols(),
                                      t.shifts.data(), d1.ptr()));
  return d1;
}

// -------------------------------------------------------------------- SGM --
struct CostVolume {  // sgm.hpp:15-33
  int width = 0, height = 0, d_max = 0;
  std::vector<float> costs;
  CostVolume() = default;
  CostVolume(int w, int h, int dm)
      : width(w), height(h), d_max(dm), costs(size_t(w) * h * (dm + 1), 0.0f) {}
  int levels() const { return d_max + 1; }
  float& at(int v, int u, int d) { return costs[(size_t(v) * width + u) * levels() + d]; }
  float at(int v, int u, int d) const { return costs[(size_t(v) * width + u) * levels() + d]; }
};
struct SgmParams {  // sgm.hpp:35-44
  float lambda1 = 8.0f, lambda2 = 32.0f;
  std::vector<std::array<int, 2>> directions = kEightDirections();
  int census_window = 5;
  static std::vector<std::array<int, 2>> kEightDirections() {
    return {{{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {1, 1}, {-1, 1}, {1, -1}, {-1, -1}}};
  }
};
inline CostVolume census_cost_volume(const GrayImage& left, const GrayImage& right, int d_max,
                                     int window, const Raster<unsigned char>* in_view = nullptr) {
  if (left.rows() != right.rows() || left.cols() != right.cols())
    throw std::invalid_argument("census_cost_volume: dimension mismatch");
  if (d_max >= left.cols()) throw std::invalid_argument("census_cost_volume: d_max >= width");
  CostVolume vol(left.cols(), left.rows(), d_max);
  detail::check(rpd_census_cost_volume(detail::ctx(), left.ptr(), right.ptr(), left.rows(),
                                       left.cols(), d_max, window,
                                       in_view ? in_view->ptr() : nullptr, vol.costs.data()));
  return vol;
}
inline CostVolume aggregate_costs(const CostVolume& vol, const SgmParams& p) {
  CostVolume out(vol.width, vol.height, vol.d_max);
  std::vector<int32_t> dirs;
  for (const auto& d : p.directions) {
    dirs.push_back(d[0]);
    dirs.push_back(d[1]);
  }
  detail::check(rpd_aggregate_costs(detail::ctx(), vol.costs.data(), vol.height, vol.width,
                                    vol.d_max, dirs.data(), int(p.directions.size()), p.lambda1,
                                    p.lambda2, out.costs.data()));
  return out;
}
inline CostVolume swap_reference(const CostVolume& vol) {
  CostVolume out(vol.width, vol.height, vol.d_max);
  detail::check(rpd_swap_reference(detail::ctx(), vol.costs.data(), vol.height, vol.width,
                                   vol.d_max, out.costs.data()));
  return out;
}
inline DisparityMap select_disparity(const CostVolume& agg) {
  DisparityMap d(agg.height, agg.width);
  detail::check(rpd_select_disparity(detail::ctx(), agg.costs.data(), agg.height, agg.width,
                                     agg.d_max, d.ptr()));
  return d;
}
inline void consistency_filter(DisparityMap& left, const DisparityMap& right, double thr) {
  detail::check(rpd_consistency_filter(detail::ctx(), left.ptr(), right.ptr(), left.rows(),
                                       left.cols(), thr));
}
struct MatchResult {  // sgm.hpp:69-73
  DisparityMap d0, d1;
  RowShiftTable shifts;
};
inline MatchResult match_pair(const GrayImage& left, const GrayImage& right, const RoadModel& m,
                              const PipelineConfig& cfg, int d_max) {
  if (left.rows() != right.rows() || left.cols() != right.cols())
    throw std::invalid_argument("match_pair: dimension mismatch");
  MatchResult r{DisparityMap(left.rows(), left.cols()), DisparityMap(left.rows(), left.cols()),
                RowShiftTable{std::vector<double>(size_t(left.rows())), cfg.delta_pt}};
  const rpd_road_model rm{m.a0, m.a1, m.phi};
  detail::check(rpd_match_pair(detail::ctx(), left.ptr(), right.ptr(), left.rows(), left.cols(),
                               &rm, &cfg, d_max, r.d0.ptr(), r.d1.ptr(), r.shifts.shifts.data()));
  return r;
}

// ---------------------------------------------------------- road geometry --
struct RoadObservations {  // road_geometry.hpp:12-18
  std::vector<double> d, u, v;
  long count() const { return long(d.size()); }
};
struct LineFit {  // road_geometry.hpp:20-23
  RoadModel model;
  double e0min = 0.0;
};
struct RoadFit {  // road_geometry.hpp:34-38
  RoadModel model;
  double e0min = 0.0;
  long used = 0;
};
struct RectRoi {  // road_geometry.hpp:45-47
  int u0, v0, width, height;
};
struct TransformResult {  // road_geometry.hpp:55-58
  DisparityMap d2;
  long clamped = 0;
};
inline LineFit fit_line(const RoadObservations& o, double phi) {
  rpd_line_fit f{};
  detail::check(rpd_fit_line(detail::ctx(), o.d.data(), o.u.data(), o.v.data(), o.count(), phi, &f));
  return LineFit{{f.model.a0, f.model.a1, f.model.phi}, f.e0min};
}
inline RoadModel estimate_roll(const RoadObservations& o, double lo, double hi, double tol) {
  rpd_road_model m{};
  detail::check(rpd_estimate_roll(detail::ctx(), o.d.data(), o.u.data(), o.v.data(), o.count(),
                                  lo, hi, tol, &m));
  return RoadModel{m.a0, m.a1, m.phi};
}
inline RoadFit fit_road(const RoadObservations& o, double bracket, double tol) {
  rpd_road_fit f{};
  detail::check(rpd_fit_road(detail::ctx(), o.d.data(), o.u.data(), o.v.data(), o.count(),
                             bracket, tol, &f));
  return RoadFit{{f.model.a0, f.model.a1, f.model.phi}, f.e0min, long(f.used)};
}
inline RoadObservations sample_observations(const DisparityMap& d1, const RectRoi* roi = nullptr,
                                            long cap = 100000) {
  const size_t n = std::min<size_t>(size_t(d1.rows()) * d1.cols(), size_t(cap));
  RoadObservations o;
  o.d.resize(n);
  o.u.resize(n);
  o.v.resize(n);
  int64_t k = 0;
  rpd_rect_roi r{};
  if (roi) r = rpd_rect_roi{roi->u0, roi->v0, roi->width, roi->height};
  detail::check(rpd_sample_observations(detail::ctx(), d1.ptr(), d1.rows(), d1.cols(),
                                        roi ? &r : nullptr, cap, o.d.data(), o.u.data(),
                                        o.v.data(), &k));
  o.d.resize(size_t(k));
  o.u.resize(size_t(k));
  o.v.resize(size_t(k));
  return o;
}
inline TransformResult transform_disparity(const DisparityMap& d1, const RoadModel& m,
                                           double delta_dt) {
  TransformResult t{DisparityMap(d1.rows(), d1.cols()), 0};
  const rpd_road_model rm{m.a0, m.a1, m.phi};
  int64_t c = 0;
  detail::check(rpd_transform_disparity(detail::ctx(), d1.ptr(), d1.rows(), d1.cols(), &rm,
                                        delta_dt, t.d2.ptr(), &c));
  t.clamped = long(c);
  return t;
}

// ----------------------------------------------------------- segmentation --
struct SuperpixelMap {  // segmentation.hpp:10-20
  struct Center {
    double cu = 0.0, cv = 0.0, value = 0.0;
  };
  LabelMap labels;
  std::vector<Center> centers;
  int count = 0;
  double spacing = 0.0;
};
struct Histogram2D {  // segmentation.hpp:34-41
  double bin_width = 0.25;
  double origin = 0.0;
  Raster<long long> counts;
  long long total = 0;
  double center(long bin) const { return origin + (bin + 0.5) * bin_width; }
};
struct ThresholdResult {  // segmentation.hpp:48-55
  double t_r = 0.0, t_s = 0.0, mu1 = 0.0, mu2 = 0.0, excluded_fraction = 0.0;
  bool degenerate = false;
};
// SLIC keeps at most its nu * nv seeds (segmentation.cpp:181-184): the
// capacity of the centre records of slic() / detect_potholes_pipeline().
inline int slic_seed_count(int h, int w, int p) {
  if (h <= 0 || w <= 0 || p <= 0) return 1;
  const int nu = std::max(1, int(std::lround(std::sqrt(double(p) * w / h))));
  const int nv = std::max(1, int(std::lround(double(p) / nu)));
  return std::max(1, std::min(h * w, nu * nv));
}
inline SuperpixelMap slic(const DisparityMap& d2, int p, double compactness, int iterations) {
  SuperpixelMap sp;
  sp.labels = LabelMap(d2.rows(), d2.cols());
  const int cap = slic_seed_count(d2.rows(), d2.cols(), p);
  std::vector<rpd_center> c(static_cast<size_t>(cap));
  int32_t count = 0;
  detail::check(rpd_slic(detail::ctx(), d2.ptr(), d2.rows(), d2.cols(), p, compactness,
                         iterations, sp.labels.ptr(), c.data(), cap, &count, &sp.spacing));
  sp.count = count;
  for (int k = 0; k < std::min(count, cap); ++k)
    sp.centers.push_back({c[size_t(k)].cu, c[size_t(k)].cv, c[size_t(k)].value});
  return sp;
}
inline DisparityMap pool_superpixels(const DisparityMap& d2, const SuperpixelMap& sp) {
  if (d2.rows() != sp.labels.rows() || d2.cols() != sp.labels.cols())
    throw std::invalid_argument("pool_superpixels: dimension mismatch");
  DisparityMap d3(d2.rows(), d2.cols());
  detail::check(rpd_pool_superpixels(detail::ctx(), d2.ptr(), sp.labels.ptr(), sp.count,
                                     d2.rows(), d2.cols(), d3.ptr()));
  return d3;
}
inline Histogram2D build_histogram(const DisparityMap& d2, double bin_width) {
  Histogram2D hist;
  hist.bin_width = bin_width;
  int64_t n = 0, total = 0;
  const rpd_status st = rpd_build_histogram(detail::ctx(), d2.ptr(), d2.rows(), d2.cols(),
                                            bin_width, nullptr, 0, &n, &hist.origin, &total);
  if (st != RPD_ECAPACITY) detail::check(st);
  hist.counts = Raster<long long>(int(n), int(n));
  if (n > 0)
    detail::check(rpd_build_histogram(detail::ctx(), d2.ptr(), d2.rows(), d2.cols(), bin_width,
                                      reinterpret_cast<int64_t*>(hist.counts.ptr()), n, &n,
                                      &hist.origin, &total));
  hist.total = total;
  return hist;
}
inline ThresholdResult find_road_threshold(const Histogram2D& h, double delta_pd,
                                           double tau = 3.0) {
  rpd_threshold t{};
  detail::check(rpd_find_road_threshold(detail::ctx(),
                                        reinterpret_cast<const int64_t*>(h.counts.ptr()),
                                        h.counts.rows(), h.bin_width, h.origin, h.total, delta_pd,
                                        tau, &t));
  return ThresholdResult{t.t_r, t.t_s, t.mu1, t.mu2, t.excluded_fraction, t.degenerate != 0};
}
inline LabelMap connected_components(const LabelMap& mask, int connectivity = 8) {
  LabelMap out(mask.rows(), mask.cols());
  detail::check(rpd_connected_components(detail::ctx(), mask.ptr(), mask.rows(), mask.cols(),
                                         connectivity, out.ptr()));
  return out;
}
inline LabelMap detect_potholes(const DisparityMap& d3, const SuperpixelMap& sp,
                                const ThresholdResult& thr, int border_margin,
                                int min_superpixels, int connectivity = 8) {
  LabelMap out(d3.rows(), d3.cols());
  const rpd_threshold t{thr.t_r, thr.t_s, thr.mu1, thr.mu2, thr.excluded_fraction,
                        thr.degenerate ? 1 : 0};
  detail::check(rpd_detect_potholes(detail::ctx(), d3.ptr(), sp.labels.ptr(), sp.spacing,
                                    d3.rows(), d3.cols(), &t, border_margin, min_superpixels,
                                    connectivity, out.ptr()));
  return out;
}

// ------------------------------------------------------------- evaluation --
inline void check_same_shape(int h0, int w0, int h1, int w1, const char* what) {
  if (h0 != h1 || w0 != w1) throw std::invalid_argument(std::string(what) + ": dimension mismatch");
}
inline double pep(const DisparityMap& est, const DisparityMap& gt, double eps) {  // :14
  check_same_shape(est.rows(), est.cols(), gt.rows(), gt.cols(), "pep");
  double out = 0.0;
  detail::check(rpd_pep(detail::ctx(), est.ptr(), gt.ptr(), est.rows(), est.cols(), eps, &out));
  return out;
}
inline double rmse(const DisparityMap& est, const DisparityMap& gt) {  // :29
  check_same_shape(est.rows(), est.cols(), gt.rows(), gt.cols(), "rmse");
  double out = 0.0;
  detail::check(rpd_rmse(detail::ctx(), est.ptr(), gt.ptr(), est.rows(), est.cols(), &out));
  return out;
}
struct ConfusionCounts {  // evaluation.hpp:44-47
  long n_tp = 0, n_fp = 0, n_fn = 0, n_tn = 0;
  long total() const { return n_tp + n_fp + n_fn + n_tn; }
};
struct PixelMetrics {  // evaluation.hpp:49-57
  ConfusionCounts counts;
  double precision = 0.0, recall = 0.0, accuracy = 0.0, fscore = 0.0;
  bool degenerate_precision = false, degenerate_recall = false;
};
inline double fscore(double precision, double recall) { return rpd_fscore(precision, recall); }
inline PixelMetrics pixel_metrics(const LabelMap& pred, const LabelMap& gt_mask) {  // :69
  check_same_shape(pred.rows(), pred.cols(), gt_mask.rows(), gt_mask.cols(), "pixel_metrics");
  rpd_pixel_report r{};
  detail::check(rpd_pixel_metrics(detail::ctx(), pred.ptr(), gt_mask.ptr(), pred.rows(),
                                   pred.cols(), &r));
  PixelMetrics m;
  m.counts = {long(r.counts.n_tp), long(r.counts.n_fp), long(r.counts.n_fn), long(r.counts.n_tn)};
  m.precision = r.precision;
  m.recall = r.recall;
  m.accuracy = r.accuracy;
  m.fscore = r.fscore;
  m.degenerate_precision = r.degenerate_precision != 0;
  m.degenerate_recall = r.degenerate_recall != 0;
  return m;
}
struct InstanceReport {  // evaluation.hpp:91-95
  int correct = 0, incorrect = 0, misdetection = 0;
};
inline InstanceReport instance_metrics(const LabelMap& pred, const LabelMap& gt_instances,
                                       double iou_min = 0.5) {  // :97
  check_same_shape(pred.rows(), pred.cols(), gt_instances.rows(), gt_instances.cols(),
                   "instance_metrics");
  rpd_instance_report r{};
  detail::check(rpd_instance_metrics(detail::ctx(), pred.ptr(), gt_instances.ptr(), pred.rows(),
                                     pred.cols(), iou_min, &r));
  return InstanceReport{r.correct, r.incorrect, r.misdetection};
}

// ------------------------------------------------ 3-D reprojection + PLY --
struct StereoRig {  // types.hpp:25-30
  double focal = 700.0, baseline = 0.12, cu = 0.0, cv = 0.0;
};
struct Point3 {  // types.hpp:43-45
  float x, y, z;
};
using PointCloud = std::vector<Point3>;
inline StereoRig rig_from_config(const PipelineConfig& c, int width, int height) {
  const rpd_stereo_rig r = rpd_rig_from_config(&c, width, height);
  return StereoRig{r.focal, r.baseline, r.cu, r.cv};
}
inline PointCloud reproject_masked_impl(const DisparityMap& d1, const LabelMap* labels, int label,
                                        const StereoRig& rig) {
  const rpd_stereo_rig r{rig.focal, rig.baseline, rig.cu, rig.cv};
  PointCloud cloud(size_t(std::max(1, d1.rows() * d1.cols())));
  int64_t n = 0;
  static_assert(sizeof(Point3) == sizeof(rpd_point3), "layout");
  auto* out = reinterpret_cast<rpd_point3*>(cloud.data());
  if (labels)
    detail::check(rpd_reproject_masked(detail::ctx(), d1.ptr(), labels->ptr(), d1.rows(),
                                       d1.cols(), label, &r, out, int64_t(cloud.size()), &n));
  else
    detail::check(rpd_reproject(detail::ctx(), d1.ptr(), d1.rows(), d1.cols(), &r, out,
                                int64_t(cloud.size()), &n));
  cloud.resize(size_t(n));
  return cloud;
}
inline PointCloud reproject(const DisparityMap& d1, const StereoRig& rig) {  // :65
  return reproject_masked_impl(d1, nullptr, 0, rig);
}
inline PointCloud reproject_masked(const DisparityMap& d1, const LabelMap& labels, int label,
                                   const StereoRig& rig) {  // :67
  check_same_shape(d1.rows(), d1.cols(), labels.rows(), labels.cols(), "reproject_masked");
  return reproject_masked_impl(d1, &labels, label, rig);
}
inline double closest_distance_error(const PointCloud& test, const PointCloud& truth) {  // :72
  double out = 0.0;
  detail::check(rpd_closest_distance_error(
      detail::ctx(), reinterpret_cast<const rpd_point3*>(test.data()), int64_t(test.size()),
      reinterpret_cast<const rpd_point3*>(truth.data()), int64_t(truth.size()), &out));
  return out;
}
inline void save_ply(const PointCloud& cloud, const std::string& path) {  // :190-197
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write: " + path);
  out << "ply\nformat ascii 1.0\nelement vertex " << cloud.size()
      << "\nproperty float x\nproperty float y\nproperty float z\nend_header\n";
  for (const auto& p : cloud) out << p.x << " " << p.y << " " << p.z << "\n";
  if (!out) throw std::runtime_error("write failed: " + path);
}
inline PointCloud load_ply(const std::string& path) {  // :199-225
  std::ifstream in(path);
  if (!in) throw std::runtime_error("not found: " + path);
  std::string line;
  std::size_t n = 0;
  bool header_done = false;
  while (std::getline(in, line)) {
    std::istringstream ss(line);
    std::string tok;
    ss >> tok;
    if (tok == "element") {
      std::string what;
      ss >> what >> n;
    } else if (tok == "end_header") {
      header_done = true;
      break;
    }
  }
  if (!header_done) throw std::runtime_error("bad PLY header: " + path);
  PointCloud cloud;
  cloud.reserve(n);
  for (std::size_t i = 0; i < n; ++i) {
    Point3 p;
    if (!(in >> p.x >> p.y >> p.z)) throw std::runtime_error("truncated PLY: " + path);
    cloud.push_back(p);
  }
  return cloud;
}

// -------------------------------------------------- synthetic scenes --
struct PotholeSpec {  // synth.hpp:12-18
  double cu = 0.0, cv = 0.0, ru = 10.0, rv = 10.0, depth = 2.0;
};
struct SceneSpec {  // synth.hpp:20-30
  int width = 640;
  int height = 480;
  StereoRig rig;
  double a0 = 5.0;
  double a1 = 0.08;
  double phi_true = 0.0;
  std::vector<PotholeSpec> potholes;
  std::uint32_t texture_seed = 1;
  double noise_sigma = 0.0;
};
struct SceneTruth {  // synth.hpp:32-38
  GrayImage left, right;
  DisparityMap gt_disparity;
  LabelMap gt_mask;
  SceneSpec spec;
};
struct BatchRanges {  // synth.hpp:45-53
  double depth_min = 1.5, depth_max = 4.0;
  double radius_min = 22.0, radius_max = 48.0;
  double a0_min = 4.0, a0_max = 7.0;
  double a1_min = 0.07, a1_max = 0.09;
  double phi_abs_max = 0.035;
  double noise_sigma = 0.0;
  int margin = 40;
};
inline SceneTruth generate_scene(const SceneSpec& spec) {  // synth.hpp:43
  std::vector<rpd_pothole_spec> pots;
  for (const auto& p : spec.potholes) pots.push_back({p.cu, p.cv, p.ru, p.rv, p.depth});
  rpd_scene_spec c{};
  c.width = spec.width;
  c.height = spec.height;
  c.rig = rpd_stereo_rig{spec.rig.focal, spec.rig.baseline, spec.rig.cu, spec.rig.cv};
  c.a0 = spec.a0;
  c.a1 = spec.a1;
  c.phi_true = spec.phi_true;
  c.texture_seed = spec.texture_seed;
  c.noise_sigma = spec.noise_sigma;
  c.n_potholes = int(pots.size());
  c.potholes = pots.data();
  SceneTruth t;
  const int h = std::max(spec.height, 0), w = std::max(spec.width, 0);
  t.left = GrayImage(h, w);
  t.right = GrayImage(h, w);
  t.gt_disparity = DisparityMap(h, w);
  t.gt_mask = LabelMap(h, w);
  detail::check(rpd_generate_scene(detail::ctx(), &c, t.left.ptr(), t.right.ptr(),
                                   t.gt_disparity.ptr(), t.gt_mask.ptr()));
  t.spec = spec;
  return t;
}
inline std::vector<SceneTruth> scene_batch(int count, std::uint32_t base_seed,
                                           const BatchRanges& r = {}) {  // synth.hpp:56-57
  if (count < 1) throw std::invalid_argument("scene_batch: count must be >= 1");
  const rpd_batch_ranges rc{r.depth_min, r.depth_max, r.radius_min, r.radius_max, r.a0_min,
                            r.a0_max,    r.a1_min,    r.a1_max,     r.phi_abs_max, r.noise_sigma,
                            r.margin};
  std::vector<SceneTruth> out;
  for (int i = 0; i < count; ++i) {
    rpd_scene_spec c{};
    rpd_pothole_spec pots[3];
    detail::check(rpd_scene_batch_spec(base_seed, i, &rc, &c, pots));
    SceneSpec s;
    s.width = c.width;
    s.height = c.height;
    s.rig = StereoRig{c.rig.focal, c.rig.baseline, c.rig.cu, c.rig.cv};
    s.a0 = c.a0;
    s.a1 = c.a1;
    s.phi_true = c.phi_true;
    s.texture_seed = c.texture_seed;
    s.noise_sigma = c.noise_sigma;
    for (int k = 0; k < c.n_potholes; ++k)
      s.potholes.push_back({pots[k].cu, pots[k].cv, pots[k].ru, pots[k].rv, pots[k].depth});
    out.push_back(generate_scene(s));
  }
  return out;
}

// --------------------------------------------------------------- pipeline --
struct StageTime {  // pipeline.hpp:21-24
  std::string name;
  double ms;
};
struct DetectResult {  // pipeline.hpp:26-38
  DisparityMap d0, d1, d2, d3;
  SuperpixelMap superpixels;
  LabelMap labels;
  RoadFit fit;
  ThresholdResult threshold;
  long clamped = 0;
  std::vector<StageTime> stage_times;  // device time per StageClock lap
  double total_ms = 0.0;
};
inline DetectResult detect_potholes_pipeline(const GrayImage& left, const GrayImage& right,
                                             const PipelineConfig& cfg) {
  if (left.rows() != right.rows() || left.cols() != right.cols())
    throw std::invalid_argument("match_pair: dimension mismatch");
  const int h = left.rows(), w = left.cols();
  DetectResult r;
  r.d0 = r.d1 = r.d2 = r.d3 = DisparityMap(h, w);
  r.labels = LabelMap(h, w);
  r.superpixels.labels = LabelMap(h, w);
  const int cap = slic_seed_count(h, w, cfg.superpixels);
  std::vector<rpd_center> centers(size_t(cap), rpd_center{});
  rpd_detect_out out{};
  out.d0 = r.d0.ptr();
  out.d1 = r.d1.ptr();
  out.d2 = r.d2.ptr();
  out.d3 = r.d3.ptr();
  out.labels = r.labels.ptr();
  out.sp_labels = r.superpixels.labels.ptr();
  out.centers = centers.data();
  out.centers_cap = int(centers.size());
  detail::check(rpd_detect(detail::ctx(), left.ptr(), right.ptr(), h, w, &cfg, &out));
  r.superpixels.count = out.sp_count;
  r.superpixels.spacing = out.sp_spacing;
  for (int k = 0; k < std::min(out.sp_count, cap); ++k)
    r.superpixels.centers.push_back({centers[size_t(k)].cu, centers[size_t(k)].cv,
                                     centers[size_t(k)].value});
  r.fit = RoadFit{{out.fit.model.a0, out.fit.model.a1, out.fit.model.phi}, out.fit.e0min,
                  long(out.fit.used)};
  r.threshold = ThresholdResult{out.threshold.t_r, out.threshold.t_s, out.threshold.mu1,
                                out.threshold.mu2, out.threshold.excluded_fraction,
                                out.threshold.degenerate != 0};
  r.clamped = long(out.clamped);
  static const char* names[RPD_NUM_STAGES] = {"sgm_bootstrap", "road_fit", "sgm_pt",
                                              "road_refit", "disparity_transform", "slic",
                                              "detect"};
  for (int i = 0; i < RPD_NUM_STAGES; ++i) r.stage_times.push_back({names[i], out.stage_ms[i]});
  r.total_ms = out.total_ms;
  return r;
}

}  // namespace rpd_b200
