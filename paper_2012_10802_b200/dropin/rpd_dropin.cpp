// rpd_dropin.cpp — the reference's C++ API (`namespace rpd`, declared by the
// reference's own include/rpd/*.hpp, compiled against them unchanged)
// implemented on the B200 library's C-ABI (include/rpd_b200.h ->
// paper_2012_10802_b200/_lib/librpd_b200.so).
//
// The drop-in for C++ callers of the reference: compile this file against the
// reference headers and Eigen, and link it with -lrpd_b200 INSTEAD OF the
// reference's src/{sgm,road_geometry,segmentation,pipeline,config,synth}.cpp
// (INTEGRATION.md §A).  The reference's own test files and acceptance gate,
// compiled unmodified, then run on the CUDA kernels (tests/cpp/refsuite,
// tests/test_reference_suite.py; there oracle/ref_shim stands in for Eigen).
// Every hot-path function below forwards to one C-ABI entry point; rasters
// are the reference's Eigen row-major arrays, whose data() is the C-ABI layout.
// Status codes map back onto the reference's exception types.  The header-
// only functions of perspective.hpp / evaluation.hpp stay the reference's.

#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "rpd/config.hpp"
#include "rpd/image_io.hpp"
#include "rpd/pipeline.hpp"
#include "rpd/road_geometry.hpp"
#include "rpd/segmentation.hpp"
#include "rpd/sgm.hpp"
#include "rpd/synth.hpp"
#include "rpd_b200.h"

namespace {

// One context per host thread on device 0 (the reference is reentrant).
rpd_ctx* ctx() {
  struct Holder {
    rpd_ctx* c = nullptr;
    ~Holder() {
      if (c) rpd_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c && rpd_ctx_create(0, 0, 0, 0, &h.c) != RPD_OK)
    throw std::runtime_error("rpd_b200: no CUDA device");
  return h.c;
}

void check(rpd_status st) {
  if (st == RPD_OK) return;
  const std::string msg = rpd_last_error(ctx());
  switch (st) {
    case RPD_EINVAL: throw std::invalid_argument(msg);
    case RPD_EDEGENERATE: throw std::runtime_error(msg);
    default: throw std::runtime_error("rpd_b200: " + msg);
  }
}

template <typename T>
T* ptr(rpd::Raster<T>& r) {
  return r.data();
}

rpd_config to_c(const rpd::PipelineConfig& p) {
  rpd_config c;
  rpd_config_default(&c);
  c.delta_pt = p.delta_pt;
  c.delta_dt = p.delta_dt;
  c.delta_pd = p.delta_pd;
  c.d_max = p.d_max;
  c.d_max_pt = p.d_max_pt;
  c.lambda1 = p.lambda1;
  c.lambda2 = p.lambda2;
  c.census_window = p.census_window;
  c.lr_threshold = p.lr_threshold;
  c.superpixels = p.superpixels;
  c.compactness = p.compactness;
  c.slic_iterations = p.slic_iterations;
  c.hist_bin_width = p.hist_bin_width;
  c.tau_diag = p.tau_diag;
  c.border_margin = p.border_margin;
  c.min_superpixels = p.min_superpixels;
  c.connectivity = p.connectivity;
  c.roll_bracket = p.roll_bracket;
  c.roll_tol = p.roll_tol;
  c.focal = p.focal;
  c.baseline = p.baseline;
  c.cu = p.cu;
  c.cv = p.cv;
  c.sgm_paths = 8;  // the reference always aggregates the eight directions
  return c;
}

rpd::CostVolume volume_like(int w, int h, int d_max) { return rpd::CostVolume(w, h, d_max); }

}  // namespace

namespace rpd {

// ---- config.hpp ------------------------------------------------------------
void PipelineConfig::validate() const {
  const rpd_config c = to_c(*this);
  check(rpd_config_validate(ctx(), &c));
}

void apply_key_value(PipelineConfig& p, const std::string& key, const std::string& value) {
  rpd_config c = to_c(p);
  check(rpd_config_set(ctx(), &c, key.c_str(), value.c_str()));
  p.delta_pt = c.delta_pt;
  p.delta_dt = c.delta_dt;
  p.delta_pd = c.delta_pd;
  p.d_max = c.d_max;
  p.d_max_pt = c.d_max_pt;
  p.lambda1 = c.lambda1;
  p.lambda2 = c.lambda2;
  p.census_window = c.census_window;
  p.lr_threshold = c.lr_threshold;
  p.superpixels = c.superpixels;
  p.compactness = c.compactness;
  p.slic_iterations = c.slic_iterations;
  p.hist_bin_width = c.hist_bin_width;
  p.tau_diag = c.tau_diag;
  p.border_margin = c.border_margin;
  p.min_superpixels = c.min_superpixels;
  p.connectivity = c.connectivity;
  p.roll_bracket = c.roll_bracket;
  p.roll_tol = c.roll_tol;
  p.focal = c.focal;
  p.baseline = c.baseline;
  p.cu = c.cu;
  p.cv = c.cv;
}

// ---- sgm.hpp -----------------------------------------------------------------
CostVolume census_cost_volume(const GrayImage& left, const GrayImage& right_warped, int d_max,
                              int window, const Raster<unsigned char>* right_in_view) {
  if (left.rows() != right_warped.rows() || left.cols() != right_warped.cols())
    throw std::invalid_argument("census_cost_volume: dimension mismatch");
  const int h = int(left.rows()), w = int(left.cols());
  CostVolume out = volume_like(w, h, d_max < 0 ? 0 : d_max);
  check(rpd_census_cost_volume(ctx(), left.data(), right_warped.data(), h, w, d_max, window,
                               right_in_view ? right_in_view->data() : nullptr,
                               out.costs.data()));
  return out;
}

CostVolume aggregate_costs(const CostVolume& v, const SgmParams& params) {
  std::vector<int32_t> dirs;
  for (const auto& d : params.directions) {
    dirs.push_back(d[0]);
    dirs.push_back(d[1]);
  }
  CostVolume out = volume_like(v.width, v.height, v.d_max);
  check(rpd_aggregate_costs(ctx(), v.costs.data(), v.height, v.width, v.d_max, dirs.data(),
                            int(params.directions.size()), params.lambda1, params.lambda2,
                            out.costs.data()));
  return out;
}

CostVolume swap_reference(const CostVolume& v) {
  CostVolume out = volume_like(v.width, v.height, v.d_max);
  check(rpd_swap_reference(ctx(), v.costs.data(), v.height, v.width, v.d_max, out.costs.data()));
  return out;
}

DisparityMap select_disparity(const CostVolume& v) {
  DisparityMap d(v.height, v.width);
  check(rpd_select_disparity(ctx(), v.costs.data(), v.height, v.width, v.d_max, ptr(d)));
  return d;
}

void consistency_filter(DisparityMap& left, const DisparityMap& right, double threshold) {
  if (left.rows() != right.rows() || left.cols() != right.cols())
    throw std::invalid_argument("consistency_filter: dimension mismatch");
  check(rpd_consistency_filter(ctx(), ptr(left), right.data(), int(left.rows()),
                               int(left.cols()), threshold));
}

MatchResult match_pair(const GrayImage& left, const GrayImage& right, const RoadModel& model,
                       const PipelineConfig& config, int d_max) {
  if (left.rows() != right.rows() || left.cols() != right.cols())
    throw std::invalid_argument("match_pair: dimension mismatch");
  const int h = int(left.rows()), w = int(left.cols());
  MatchResult r;
  r.d0 = DisparityMap(h, w);
  r.d1 = DisparityMap(h, w);
  r.shifts.shifts.resize(size_t(h));
  r.shifts.delta_pt = config.delta_pt;
  const rpd_config c = to_c(config);
  const rpd_road_model m{model.a0, model.a1, model.phi};
  check(rpd_match_pair(ctx(), left.data(), right.data(), h, w, &m, &c, d_max, ptr(r.d0),
                       ptr(r.d1), r.shifts.shifts.data()));
  return r;
}

// ---- road_geometry.hpp -------------------------------------------------------
LineFit fit_line(const RoadObservations& obs, double phi) {
  rpd_line_fit f;
  check(rpd_fit_line(ctx(), obs.d.data(), obs.u.data(), obs.v.data(), obs.count(), phi, &f));
  LineFit out;
  out.model = {f.model.a0, f.model.a1, f.model.phi};
  out.e0min = f.e0min;
  return out;
}

RoadModel estimate_roll(const RoadObservations& obs, double lo, double hi, double tol) {
  rpd_road_model m;
  check(rpd_estimate_roll(ctx(), obs.d.data(), obs.u.data(), obs.v.data(), obs.count(), lo, hi,
                          tol, &m));
  return {m.a0, m.a1, m.phi};
}

RoadFit fit_road(const RoadObservations& obs, double bracket, double tol) {
  rpd_road_fit f;
  check(rpd_fit_road(ctx(), obs.d.data(), obs.u.data(), obs.v.data(), obs.count(), bracket, tol,
                     &f));
  RoadFit out;
  out.model = {f.model.a0, f.model.a1, f.model.phi};
  out.e0min = f.e0min;
  out.used = f.used;
  return out;
}

RoadObservations sample_observations(const DisparityMap& d1, std::optional<RectRoi> roi,
                                     Eigen::Index cap) {
  const int h = int(d1.rows()), w = int(d1.cols());
  const Eigen::Index n = std::min<Eigen::Index>(Eigen::Index(h) * w, cap < 0 ? 0 : cap);
  std::vector<double> d(size_t(std::max<Eigen::Index>(n, 1))), u(d.size()), v(d.size());
  int64_t k = 0;
  rpd_rect_roi r{};
  if (roi) r = {roi->u0, roi->v0, roi->width, roi->height};
  check(rpd_sample_observations(ctx(), d1.data(), h, w, roi ? &r : nullptr, cap, d.data(),
                                u.data(), v.data(), &k));
  RoadObservations obs;
  obs.d.resize(k);
  obs.u.resize(k);
  obs.v.resize(k);
  for (int64_t i = 0; i < k; ++i) {
    obs.d[i] = d[size_t(i)];
    obs.u[i] = u[size_t(i)];
    obs.v[i] = v[size_t(i)];
  }
  return obs;
}

TransformResult transform_disparity(const DisparityMap& d1, const RoadModel& model,
                                    double delta_dt) {
  TransformResult out;
  out.d2 = DisparityMap(d1.rows(), d1.cols());
  const rpd_road_model m{model.a0, model.a1, model.phi};
  int64_t clamped = 0;
  check(rpd_transform_disparity(ctx(), d1.data(), int(d1.rows()), int(d1.cols()), &m, delta_dt,
                                ptr(out.d2), &clamped));
  out.clamped = long(clamped);
  return out;
}

namespace {
rpd_stereo_rig to_rig(const StereoRig& r) { return {r.focal, r.baseline, r.cu, r.cv}; }
PointCloud run_reproject(const DisparityMap& d1, const LabelMap* labels, int label,
                         const StereoRig& rig) {
  const rpd_stereo_rig c = to_rig(rig);
  const int h = int(d1.rows()), w = int(d1.cols());
  std::vector<rpd_point3> pts(size_t(std::max(1, h * w)));
  int64_t n = 0;
  if (labels)
    check(rpd_reproject_masked(ctx(), d1.data(), labels->data(), h, w, label, &c, pts.data(),
                               int64_t(pts.size()), &n));
  else
    check(rpd_reproject(ctx(), d1.data(), h, w, &c, pts.data(), int64_t(pts.size()), &n));
  PointCloud out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[size_t(i)] = {pts[size_t(i)].x, pts[size_t(i)].y,
                                                    pts[size_t(i)].z};
  return out;
}
}  // namespace

PointCloud reproject(const DisparityMap& d1, const StereoRig& rig) {
  return run_reproject(d1, nullptr, 0, rig);
}

PointCloud reproject_masked(const DisparityMap& d1, const LabelMap& labels, int label,
                            const StereoRig& rig) {
  return run_reproject(d1, &labels, label, rig);
}

double closest_distance_error(const PointCloud& test, const PointCloud& truth) {
  static_assert(sizeof(Point3) == sizeof(rpd_point3), "Point3 layout");
  double e = 0.0;
  check(rpd_closest_distance_error(ctx(), reinterpret_cast<const rpd_point3*>(test.data()),
                                   int64_t(test.size()),
                                   reinterpret_cast<const rpd_point3*>(truth.data()),
                                   int64_t(truth.size()), &e));
  return e;
}

// ASCII PLY (the file container is host I/O, as paper_2012_10802_b200/ply.py)
void save_ply(const PointCloud& cloud, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write: " + path);
  out << "ply\nformat ascii 1.0\nelement vertex " << cloud.size()
      << "\nproperty float x\nproperty float y\nproperty float z\nend_header\n";
  out.precision(std::numeric_limits<float>::max_digits10);
  for (const Point3& p : cloud) out << p.x << ' ' << p.y << ' ' << p.z << '\n';
}

PointCloud load_ply(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("not found: " + path);
  std::string line;
  size_t n = 0;
  bool header = false;
  while (std::getline(in, line)) {
    std::istringstream ss(line);
    std::string tok;
    ss >> tok;
    if (tok == "element") {
      std::string what;
      ss >> what >> n;
    } else if (tok == "end_header") {
      header = true;
      break;
    }
  }
  if (!header) throw std::runtime_error("bad PLY header: " + path);
  PointCloud cloud(n);
  for (Point3& p : cloud)
    if (!(in >> p.x >> p.y >> p.z)) throw std::runtime_error("truncated PLY: " + path);
  return cloud;
}

// SLIC keeps at most its nu * nv seeds (segmentation.cpp:181-184): the
// capacity of the centre records.
int slic_seed_count(int h, int w, int p) {
  if (h <= 0 || w <= 0 || p <= 0) return 1;
  const int nu = std::max(1, int(std::lround(std::sqrt(double(p) * w / h))));
  const int nv = std::max(1, int(std::lround(double(p) / nu)));
  return std::max(1, std::min(h * w, nu * nv));
}

// ---- segmentation.hpp --------------------------------------------------------
SuperpixelMap slic(const DisparityMap& d2, int p, double compactness, int iterations) {
  const int h = int(d2.rows()), w = int(d2.cols());
  SuperpixelMap sp;
  sp.labels = LabelMap(h, w);
  std::vector<rpd_center> cs(size_t(slic_seed_count(h, w, p)));
  int32_t count = 0;
  double spacing = 0.0;
  check(rpd_slic(ctx(), d2.data(), h, w, p, compactness, iterations, ptr(sp.labels), cs.data(),
                 int(cs.size()), &count, &spacing));
  sp.count = count;
  sp.spacing = spacing;
  const int nc = std::min(count, int(cs.size()));
  sp.centers.resize(size_t(nc));
  for (int k = 0; k < nc; ++k)
    sp.centers[size_t(k)] = {cs[size_t(k)].cu, cs[size_t(k)].cv, cs[size_t(k)].value};
  return sp;
}

DisparityMap pool_superpixels(const DisparityMap& d2, const SuperpixelMap& sp) {
  if (d2.rows() != sp.labels.rows() || d2.cols() != sp.labels.cols())
    throw std::invalid_argument("pool_superpixels: dimension mismatch");
  DisparityMap d3(d2.rows(), d2.cols());
  check(rpd_pool_superpixels(ctx(), d2.data(), sp.labels.data(), sp.count, int(d2.rows()),
                             int(d2.cols()), ptr(d3)));
  return d3;
}

Histogram2D build_histogram(const DisparityMap& d2, double bin_width) {
  Histogram2D hist;
  hist.bin_width = bin_width;
  int64_t n = 0, total = 0;
  double origin = 0.0;
  rpd_status st = rpd_build_histogram(ctx(), d2.data(), int(d2.rows()), int(d2.cols()),
                                      bin_width, nullptr, 0, &n, &origin, &total);
  if (st != RPD_ECAPACITY) check(st);
  std::vector<int64_t> counts(size_t(std::max<int64_t>(1, n * n)));
  check(rpd_build_histogram(ctx(), d2.data(), int(d2.rows()), int(d2.cols()), bin_width,
                            counts.data(), n, &n, &origin, &total));
  hist.origin = origin;
  hist.total = long(total);
  hist.counts = Raster<long>::Zero(n, n);
  for (int64_t i = 0; i < n * n; ++i) hist.counts.data()[i] = long(counts[size_t(i)]);
  return hist;
}

ThresholdResult find_road_threshold(const Histogram2D& hist, double delta_pd, double tau) {
  const int64_t n = hist.counts.rows();
  std::vector<int64_t> counts(size_t(std::max<int64_t>(1, n * n)));
  for (int64_t i = 0; i < n * n; ++i) counts[size_t(i)] = hist.counts.data()[i];
  rpd_threshold t;
  check(rpd_find_road_threshold(ctx(), counts.data(), n, hist.bin_width, hist.origin, hist.total,
                                delta_pd, tau, &t));
  ThresholdResult r;
  r.t_r = t.t_r;
  r.t_s = t.t_s;
  r.mu1 = t.mu1;
  r.mu2 = t.mu2;
  r.excluded_fraction = t.excluded_fraction;
  r.degenerate = t.degenerate != 0;
  return r;
}

LabelMap connected_components(const LabelMap& mask, int connectivity) {
  LabelMap out(mask.rows(), mask.cols());
  check(rpd_connected_components(ctx(), mask.data(), int(mask.rows()), int(mask.cols()),
                                 connectivity, ptr(out)));
  return out;
}

LabelMap detect_potholes(const DisparityMap& d3, const SuperpixelMap& sp,
                         const ThresholdResult& thr, int border_margin, int min_superpixels,
                         int connectivity) {
  if (d3.rows() != sp.labels.rows() || d3.cols() != sp.labels.cols())
    throw std::invalid_argument("detect_potholes: dimension mismatch");
  LabelMap out(d3.rows(), d3.cols());
  const rpd_threshold t{thr.t_r, thr.t_s, thr.mu1, thr.mu2, thr.excluded_fraction,
                        thr.degenerate ? 1 : 0};
  check(rpd_detect_potholes(ctx(), d3.data(), sp.labels.data(), sp.spacing, int(d3.rows()),
                            int(d3.cols()), &t, border_margin, min_superpixels, connectivity,
                            ptr(out)));
  return out;
}

// ---- pipeline.hpp ------------------------------------------------------------
DetectResult detect_potholes_pipeline(const GrayImage& left, const GrayImage& right,
                                      const PipelineConfig& config) {
  config.validate();
  if (left.rows() != right.rows() || left.cols() != right.cols())
    throw std::invalid_argument("match_pair: dimension mismatch");
  const int h = int(left.rows()), w = int(left.cols());
  DetectResult r;
  r.d0 = DisparityMap(h, w);
  r.d1 = DisparityMap(h, w);
  r.d2 = DisparityMap(h, w);
  r.d3 = DisparityMap(h, w);
  r.labels = LabelMap(h, w);
  r.superpixels.labels = LabelMap(h, w);
  std::vector<rpd_center> cs(size_t(slic_seed_count(h, w, config.superpixels)));
  rpd_detect_out o{};
  o.d0 = ptr(r.d0);
  o.d1 = ptr(r.d1);
  o.d2 = ptr(r.d2);
  o.d3 = ptr(r.d3);
  o.labels = ptr(r.labels);
  o.sp_labels = ptr(r.superpixels.labels);
  o.centers = cs.data();
  o.centers_cap = int(cs.size());
  const rpd_config c = to_c(config);
  const rpd_status st = rpd_detect(ctx(), left.data(), right.data(), h, w, &c, &o);
  if (st == RPD_EDEGENERATE) throw DegenerateFitError(rpd_last_error(ctx()));
  check(st);
  r.superpixels.count = o.sp_count;
  r.superpixels.spacing = o.sp_spacing;
  const int nc = std::min(o.sp_count, int(cs.size()));
  r.superpixels.centers.resize(size_t(nc));
  for (int k = 0; k < nc; ++k)
    r.superpixels.centers[size_t(k)] = {cs[size_t(k)].cu, cs[size_t(k)].cv, cs[size_t(k)].value};
  r.fit.model = {o.fit.model.a0, o.fit.model.a1, o.fit.model.phi};
  r.fit.e0min = o.fit.e0min;
  r.fit.used = o.fit.used;
  r.threshold = {o.threshold.t_r, o.threshold.t_s, o.threshold.mu1, o.threshold.mu2,
                 o.threshold.excluded_fraction, o.threshold.degenerate != 0};
  r.clamped = long(o.clamped);
  static const char* kNames[RPD_NUM_STAGES] = {"sgm_bootstrap", "road_fit", "sgm_pt",
                                               "road_refit", "disparity_transform", "slic",
                                               "detect"};
  for (int s = 0; s < RPD_NUM_STAGES; ++s) r.stage_times.push_back({kNames[s], o.stage_ms[s]});
  r.total_ms = o.total_ms;
  return r;
}

StereoRig rig_from_config(const PipelineConfig& config, int width, int height) {
  const rpd_config c = to_c(config);
  const rpd_stereo_rig g = rpd_rig_from_config(&c, width, height);
  StereoRig r;
  r.focal = g.focal;
  r.baseline = g.baseline;
  r.cu = g.cu;
  r.cv = g.cv;
  return r;
}

// ---- synth.hpp (the device scene generator) -------------
namespace {
rpd_scene_spec to_spec(const SceneSpec& s, std::vector<rpd_pothole_spec>& holes) {
  rpd_scene_spec c;
  rpd_scene_spec_default(&c);
  c.width = s.width;
  c.height = s.height;
  c.rig = to_rig(s.rig);
  c.a0 = s.a0;
  c.a1 = s.a1;
  c.phi_true = s.phi_true;
  c.texture_seed = s.texture_seed;
  c.noise_sigma = s.noise_sigma;
  holes.clear();
  for (const PotholeSpec& p : s.potholes) holes.push_back({p.cu, p.cv, p.ru, p.rv, p.depth});
  c.n_potholes = int(holes.size());
  c.potholes = holes.empty() ? nullptr : holes.data();
  return c;
}
}  // namespace

SceneTruth generate_scene(const SceneSpec& spec) {
  std::vector<rpd_pothole_spec> holes;
  const rpd_scene_spec c = to_spec(spec, holes);
  SceneTruth t;
  t.spec = spec;
  t.left = GrayImage(spec.height, spec.width);
  t.right = GrayImage(spec.height, spec.width);
  t.gt_disparity = DisparityMap(spec.height, spec.width);
  t.gt_mask = LabelMap(spec.height, spec.width);
  check(rpd_generate_scene(ctx(), &c, ptr(t.left), ptr(t.right), ptr(t.gt_disparity),
                           ptr(t.gt_mask)));
  return t;
}

std::vector<SceneTruth> scene_batch(int count, std::uint32_t base_seed,
                                    const BatchRanges& ranges) {
  rpd_batch_ranges r;
  r.depth_min = ranges.depth_min;
  r.depth_max = ranges.depth_max;
  r.radius_min = ranges.radius_min;
  r.radius_max = ranges.radius_max;
  r.a0_min = ranges.a0_min;
  r.a0_max = ranges.a0_max;
  r.a1_min = ranges.a1_min;
  r.a1_max = ranges.a1_max;
  r.phi_abs_max = ranges.phi_abs_max;
  r.noise_sigma = ranges.noise_sigma;
  r.margin = ranges.margin;
  std::vector<SceneTruth> out;
  for (int i = 0; i < count; ++i) {
    rpd_scene_spec s;
    rpd_pothole_spec holes[3];
    check(rpd_scene_batch_spec(base_seed, i, &r, &s, holes));
    SceneSpec spec;
    spec.width = s.width;
    spec.height = s.height;
    spec.rig = {s.rig.focal, s.rig.baseline, s.rig.cu, s.rig.cv};
    spec.a0 = s.a0;
    spec.a1 = s.a1;
    spec.phi_true = s.phi_true;
    spec.texture_seed = s.texture_seed;
    spec.noise_sigma = s.noise_sigma;
    for (int k = 0; k < s.n_potholes; ++k)
      spec.potholes.push_back({holes[k].cu, holes[k].cv, holes[k].ru, holes[k].rv,
                               holes[k].depth});
    out.push_back(generate_scene(spec));
  }
  return out;
}

// ---- image_io.hpp: file containers are out of the GPU library's scope here
// (libpng is absent); the acceptance gate only reaches them with a dataset.
GrayImage load_gray_image(const std::string& path) {
  throw std::runtime_error("image I/O not available in the drop-in test build: " + path);
}
LabelMap load_labels(const std::string& path) {
  throw std::runtime_error("image I/O not available in the drop-in test build: " + path);
}

}  // namespace rpd
