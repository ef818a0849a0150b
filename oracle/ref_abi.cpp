// ref_abi.cpp — C-ABI wrapper over the LITERAL reference library (TEST
// INFRASTRUCTURE ONLY; SURVEY.md §8(c) Route 2).
//
// oracle/Makefile compiles the untouched reference sources where they lie,
// /root/reference/proj/src/{config,sgm,road_geometry,segmentation,pipeline,
// synth}.cpp, against the from-scratch Eigen subset in oracle/ref_shim/ and
// links them with this file into oracle/_ref/librpd_ref.so (git-ignored).
// Nothing here restates an algorithm: every entry point converts the C-ABI
// buffers (include/rpd_b200.h) into the reference's types, calls the
// reference function named in the comment, and maps its exceptions onto the
// ABI status codes.  Two compositions exist because the reference has no
// path-count key (sgm.cpp:183-186 always uses kEightDirections):
//   * match_pair / detect with sgm_paths == 4 (BASELINE config 1) call the
//     reference's own stages in match_pair's order (sgm.cpp:172-226) and
//     pipeline order (pipeline.cpp:47-109) with the first four directions;
//     the two post-filter loops of match_pair (sgm.cpp:196-222) have no
//     function of their own and are repeated here verbatim in meaning.
//   * rpd_match_pair_dump exposes match_pair's intermediates (the same calls).
// sgm_paths == 8 runs detect_potholes_pipeline / match_pair themselves.
//
// image_io.cpp needs libpng (absent); its entry points are
// stubs that throw, so synth.cpp's write_scene/load_scene fail loudly.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "rpd/config.hpp"
#include "rpd/image_io.hpp"
#include "rpd/perspective.hpp"
#include "rpd/pipeline.hpp"
#include "rpd/road_geometry.hpp"
#include "rpd/segmentation.hpp"
#include "rpd/sgm.hpp"
#include "rpd/synth.hpp"
#include "rpd_b200.h"

// ---- image_io.hpp stubs (libpng absent) ------------------------------------
namespace rpd {
namespace {
[[noreturn]] void no_io() { throw std::runtime_error("image_io: not built (libpng absent)"); }
}  // namespace
GrayImage load_gray_image(const std::string&) { no_io(); }
void save_gray_image(const GrayImage&, const std::string&) { no_io(); }
DisparityMap load_disparity(const std::string&) { no_io(); }
void save_disparity(const DisparityMap&, const std::string&) { no_io(); }
LabelMap load_labels(const std::string&) { no_io(); }
void save_labels(const LabelMap&, const std::string&) { no_io(); }
void save_overlay(const GrayImage&, const LabelMap&, const std::string&) { no_io(); }
}  // namespace rpd

struct rpd_ctx {
  std::string err;
};

namespace {

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

template <typename T, typename S>
rpd::Raster<T> to_raster(const S* p, int h, int w) {
  rpd::Raster<T> r(h, w);
  for (long i = 0; i < long(h) * w; ++i) r.data()[i] = T(p[i]);
  return r;
}
template <typename T, typename D>
void put(D* dst, const rpd::Raster<T>& r) {
  if (!dst) return;
  for (long i = 0; i < long(r.size()); ++i) dst[i] = D(r.data()[i]);
}

rpd::PipelineConfig to_config(const rpd_config& c) {  // config.hpp:10-36, same names
  rpd::PipelineConfig p;
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
  return p;
}

void from_config(const rpd::PipelineConfig& p, int paths, rpd_config* c) {
  c->delta_pt = p.delta_pt;
  c->delta_dt = p.delta_dt;
  c->delta_pd = p.delta_pd;
  c->d_max = p.d_max;
  c->d_max_pt = p.d_max_pt;
  c->lambda1 = p.lambda1;
  c->lambda2 = p.lambda2;
  c->census_window = p.census_window;
  c->lr_threshold = p.lr_threshold;
  c->superpixels = p.superpixels;
  c->compactness = p.compactness;
  c->slic_iterations = p.slic_iterations;
  c->hist_bin_width = p.hist_bin_width;
  c->tau_diag = p.tau_diag;
  c->border_margin = p.border_margin;
  c->min_superpixels = p.min_superpixels;
  c->connectivity = p.connectivity;
  c->roll_bracket = p.roll_bracket;
  c->roll_tol = p.roll_tol;
  c->focal = p.focal;
  c->baseline = p.baseline;
  c->cu = p.cu;
  c->cv = p.cv;
  c->sgm_paths = paths;
}

int checked_paths(const rpd_config& c) {
  if (c.sgm_paths != 4 && c.sgm_paths != 8)
    throw std::invalid_argument("config: sgm_paths must be 4 or 8");
  return c.sgm_paths;
}

rpd::SgmParams params_of(const rpd::PipelineConfig& c, int paths) {  // sgm.cpp:183-186
  rpd::SgmParams p;
  p.lambda1 = static_cast<float>(c.lambda1);
  p.lambda2 = static_cast<float>(c.lambda2);
  p.census_window = c.census_window;
  p.directions.resize(size_t(paths));  // first `paths` of kEightDirections
  return p;
}

// match_pair (sgm.cpp:172-226) with a configurable path count: the same
// reference calls in the same order; only the post-filter loops (196-222)
// are repeated here.
rpd::MatchResult match_pair_paths(const rpd::GrayImage& left, const rpd::GrayImage& right,
                                  const rpd::RoadModel& model, const rpd::PipelineConfig& config,
                                  int d_max, int paths) {
  if (paths == 8) return rpd::match_pair(left, right, model, config, d_max);
  if (left.rows() != right.rows() || left.cols() != right.cols())
    throw std::invalid_argument("match_pair: dimension mismatch");
  rpd::MatchResult result;
  result.shifts = rpd::compute_row_shifts(model, int(left.cols()), int(left.rows()),
                                          config.delta_pt);
  rpd::WarpResult warped = rpd::warp_right_image(right, result.shifts);
  const rpd::SgmParams params = params_of(config, paths);
  rpd::CostVolume raw =
      rpd::census_cost_volume(left, warped.image, d_max, config.census_window, &warped.in_view);
  result.d0 = rpd::select_disparity(rpd::aggregate_costs(raw, params));
  rpd::DisparityMap right_disp =
      rpd::select_disparity(rpd::aggregate_costs(rpd::swap_reference(raw), params));
  rpd::consistency_filter(result.d0, right_disp, config.lr_threshold);
  for (int v = 0; v < left.rows(); ++v)
    for (int u = 0; u < left.cols(); ++u) {
      if (!rpd::is_valid(result.d0(v, u))) continue;
      float lo = std::numeric_limits<float>::max();
      float hi = std::numeric_limits<float>::lowest();
      for (int d = 0; d <= d_max; ++d) {
        const int ur = u - d;
        if (ur < 0 || !warped.in_view(v, ur)) continue;
        lo = std::min(lo, raw.at(v, u, d));
        hi = std::max(hi, raw.at(v, u, d));
      }
      if (hi <= lo) result.d0(v, u) = rpd::kInvalidDisparity;
    }
  for (int v = 0; v < left.rows(); ++v)
    for (int u = 0; u < left.cols(); ++u) {
      const float d = result.d0(v, u);
      if (!rpd::is_valid(d)) continue;
      const int ur = u - static_cast<int>(std::lround(d));
      if (ur < 0 || !warped.in_view(v, ur)) result.d0(v, u) = rpd::kInvalidDisparity;
    }
  result.d1 = rpd::restore_disparity(result.d0, result.shifts);
  return result;
}

rpd::GrayImage half_of(const rpd::GrayImage& img) {  // pipeline.cpp:25-34 (file-local there)
  const int h = int(img.rows()) / 2, w = int(img.cols()) / 2;
  rpd::GrayImage out(h, w);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u)
      out(v, u) = 0.25f * (img(2 * v, 2 * u) + img(2 * v, 2 * u + 1) + img(2 * v + 1, 2 * u) +
                           img(2 * v + 1, 2 * u + 1));
  return out;
}

void fill_out(const rpd::DetectResult& r, const rpd::RoadFit* coarse, rpd_detect_out* out) {
  put(out->d0, r.d0);
  put(out->d1, r.d1);
  put(out->d2, r.d2);
  put(out->d3, r.d3);
  put(out->labels, r.labels);
  put(out->sp_labels, r.superpixels.labels);
  if (out->centers)
    for (int k = 0; k < std::min(out->centers_cap, r.superpixels.count); ++k) {
      const auto& c = r.superpixels.centers[size_t(k)];
      out->centers[k] = {c.cu, c.cv, c.value};
    }
  out->sp_count = r.superpixels.count;
  out->sp_spacing = r.superpixels.spacing;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  out->coarse_fit = coarse ? rpd_road_fit{{coarse->model.a0, coarse->model.a1, coarse->model.phi},
                                          coarse->e0min, int64_t(coarse->used)}
                           : rpd_road_fit{{nan, nan, nan}, nan, -1};  // not in DetectResult
  out->fit = {{r.fit.model.a0, r.fit.model.a1, r.fit.model.phi}, r.fit.e0min,
              int64_t(r.fit.used)};
  out->threshold = {r.threshold.t_r, r.threshold.t_s, r.threshold.mu1, r.threshold.mu2,
                    r.threshold.excluded_fraction, r.threshold.degenerate ? 1 : 0};
  out->clamped = r.clamped;
  out->n_potholes = r.labels.size() ? r.labels.maxCoeff() : 0;
  static const char* kNames[RPD_NUM_STAGES] = {"sgm_bootstrap", "road_fit", "sgm_pt",
                                               "road_refit", "disparity_transform", "slic",
                                               "detect"};
  for (int s = 0; s < RPD_NUM_STAGES; ++s) {
    out->stage_ms[s] = 0.0;
    for (const auto& t : r.stage_times)
      if (t.name == kNames[s]) out->stage_ms[s] = t.ms;
  }
  out->total_ms = r.total_ms;
}

// detect_potholes_pipeline (pipeline.cpp:47-109).  sgm_paths == 8 is the
// reference function itself; 4 is the same sequence of reference calls with
// match_pair_paths (stage laps are not recorded there).
void detect_impl(const rpd::GrayImage& left, const rpd::GrayImage& right, const rpd_config& c,
                 rpd_detect_out* out) {
  const int paths = checked_paths(c);
  const rpd::PipelineConfig config = to_config(c);
  if (paths == 8) {
    fill_out(rpd::detect_potholes_pipeline(left, right, config), nullptr, out);
    return;
  }
  config.validate();
  if (left.rows() != right.rows() || left.cols() != right.cols())
    throw std::invalid_argument("match_pair: dimension mismatch");
  rpd::DetectResult result;
  const bool halve = left.rows() >= 64 && left.cols() >= 64;
  rpd::PipelineConfig boot = config;
  if (halve) boot.d_max = (config.d_max + 1) / 2;
  rpd::MatchResult bootstrap =
      halve ? match_pair_paths(half_of(left), half_of(right), rpd::RoadModel{}, boot, boot.d_max,
                               paths)
            : match_pair_paths(left, right, rpd::RoadModel{}, config, config.d_max, paths);
  rpd::RoadFit coarse;
  try {
    coarse = rpd::fit_road(rpd::sample_observations(bootstrap.d1), config.roll_bracket,
                           config.roll_tol);
  } catch (const std::runtime_error& e) {
    throw rpd::DegenerateFitError(std::string("road fit failed: ") + e.what());
  }
  if (halve) coarse.model.a0 *= 2.0;
  rpd::MatchResult refined =
      match_pair_paths(left, right, coarse.model, config, config.d_max_pt, paths);
  result.d0 = refined.d0;
  result.d1 = refined.d1;
  try {
    result.fit = rpd::fit_road(rpd::sample_observations(result.d1), config.roll_bracket,
                               config.roll_tol);
  } catch (const std::runtime_error& e) {
    throw rpd::DegenerateFitError(std::string("road refit failed: ") + e.what());
  }
  rpd::TransformResult dt = rpd::transform_disparity(result.d1, result.fit.model, config.delta_dt);
  result.d2 = std::move(dt.d2);
  result.clamped = dt.clamped;
  result.superpixels =
      rpd::slic(result.d2, config.superpixels, config.compactness, config.slic_iterations);
  result.d3 = rpd::pool_superpixels(result.d2, result.superpixels);
  rpd::Histogram2D hist = rpd::build_histogram(result.d2, config.hist_bin_width);
  result.threshold = rpd::find_road_threshold(hist, config.delta_pd, config.tau_diag);
  result.labels = rpd::detect_potholes(result.d3, result.superpixels, result.threshold,
                                       config.border_margin, config.min_superpixels,
                                       config.connectivity);
  fill_out(result, &coarse, out);
}

rpd::CostVolume to_volume(const float* costs, int h, int w, int d_max) {
  if (h <= 0 || w <= 0 || d_max < 0) throw std::invalid_argument("cost volume: bad dimensions");
  rpd::CostVolume v(w, h, d_max);
  std::memcpy(v.costs.data(), costs, sizeof(float) * v.costs.size());
  return v;
}
void put_volume(float* dst, const rpd::CostVolume& v) {
  if (dst) std::memcpy(dst, v.costs.data(), sizeof(float) * v.costs.size());
}

rpd::RoadObservations to_obs(const double* d, const double* u, const double* v, int64_t k) {
  rpd::RoadObservations o;
  o.d.resize(k);
  o.u.resize(k);
  o.v.resize(k);
  for (int64_t i = 0; i < k; ++i) {
    o.d[i] = d[i];
    o.u[i] = u[i];
    o.v[i] = v[i];
  }
  return o;
}

rpd::RowShiftTable to_table(const double* shifts, int h) {
  rpd::RowShiftTable t;
  t.shifts.assign(shifts, shifts + h);
  return t;
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

void rpd_config_default(rpd_config* cfg) { from_config(rpd::PipelineConfig{}, 8, cfg); }

rpd_status rpd_config_validate(rpd_ctx* ctx, const rpd_config* cfg) {
  return guard(ctx, [&] {
    checked_paths(*cfg);
    to_config(*cfg).validate();  // config.cpp:9-22
  });
}

rpd_status rpd_config_set(rpd_ctx* ctx, rpd_config* c, const char* key, const char* value) {
  return guard(ctx, [&] {
    const std::string k = key;
    if (k == "sgm_paths") {  // the one extension key (not in config.cpp)
      c->sgm_paths = std::stoi(value);
      return;
    }
    rpd::PipelineConfig p = to_config(*c);
    rpd::apply_key_value(p, k, value);  // config.cpp:24-51
    from_config(p, c->sgm_paths, c);
  });
}

rpd_status rpd_detect(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                      const rpd_config* cfg, rpd_detect_out* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    detect_impl(to_raster<float>(left, h, w), to_raster<float>(right, h, w), *cfg, out);
  });
}

rpd_status rpd_detect_u8(rpd_ctx* ctx, const uint8_t* left, const uint8_t* right, int h, int w,
                         const rpd_config* cfg, rpd_detect_out* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    detect_impl(to_raster<float>(left, h, w), to_raster<float>(right, h, w), *cfg, out);
  });
}

rpd_status rpd_compute_row_shifts(rpd_ctx* ctx, const rpd_road_model* m, int w, int h,
                                  double delta_pt, double* shifts) {
  return guard(ctx, [&] {
    const rpd::RowShiftTable t = rpd::compute_row_shifts({m->a0, m->a1, m->phi}, w, h, delta_pt);
    std::copy(t.shifts.begin(), t.shifts.end(), shifts);
  });
}

rpd_status rpd_warp_right_image(rpd_ctx* ctx, const float* right, int h, int w,
                                const double* shifts, float* image, uint8_t* in_view) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const rpd::WarpResult r = rpd::warp_right_image(to_raster<float>(right, h, w),
                                                    to_table(shifts, h));
    put(image, r.image);
    put(in_view, r.in_view);
  });
}

rpd_status rpd_restore_disparity(rpd_ctx* ctx, const float* d0, int h, int w,
                                 const double* shifts, float* d1) {
  return guard(ctx, [&] {
    check_dims(h, w);
    put(d1, rpd::restore_disparity(to_raster<float>(d0, h, w), to_table(shifts, h)));
  });
}

rpd_status rpd_census_cost_volume(rpd_ctx* ctx, const float* left, const float* right, int h,
                                  int w, int d_max, int window, const uint8_t* in_view,
                                  float* costs) {
  return guard(ctx, [&] {
    check_dims(h, w);
    rpd::Raster<unsigned char> iv;
    if (in_view) iv = to_raster<unsigned char>(in_view, h, w);
    put_volume(costs, rpd::census_cost_volume(to_raster<float>(left, h, w),
                                              to_raster<float>(right, h, w), d_max, window,
                                              in_view ? &iv : nullptr));
  });
}

rpd_status rpd_aggregate_costs(rpd_ctx* ctx, const float* costs, int h, int w, int d_max,
                               const int32_t* dirs, int ndirs, float l1, float l2, float* agg) {
  return guard(ctx, [&] {
    rpd::SgmParams p;
    p.lambda1 = l1;
    p.lambda2 = l2;
    p.directions.clear();
    for (int i = 0; i < ndirs; ++i) p.directions.push_back({dirs[2 * i], dirs[2 * i + 1]});
    put_volume(agg, rpd::aggregate_costs(to_volume(costs, h, w, d_max), p));
  });
}

rpd_status rpd_swap_reference(rpd_ctx* ctx, const float* costs, int h, int w, int d_max,
                              float* right_costs) {
  return guard(ctx, [&] {
    put_volume(right_costs, rpd::swap_reference(to_volume(costs, h, w, d_max)));
  });
}

rpd_status rpd_select_disparity(rpd_ctx* ctx, const float* agg, int h, int w, int d_max,
                                float* disp) {
  return guard(ctx, [&] { put(disp, rpd::select_disparity(to_volume(agg, h, w, d_max))); });
}

rpd_status rpd_consistency_filter(rpd_ctx* ctx, float* left, const float* right, int h, int w,
                                  double thr) {
  return guard(ctx, [&] {
    check_dims(h, w);
    rpd::DisparityMap l = to_raster<float>(left, h, w);
    rpd::consistency_filter(l, to_raster<float>(right, h, w), thr);
    put(left, l);
  });
}

rpd_status rpd_match_pair(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                          const rpd_road_model* m, const rpd_config* cfg, int d_max, float* d0,
                          float* d1, double* shifts) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const rpd::MatchResult r =
        match_pair_paths(to_raster<float>(left, h, w), to_raster<float>(right, h, w),
                         {m->a0, m->a1, m->phi}, to_config(*cfg), d_max, checked_paths(*cfg));
    put(d0, r.d0);
    put(d1, r.d1);
    if (shifts) std::copy(r.shifts.shifts.begin(), r.shifts.shifts.end(), shifts);
  });
}

rpd_status rpd_match_pair_dump(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                               const rpd_road_model* m, const rpd_config* cfg, int d_max,
                               float* cost, float* agg_left, float* agg_right, float* disp_left,
                               float* disp_right) {
  const rpd_sgm_dump d{cost, nullptr, agg_left, agg_right, disp_left, disp_right};
  return rpd_match_pair_dump_ex(ctx, left, right, h, w, m, cfg, d_max, &d);
}

rpd_status rpd_match_pair_dump_ex(rpd_ctx* ctx, const float* left, const float* right, int h,
                                  int w, const rpd_road_model* m, const rpd_config* cfg,
                                  int d_max, const rpd_sgm_dump* out) {
  float* cost = out->cost;
  float* agg_left = out->agg_left;
  float* agg_right = out->agg_right;
  float* disp_left = out->disp_left;
  float* disp_right = out->disp_right;
  return guard(ctx, [&] {  // the intermediates of sgm.cpp:179-194, same calls
    check_dims(h, w);
    const rpd::PipelineConfig c = to_config(*cfg);
    const rpd::RowShiftTable t = rpd::compute_row_shifts({m->a0, m->a1, m->phi}, w, h,
                                                         c.delta_pt);
    const rpd::WarpResult wr = rpd::warp_right_image(to_raster<float>(right, h, w), t);
    const rpd::SgmParams params = params_of(c, checked_paths(*cfg));
    const rpd::CostVolume raw = rpd::census_cost_volume(to_raster<float>(left, h, w), wr.image,
                                                        d_max, c.census_window, &wr.in_view);
    const rpd::CostVolume al = rpd::aggregate_costs(raw, params);
    const rpd::CostVolume cr = rpd::swap_reference(raw);
    const rpd::CostVolume ar = rpd::aggregate_costs(cr, params);
    put_volume(cost, raw);
    put_volume(out->cost_right, cr);
    put_volume(agg_left, al);
    put_volume(agg_right, ar);
    put(disp_left, rpd::select_disparity(al));
    put(disp_right, rpd::select_disparity(ar));
  });
}

rpd_status rpd_sample_observations(rpd_ctx* ctx, const float* d1, int h, int w,
                                   const rpd_rect_roi* roi, int64_t cap, double* d, double* u,
                                   double* v, int64_t* count) {
  return guard(ctx, [&] {
    check_dims(h, w);
    std::optional<rpd::RectRoi> r;
    if (roi) r = rpd::RectRoi{roi->u0, roi->v0, roi->width, roi->height};
    const rpd::RoadObservations o = rpd::sample_observations(to_raster<float>(d1, h, w), r, cap);
    for (long i = 0; i < long(o.count()); ++i) {
      d[i] = o.d[i];
      u[i] = o.u[i];
      v[i] = o.v[i];
    }
    *count = int64_t(o.count());
  });
}

rpd_status rpd_fit_line(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                        int64_t k, double phi, rpd_line_fit* out) {
  return guard(ctx, [&] {
    const rpd::LineFit f = rpd::fit_line(to_obs(d, u, v, k), phi);
    *out = {{f.model.a0, f.model.a1, f.model.phi}, f.e0min};
  });
}

rpd_status rpd_estimate_roll(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                             int64_t k, double lo, double hi, double tol, rpd_road_model* out) {
  return guard(ctx, [&] {
    const rpd::RoadModel m = rpd::estimate_roll(to_obs(d, u, v, k), lo, hi, tol);
    *out = {m.a0, m.a1, m.phi};
  });
}

rpd_status rpd_fit_road(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                        int64_t k, double bracket, double tol, rpd_road_fit* out) {
  return guard(ctx, [&] {
    const rpd::RoadFit f = rpd::fit_road(to_obs(d, u, v, k), bracket, tol);
    *out = {{f.model.a0, f.model.a1, f.model.phi}, f.e0min, int64_t(f.used)};
  });
}

rpd_status rpd_transform_disparity(rpd_ctx* ctx, const float* d1, int h, int w,
                                   const rpd_road_model* m, double delta_dt, float* d2,
                                   int64_t* clamped) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const rpd::TransformResult r =
        rpd::transform_disparity(to_raster<float>(d1, h, w), {m->a0, m->a1, m->phi}, delta_dt);
    put(d2, r.d2);
    if (clamped) *clamped = r.clamped;
  });
}

rpd_status rpd_slic(rpd_ctx* ctx, const float* d2, int h, int w, int p, double m, int iters,
                    int32_t* labels, rpd_center* centers, int cap, int32_t* count,
                    double* spacing) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const rpd::SuperpixelMap sp = rpd::slic(to_raster<float>(d2, h, w), p, m, iters);
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
    rpd::SuperpixelMap sp;
    sp.labels = to_raster<int>(lab, h, w);
    sp.count = count;
    for (long i = 0; i < long(sp.labels.size()); ++i)  // indexes sum[] unchecked (:239)
      if (sp.labels.data()[i] < 0 || sp.labels.data()[i] > count)
        throw std::invalid_argument("pool_superpixels: label out of range");
    sp.centers.resize(size_t(std::max(count, 0)));
    put(d3, rpd::pool_superpixels(to_raster<float>(d2, h, w), sp));
  });
}

rpd_status rpd_build_histogram(rpd_ctx* ctx, const float* d2, int h, int w, double bw,
                               int64_t* counts, int64_t cap_n, int64_t* n, double* origin,
                               int64_t* total) {
  rpd_status st = RPD_OK;
  const rpd_status g = guard(ctx, [&] {
    check_dims(h, w);
    const rpd::Histogram2D hist = rpd::build_histogram(to_raster<float>(d2, h, w), bw);
    *n = int64_t(hist.counts.rows());
    *origin = hist.origin;
    *total = hist.total;
    if (*n > cap_n) {
      st = RPD_ECAPACITY;
      if (ctx) ctx->err = "build_histogram: counts buffer too small";
      return;
    }
    if (counts) put(counts, hist.counts);
  });
  return g != RPD_OK ? g : st;
}

rpd_status rpd_find_road_threshold(rpd_ctx* ctx, const int64_t* counts, int64_t n, double bw,
                                   double origin, int64_t total, double delta_pd, double tau,
                                   rpd_threshold* out) {
  return guard(ctx, [&] {
    rpd::Histogram2D hist;
    hist.bin_width = bw;
    hist.origin = origin;
    hist.total = total;
    hist.counts = to_raster<long>(counts, int(n), int(n));
    const rpd::ThresholdResult t = rpd::find_road_threshold(hist, delta_pd, tau);
    *out = {t.t_r, t.t_s, t.mu1, t.mu2, t.excluded_fraction, t.degenerate ? 1 : 0};
  });
}

rpd_status rpd_connected_components(rpd_ctx* ctx, const int32_t* mask, int h, int w, int conn,
                                    int32_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    put(out, rpd::connected_components(to_raster<int>(mask, h, w), conn));
  });
}

rpd_status rpd_detect_potholes(rpd_ctx* ctx, const float* d3, const int32_t* sp_labels,
                               double spacing, int h, int w, const rpd_threshold* thr,
                               int margin, int min_sp, int conn, int32_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    rpd::SuperpixelMap sp;
    sp.labels = to_raster<int>(sp_labels, h, w);
    sp.spacing = spacing;
    sp.count = sp.labels.size() ? sp.labels.maxCoeff() : 0;
    sp.centers.resize(size_t(std::max(sp.count, 0)));
    rpd::ThresholdResult t;
    t.t_r = thr->t_r;
    t.t_s = thr->t_s;
    t.mu1 = thr->mu1;
    t.mu2 = thr->mu2;
    t.excluded_fraction = thr->excluded_fraction;
    t.degenerate = thr->degenerate != 0;
    put(out, rpd::detect_potholes(to_raster<float>(d3, h, w), sp, t, margin, min_sp, conn));
  });
}

}  // extern "C"
