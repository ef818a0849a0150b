// config.cpp — PipelineConfig defaults / validation / key=value parsing.
// Reference: include/rpd/config.hpp:10-36, src/config.cpp:9-77.
#include <cmath>
#include <string>

#include "host.hpp"

namespace rpdg {

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
  auto fail = [](const char* m) { throw InvalidArg(std::string("config: ") + m); };
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

void config_set(rpd_config* c, const std::string& key, const std::string& value) {
  // config.cpp:24-51 (std::stod / std::stoi semantics, unknown keys rejected)
  auto d = [&] {
    try {
      return std::stod(value);
    } catch (const std::exception&) {
      throw InvalidArg("config: bad value for '" + key + "'");
    }
  };
  auto i = [&] {
    try {
      return std::stoi(value);
    } catch (const std::exception&) {
      throw InvalidArg("config: bad value for '" + key + "'");
    }
  };
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
  else throw InvalidArg("config: unknown key '" + key + "'");
}

DevModel host_model(const rpd_road_model& m) {
  DevModel d;
  d.a0 = m.a0;
  d.a1 = m.a1;
  d.phi = m.phi;
  d.c = std::cos(m.phi);
  d.s = std::sin(m.phi);
  return d;
}

}  // namespace rpdg
