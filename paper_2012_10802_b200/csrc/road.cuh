// road.cuh — road-model fit and disparity transformation on the device
// (road_geometry.cpp:12-151 of the reference).
#pragma once

#include "common.cuh"

namespace rpdg {

// Observations in the device's compact format: u | v<<16 and the float d1
// value (exact: the pipeline's observations are pixel coordinates and float
// disparities, road_geometry.cpp:103-134).
struct ObsBuffers {
  uint32_t* uv = nullptr;
  float* d = nullptr;
  int* count = nullptr;  // device int: k
};

struct FitOut {
  double a0, a1, phi, e0min;
  long long used;
  DevModel model;  // a0 (scaled), a1, phi and device cos/sin of phi
};

// sample_observations: valid pixels of d1 inside roi in scan order, strided
// down to min(n, cap).  n < 3 records `where` as a degenerate failure.
void sample_observations_dev(rpd_ctx* ctx, const float* d1, int h, int w, const rpd_rect_roi* roi,
                             long long cap, ObsBuffers obs, int where);

enum FitMode : int { kFitLine = 0, kEstimateRoll = 1, kFitRoad = 2 };

// Runs fit_line / estimate_roll / fit_road over device observations with one
// 8-CTA cluster.  compact obs: (uv, d) as produced by sample_observations_dev;
// otherwise dd/du/dv doubles with host count k.  The result (with a0 *=
// a0_scale applied, pipeline.cpp:73) lands in *out (device).
struct FitRequest {
  int mode = kFitRoad;
  bool compact = true;
  ObsBuffers obs;                // compact input
  const double* dd = nullptr;    // double input
  const double* du = nullptr;
  const double* dv = nullptr;
  long long k_host = 0;
  long long kmax = 0;            // compact input: capacity (observation cap); 0 = max
  double phi = 0.0;              // kFitLine
  double lo = 0.0, hi = 0.0;     // kEstimateRoll bracket, kFitRoad uses [-hi, hi]
  double tol = 1e-4;
  double a0_scale = 1.0;
  int where = kWhereFit;
  FitOut* out = nullptr;
};
void fit_dev(rpd_ctx* ctx, const FitRequest& req);

// transform_disparity (road_geometry.cpp:136-151).  *clamped (device int64)
// receives the clamp count (accumulated; zero it first).
void transform_disparity_dev(const float* d1, int h, int w, const DevModel* model, double delta_dt,
                             float* d2, unsigned long long* clamped, cudaStream_t st);

// Correctly rounded (double-double) sin/cos used for every device-side roll
// angle (the host path uses glibc).
__device__ void dd_sincos(double x, double* s, double* c);

}  // namespace rpdg
