// seg.cuh — SLIC superpixels, pooling, 2-D histogram / threshold, CCL and
// pothole labelling on the device (segmentation.cpp of the reference).
#pragma once

#include "common.cuh"

namespace rpdg {

// Exact signed 128-bit fixed-point accumulator (value * 2^100) so per-label
// double sums are independent of atomic order (segmentation.cpp:74-93,
// 231-249 accumulate in scan order).
struct Acc128 {
  unsigned long long lo;
  long long hi;
};

struct SlicOut {
  int32_t* labels;      // device H*W
  double* centers;      // device, 3 doubles per centre (cu, cv, value), capacity K
  int* count;           // device int
  double spacing;       // host
  int k_seeds;          // host: nu*nv
};

// slic, segmentation.cpp:170-229.  d2 device float H*W.
// d3 != nullptr: pool_superpixels (segmentation.cpp:231-249) of d2 over the
// result as well, fused into slic's final update_centers pass.
SlicOut slic_dev(rpd_ctx* ctx, const float* d2, int h, int w, int p, double compactness,
                 int iterations, float* d3 = nullptr);

// pool_superpixels, segmentation.cpp:231-249.  count_dev or count_host gives
// the label range [0, count].
void pool_superpixels_dev(rpd_ctx* ctx, const float* d2, const int32_t* labels, int h, int w,
                          int max_count, float* d3);

// Band histogram of build_histogram (segmentation.cpp:251-296) consumed by
// find_road_threshold (298-359).  Only |i-j| <= band is stored; everything
// else is provably excluded by the |g1-g2| > tau test and is counted.
struct HistDev {
  long long* bins;   // rows x (2*half+1), row = g1 bin, column = g2 bin - g1 bin + half
  int half;
  long long cap_rows;
  long long* meta;   // [n, total, excluded outside the band, lo key, hi key]
  double* origin;    // device double
};
HistDev build_histogram_dev(rpd_ctx* ctx, const float* d2, int h, int w, double bin_width,
                            double tau);
// Full n*n histogram for the build_histogram ABI.
void build_histogram_full_dev(rpd_ctx* ctx, const float* d2, int h, int w, double bin_width,
                              long long* n_out, double* origin_out, long long* total_out,
                              long long* counts_host, long long cap_n);
// find_road_threshold on a band histogram (or on a full histogram uploaded as
// band == n-1).  Result written to *out (device rpd_threshold).
void find_threshold_dev(rpd_ctx* ctx, const HistDev& hd, double bin_width, double delta_pd,
                        double tau, rpd_threshold* out, int where);

// find_road_threshold on a caller-provided dense n x n histogram (device).
void threshold_from_full_dev(rpd_ctx* ctx, const long long* counts_dev, long long n, double bw,
                             double origin, long long total, double delta_pd, double tau,
                             rpd_threshold* out);

// connected_components, segmentation.cpp:361-390 (mask: nonzero = foreground).
void connected_components_dev(rpd_ctx* ctx, const int32_t* mask, int h, int w, int connectivity,
                              int32_t* out);
// detect_potholes, segmentation.cpp:392-434.
void detect_potholes_dev(rpd_ctx* ctx, const float* d3, const int32_t* sp_labels, double spacing,
                         int h, int w, const rpd_threshold* thr_dev, int border_margin,
                         int min_superpixels, int connectivity, int32_t* out, int* n_out);

}  // namespace rpdg
