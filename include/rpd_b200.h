/*
 * rpd_b200.h — C-ABI of the B200-native road-pothole-detection hot path.
 *
 * This is the drop-in boundary.  Every entry point replaces one free function of
 * the reference C++ library `namespace rpd` (arxiv 2012.10802 re-implementation
 * under /root/reference/proj); the replaced declaration is cited as file:line
 * relative to /root/reference/proj.  Buffers are row-major rasters, index
 * v*W+u (types.hpp:9-10); disparities are float32 with invalid = -1.0f
 * (types.hpp:16,21); labels are int32 with 0 = background (types.hpp:19).
 * Cost volumes use the reference layout (v*W+u)*(d_max+1)+d (sgm.hpp:19).
 *
 * All host pointers are caller-owned.  The library owns only the device
 * workspaces inside an rpd_ctx.  Device-resident data: the raster arguments
 * and outputs of rpd_detect / rpd_detect_u8 / rpd_detect_fetch, the
 * evaluation metrics (rpd_pep, rpd_rmse, rpd_pixel_metrics,
 * rpd_instance_metrics), the reprojections and the image_io transforms may
 * also point to device memory of the context's GPU (unified addressing; the
 * staging copies become device-to-device), so a frame's outputs can be
 * evaluated or reprojected without a host round trip.  A context is single-threaded: one per
 * (host thread, device); concurrent contexts are fine (sgm/pipeline are
 * reentrant in the reference, rpd_cli.cpp:293-302).
 *
 * Errors: every call returns an rpd_status.  RPD_EINVAL mirrors
 * std::invalid_argument, RPD_EDEGENERATE mirrors std::runtime_error /
 * DegenerateFitError (pipeline.hpp:17-19).  rpd_last_error(ctx) holds the
 * reference-style message ("census_cost_volume: d_max >= width", ...).
 *
 * Two shared libraries export this exact symbol set:
 *   paper_2012_10802_b200/_lib/librpd_b200.so   — the product (sm_100a CUDA)
 *   oracle/_build/librpd_oracle.so               — CPU restatement, TEST ONLY
 * and oracle/_ref/librpd_ref.so (TEST ONLY) exports the hot-path subset over
 * the literal reference sources (oracle/ref_abi.cpp).
 */
#ifndef RPD_B200_H
#define RPD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RPD_ABI_VERSION 1

typedef enum rpd_status {
  RPD_OK = 0,
  RPD_EINVAL = 1,       /* std::invalid_argument */
  RPD_EDEGENERATE = 2,  /* std::runtime_error (degenerate data) / DegenerateFitError */
  RPD_ECUDA = 3,        /* CUDA runtime failure (product library only) */
  RPD_ENOMEM = 4,       /* device or host allocation failed */
  RPD_ECAPACITY = 5     /* a caller-provided output buffer is too small */
} rpd_status;

typedef struct rpd_ctx rpd_ctx;

/* RoadModel, types.hpp:33-37: d(u,v) = a0 + a1 (v cos(phi) - u sin(phi)). */
typedef struct rpd_road_model {
  double a0;
  double a1;
  double phi;
} rpd_road_model;

/* PipelineConfig, config.hpp:10-36 (same field names and defaults), plus
 * `sgm_paths` (4 or 8): the first `sgm_paths` entries of kEightDirections
 * (sgm.hpp:41-43).  The reference always uses 8 (sgm.cpp:183-186). */
typedef struct rpd_config {
  double delta_pt;
  double delta_dt;
  double delta_pd;
  int32_t d_max;
  int32_t d_max_pt;
  double lambda1;
  double lambda2;
  int32_t census_window;
  double lr_threshold;
  int32_t superpixels;
  double compactness;
  int32_t slic_iterations;
  double hist_bin_width;
  double tau_diag;
  int32_t border_margin;
  int32_t min_superpixels;
  int32_t connectivity;
  double roll_bracket;
  double roll_tol;
  double focal;
  double baseline;
  double cu;
  double cv;
  int32_t sgm_paths;
} rpd_config;

/* SuperpixelMap::Center, segmentation.hpp:11-15. */
typedef struct rpd_center {
  double cu;
  double cv;
  double value;
} rpd_center;

/* LineFit, road_geometry.hpp:20-23. */
typedef struct rpd_line_fit {
  rpd_road_model model;
  double e0min;
} rpd_line_fit;

/* RoadFit, road_geometry.hpp:34-38. */
typedef struct rpd_road_fit {
  rpd_road_model model;
  double e0min;
  int64_t used;
} rpd_road_fit;

/* RectRoi, road_geometry.hpp:45-47. */
typedef struct rpd_rect_roi {
  int32_t u0, v0, width, height;
} rpd_rect_roi;

/* ThresholdResult, segmentation.hpp:48-55. */
typedef struct rpd_threshold {
  double t_r;
  double t_s;
  double mu1;
  double mu2;
  double excluded_fraction;
  int32_t degenerate;
} rpd_threshold;

/* Stage names of StageClock laps (pipeline.cpp:64-104). */
#define RPD_NUM_STAGES 7
/* 0 sgm_bootstrap, 1 road_fit, 2 sgm_pt, 3 road_refit,
 * 4 disparity_transform, 5 slic, 6 detect */

/* DetectResult, pipeline.hpp:26-38.  Every pointer may be NULL (not copied
 * back).  Raster outputs are H*W. */
typedef struct rpd_detect_out {
  float* d0;
  float* d1;
  float* d2;
  float* d3;
  int32_t* labels;        /* final pothole labels */
  int32_t* sp_labels;     /* SuperpixelMap::labels */
  rpd_center* centers;    /* SuperpixelMap::centers, up to centers_cap */
  int32_t centers_cap;
  /* scalar results, always written */
  int32_t sp_count;
  double sp_spacing;
  rpd_road_fit coarse_fit; /* bootstrap fit after a0 *= 2 (pipeline.cpp:73) */
  rpd_road_fit fit;
  rpd_threshold threshold;
  int64_t clamped;
  int32_t n_potholes;
  double stage_ms[RPD_NUM_STAGES];
  double total_ms;
} rpd_detect_out;

/* ---- context / config ------------------------------------------------- */
int rpd_abi_version(void);
/* Creates a context on `device`.  max_h/max_w/max_levels are sizing hints
 * (workspaces grow on demand). */
rpd_status rpd_ctx_create(int device, int max_h, int max_w, int max_levels, rpd_ctx** out);
void rpd_ctx_destroy(rpd_ctx* ctx);
const char* rpd_last_error(const rpd_ctx* ctx);
/* The cudaStream_t all work of this context is ordered on (NULL for the oracle). */
void* rpd_ctx_stream(rpd_ctx* ctx);

void rpd_config_default(rpd_config* cfg);                               /* config.hpp:11-33 */
rpd_status rpd_config_validate(rpd_ctx* ctx, const rpd_config* cfg);     /* config.cpp:9-22 */
rpd_status rpd_config_set(rpd_ctx* ctx, rpd_config* cfg, const char* key,
                          const char* value);                            /* config.cpp:24-51 */

/* ---- pipeline ----------------------------------------------------------- */
/* detect_potholes_pipeline, pipeline.hpp:43-44 / pipeline.cpp:47-109.
 * left/right: H*W float32 gray images in [0,255]. */
rpd_status rpd_detect(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                      const rpd_config* cfg, rpd_detect_out* out);
/* Same, uint8 images (exact: intensities are only compared / averaged). */
rpd_status rpd_detect_u8(rpd_ctx* ctx, const uint8_t* left, const uint8_t* right, int h,
                         int w, const rpd_config* cfg, rpd_detect_out* out);

/* Streaming extension (no reference counterpart): device-resident uint8
 * inputs.  rpd_input_buffers_u8 returns the context's device input buffers
 * (fill them with cudaMemcpyAsync on rpd_ctx_stream(ctx)); rpd_detect_async_u8
 * enqueues one frame on the context stream and returns without waiting;
 * rpd_detect_fetch waits, checks the device status and copies the requested
 * outputs (same fields as rpd_detect). */
rpd_status rpd_input_buffers_u8(rpd_ctx* ctx, int h, int w, uint8_t** d_left, uint8_t** d_right);
rpd_status rpd_detect_async_u8(rpd_ctx* ctx, const uint8_t* d_left, const uint8_t* d_right,
                               int h, int w, const rpd_config* cfg);
rpd_status rpd_detect_fetch(rpd_ctx* ctx, rpd_detect_out* out);
/* Streaming from host memory (BASELINE config 5's pinned double-buffered
 * upload): enqueues the H2D copy of the pair and the frame on the context
 * stream and returns.  The copy is asynchronous when left/right are pinned
 * (rpd_host_alloc); they must stay unchanged until rpd_detect_fetch returns,
 * so a caller alternates two slots and fills the next while a frame runs. */
rpd_status rpd_detect_async_host_u8(rpd_ctx* ctx, const uint8_t* left, const uint8_t* right,
                                    int h, int w, const rpd_config* cfg);
/* Page-locked host memory for the streaming buffers (cudaHostAlloc). */
rpd_status rpd_host_alloc(size_t bytes, void** out);
void rpd_host_free(void* p);
/* Same as rpd_detect_async_u8 for device-resident float32 images (e.g. the
 * output of rpd_generate_scenes_device). */
rpd_status rpd_detect_async(rpd_ctx* ctx, const float* d_left, const float* d_right, int h, int w,
                            const rpd_config* cfg);

/* Measurement extension.  With profiling enabled, CUDA events are recorded on
 * the context stream around every SGM path-aggregation launch (the dominant
 * kernel); rpd_ctx_stats reports them for the last frame together with the
 * SURVEY §8(d) algorithmic bytes of each launch and the kernel count of the
 * last frame's captured graph. */
typedef struct rpd_stats {
  int32_t kernels_last_frame;   /* kernel launches of one rpd_detect* frame */
  int32_t graph_replayed;       /* 1 if the last frame replayed a captured graph */
  int32_t sgm_passes;           /* aggregation launches recorded (<= 2) */
  double sgm_agg_ms[2];         /* device duration of each aggregation launch */
  double sgm_agg_alg_bytes[2];  /* 2*(5P-2)*cells: u8 cost read + u16 sum read/write */
  double sgm_cells[2];          /* H*W*L of the pass */
  int32_t last_agg_kernel;      /* aggregation implementation of the context's last
                                   match_pair / aggregate_costs: RPD_AGG_* */
  int32_t agg_segmented_ctas;   /* last aggregation launch: CTAs that run a chain segment
                                   after the first (long H / V chains are cut) */
  int64_t agg_segment_reruns;   /* cumulative: segments whose warm-up state differed from
                                   the predecessor's and that were recomputed */
  int64_t slic_tiles_assigned;  /* cumulative: assignment tiles evaluated by the SLIC rounds
                                   after the first (incremental rounds) */
  int64_t slic_tiles_skipped;   /* cumulative: tiles of those rounds that no moved centre
                                   reached and that kept their labels */
  int64_t slic_centres_moved;   /* checked build only (0 otherwise): cumulative count of
                                   centres that moved in those rounds */
  int64_t slic_pixels_changed;  /* checked build only (0 otherwise): cumulative count of
                                   pixels whose label changed in those rounds */
} rpd_stats;
#define RPD_AGG_NONE 0
#define RPD_AGG_F32 1    /* generic float kernels (non-integral penalties, other directions) */
#define RPD_AGG_U8_TMA 2 /* production k_aggregate_tma (u8 paths, u16x2 DPX recurrence) */
#define RPD_AGG_U8 3     /* production u8 kernel without TMA staging (layouts TMA cannot map) */
rpd_status rpd_ctx_set_profiling(rpd_ctx* ctx, int enable);
rpd_status rpd_ctx_stats(rpd_ctx* ctx, rpd_stats* out);

/* Checked-build hook (make DEBUG_KNOBS=1 -> _lib_dbg/): every workspace
 * buffer is allocated at its exact size followed by a 4 KiB guard zone of
 * 0xA5 bytes; this reports how many guard bytes were overwritten (and the
 * first buffer's name).  The product build returns *corrupted = -1.
 * (compute-sanitizer is closed on the GPU pool; this is the out-of-bounds
 * write check that replaces memcheck.) */
rpd_status rpd_debug_guard_check(rpd_ctx* ctx, long long* corrupted, char* first, int cap);
/* Checked build: writes one byte just past a fresh `bytes`-sized workspace
 * buffer (proves the guard check fires).  RPD_EINVAL in the product. */
rpd_status rpd_debug_guard_selftest(rpd_ctx* ctx, size_t bytes);

/* Test hook: the device's roll-angle sin/cos (double-double, correctly
 * rounded with overwhelming probability) for n angles. */
rpd_status rpd_debug_sincos(rpd_ctx* ctx, const double* x, int n, double* s, double* c);

/* Test hook: the device's single-pass exclusive prefix sum (scan.cuh, the
 * ordered-compaction primitive of sample_observations, the SLIC and CCL
 * numbering): out[i] = in[0] + ... + in[i-1], *total = sum of all n. */
rpd_status rpd_debug_scan(rpd_ctx* ctx, const int32_t* in, int64_t n, int32_t* out, int32_t* total);

/* Parity extension: runs the production match_pair SGM path and materialises
 * its intermediates in the reference float layout (v*W+u)*(d_max+1)+d:
 * census_cost_volume, aggregate_costs of it and of swap_reference(it), and the
 * two select_disparity maps before the consistency filter.  NULL skips. */
rpd_status rpd_match_pair_dump(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                               const rpd_road_model* model, const rpd_config* cfg, int d_max,
                               float* cost, float* agg_left, float* agg_right, float* disp_left,
                               float* disp_right);

/* Same, with the right-reference cost volume swap_reference(cost)
 * (sgm.cpp:112-121, sgm.cpp:193) as well: the product generates it directly
 * from the census words inside the cost kernel, so this is the production
 * volume the right-reference aggregation consumed.  NULL members skip. */
typedef struct rpd_sgm_dump {
  float* cost;        /* census_cost_volume, H*W*(d_max+1) */
  float* cost_right;  /* swap_reference(cost) */
  float* agg_left;    /* aggregate_costs(cost) */
  float* agg_right;   /* aggregate_costs(swap_reference(cost)) */
  float* disp_left;   /* select_disparity(agg_left), H*W */
  float* disp_right;  /* select_disparity(agg_right) */
} rpd_sgm_dump;
rpd_status rpd_match_pair_dump_ex(rpd_ctx* ctx, const float* left, const float* right, int h,
                                  int w, const rpd_road_model* model, const rpd_config* cfg,
                                  int d_max, const rpd_sgm_dump* out);

/* ---- perspective transformation (perspective.hpp) ----------------------- */
/* compute_row_shifts, perspective.hpp:23-35; shifts: H doubles. */
rpd_status rpd_compute_row_shifts(rpd_ctx* ctx, const rpd_road_model* model, int w, int h,
                                  double delta_pt, double* shifts);
/* warp_right_image, perspective.hpp:45-66; image H*W float, in_view H*W u8. */
rpd_status rpd_warp_right_image(rpd_ctx* ctx, const float* right, int h, int w,
                                const double* shifts, float* image, uint8_t* in_view);
/* restore_disparity, perspective.hpp:69-80. */
rpd_status rpd_restore_disparity(rpd_ctx* ctx, const float* d0, int h, int w,
                                 const double* shifts, float* d1);

/* ---- SGM (sgm.hpp) ------------------------------------------------------ */
/* census_cost_volume, sgm.hpp:49-51; costs: H*W*(d_max+1) floats.
 * right_in_view may be NULL. */
rpd_status rpd_census_cost_volume(rpd_ctx* ctx, const float* left, const float* right_warped,
                                  int h, int w, int d_max, int window,
                                  const uint8_t* right_in_view, float* costs);
/* aggregate_costs, sgm.hpp:56; dirs: ndirs (du,dv) pairs.  The product runs
 * the production u8 aggregation kernels (RPD_AGG_U8_TMA) whenever their
 * result is provably the reference's: integral costs and penalties,
 * 1 <= lambda1 <= lambda2, max(cost) + lambda2 <= 255, and the direction set
 * equal to the first 4 or all 8 of kEightDirections; otherwise the generic
 * float kernels (RPD_AGG_F32). */
rpd_status rpd_aggregate_costs(rpd_ctx* ctx, const float* costs, int h, int w, int d_max,
                               const int32_t* dirs, int ndirs, float lambda1, float lambda2,
                               float* aggregated);
/* swap_reference, sgm.hpp:59. */
rpd_status rpd_swap_reference(rpd_ctx* ctx, const float* costs, int h, int w, int d_max,
                              float* right_costs);
/* select_disparity, sgm.hpp:63. */
rpd_status rpd_select_disparity(rpd_ctx* ctx, const float* aggregated, int h, int w,
                                int d_max, float* disparity);
/* consistency_filter, sgm.hpp:66-67 (in place on left_disp). */
rpd_status rpd_consistency_filter(rpd_ctx* ctx, float* left_disp, const float* right_disp,
                                  int h, int w, double threshold);
/* match_pair, sgm.hpp:77-79.  shifts (H doubles) may be NULL. */
rpd_status rpd_match_pair(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                          const rpd_road_model* model, const rpd_config* cfg, int d_max,
                          float* d0, float* d1, double* shifts);

/* ---- road geometry (road_geometry.hpp) ---------------------------------- */
/* sample_observations, road_geometry.hpp:51-53.  roi may be NULL (whole map).
 * d/u/v must hold min(#valid, cap) doubles; *count receives that number. */
rpd_status rpd_sample_observations(rpd_ctx* ctx, const float* d1, int h, int w,
                                   const rpd_rect_roi* roi, int64_t cap, double* d, double* u,
                                   double* v, int64_t* count);
/* fit_line, road_geometry.hpp:28. */
rpd_status rpd_fit_line(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                        int64_t k, double phi, rpd_line_fit* out);
/* estimate_roll, road_geometry.hpp:31-32. */
rpd_status rpd_estimate_roll(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                             int64_t k, double bracket_lo, double bracket_hi, double tol,
                             rpd_road_model* out);
/* fit_road, road_geometry.hpp:43. */
rpd_status rpd_fit_road(rpd_ctx* ctx, const double* d, const double* u, const double* v,
                        int64_t k, double bracket, double tol, rpd_road_fit* out);
/* transform_disparity, road_geometry.hpp:61-62. */
rpd_status rpd_transform_disparity(rpd_ctx* ctx, const float* d1, int h, int w,
                                   const rpd_road_model* model, double delta_dt, float* d2,
                                   int64_t* clamped);

/* ---- segmentation (segmentation.hpp) ------------------------------------ */
/* slic, segmentation.hpp:28.  labels H*W; centers up to centers_cap. */
rpd_status rpd_slic(rpd_ctx* ctx, const float* d2, int h, int w, int p, double compactness,
                    int iterations, int32_t* labels, rpd_center* centers, int centers_cap,
                    int32_t* count, double* spacing);
/* pool_superpixels, segmentation.hpp:32. */
rpd_status rpd_pool_superpixels(rpd_ctx* ctx, const float* d2, const int32_t* sp_labels,
                                int sp_count, int h, int w, float* d3);
/* build_histogram, segmentation.hpp:46.  counts: n*n int64 row-major, n <= cap_n.
 * When cap_n is too small, *n is still written and RPD_ECAPACITY returned. */
rpd_status rpd_build_histogram(rpd_ctx* ctx, const float* d2, int h, int w, double bin_width,
                               int64_t* counts, int64_t cap_n, int64_t* n, double* origin,
                               int64_t* total);
/* find_road_threshold, segmentation.hpp:60-61. */
rpd_status rpd_find_road_threshold(rpd_ctx* ctx, const int64_t* counts, int64_t n,
                                   double bin_width, double origin, int64_t total,
                                   double delta_pd, double tau, rpd_threshold* out);
/* connected_components, segmentation.hpp:65. */
rpd_status rpd_connected_components(rpd_ctx* ctx, const int32_t* mask, int h, int w,
                                    int connectivity, int32_t* out);
/* detect_potholes, segmentation.hpp:69-71. */
rpd_status rpd_detect_potholes(rpd_ctx* ctx, const float* d3, const int32_t* sp_labels,
                               double sp_spacing, int h, int w, const rpd_threshold* thr,
                               int border_margin, int min_superpixels, int connectivity,
                               int32_t* out);

/* ---- evaluation (evaluation.hpp) — SURVEY.md §8(f) row 1 ----------------- */
typedef struct rpd_confusion {
  int64_t n_tp, n_fp, n_fn, n_tn;
} rpd_confusion;

typedef struct rpd_pixel_report {
  rpd_confusion counts;
  double precision, recall, accuracy, fscore;
  int32_t degenerate_precision; /* 0/0, reported as 0 */
  int32_t degenerate_recall;
} rpd_pixel_report;

typedef struct rpd_instance_report {
  int32_t correct, incorrect, misdetection;
} rpd_instance_report;

/* pep, evaluation.hpp:14-27: percentage of pixels valid in both maps with
 * |est - gt| > eps.  RPD_EDEGENERATE when no pixel is valid in both. */
rpd_status rpd_pep(rpd_ctx* ctx, const float* est, const float* gt, int h, int w, double eps,
                   double* out);
/* rmse, evaluation.hpp:29-42 (same validity rule and failure). */
rpd_status rpd_rmse(rpd_ctx* ctx, const float* est, const float* gt, int h, int w, double* out);
/* fscore, evaluation.hpp:63-66 (host arithmetic, no context). */
double rpd_fscore(double precision, double recall);
/* pixel_metrics, evaluation.hpp:69-89: nonzero = pothole in both maps. */
rpd_status rpd_pixel_metrics(rpd_ctx* ctx, const int32_t* pred, const int32_t* gt_mask, int h,
                             int w, rpd_pixel_report* out);
/* instance_metrics, evaluation.hpp:97-149: greedy one-to-one matching by
 * descending IoU (ties: lower prediction, then lower truth id). */
rpd_status rpd_instance_metrics(rpd_ctx* ctx, const int32_t* pred, const int32_t* gt_instances,
                                int h, int w, double iou_min, rpd_instance_report* out);

/* ---- 3-D reprojection (road_geometry.hpp:64-73) — SURVEY.md §8(f) row 2 --- */
typedef struct rpd_stereo_rig {
  double focal, baseline, cu, cv; /* types.hpp:25-30 */
} rpd_stereo_rig;

typedef struct rpd_point3 {
  float x, y, z;
} rpd_point3;

/* rig_from_config, pipeline.hpp:46 (cu / cv < 0: image centre).  Host only. */
rpd_stereo_rig rpd_rig_from_config(const rpd_config* cfg, int width, int height);
/* reproject, road_geometry.hpp:65: Z = f b / d, X = (u - cu) Z / f,
 * Y = (v - cv) Z / f over valid pixels with d > 0, in scan order.  *n receives
 * the point count; RPD_ECAPACITY (and the first cap points) when n > cap. */
rpd_status rpd_reproject(rpd_ctx* ctx, const float* d1, int h, int w, const rpd_stereo_rig* rig,
                         rpd_point3* out, int64_t cap, int64_t* n);
/* reproject_masked, road_geometry.hpp:67-68: only pixels with labels == label. */
rpd_status rpd_reproject_masked(rpd_ctx* ctx, const float* d1, const int32_t* labels, int h,
                                int w, int label, const rpd_stereo_rig* rig, rpd_point3* out,
                                int64_t cap, int64_t* n);
/* Every instance cloud at once (the CLI's loop over potholes 1..max_label,
 * rpd_cli.cpp:99-104): instance k's points, in scan order, are
 * out[offsets[k-1] .. offsets[k]); offsets has max_label + 1 entries. */
rpd_status rpd_reproject_instances(rpd_ctx* ctx, const float* d1, const int32_t* labels, int h,
                                   int w, int max_label, const rpd_stereo_rig* rig,
                                   rpd_point3* out, int64_t cap, int64_t* offsets);
/* closest_distance_error, road_geometry.hpp:72: RMS distance from each test
 * point to its nearest truth point (exact brute force).  RPD_EINVAL when a
 * cloud is empty. */
rpd_status rpd_closest_distance_error(rpd_ctx* ctx, const rpd_point3* test, int64_t n_test,
                                      const rpd_point3* truth, int64_t n_truth, double* out);

/* ---- raster encodings of the on-disk formats (image_io.cpp:190-339) —
 * SURVEY.md §8(f) row 3.  The file codecs (PNG / PGM) are host-side
 * (paper_2012_10802_b200/image_io.py); these are their per-pixel transforms. */
/* save_disparity's KITTI encoding (:215-235): round(d * 256), 0 = invalid;
 * RPD_EDEGENERATE ("disparity exceeds encoding range") outside [0, 65535]. */
rpd_status rpd_encode_disparity_u16(rpd_ctx* ctx, const float* d, int h, int w, uint16_t* out);
/* load_disparity (:202-213): s / 256.0f, 0 -> invalid. */
rpd_status rpd_decode_disparity_u16(rpd_ctx* ctx, const uint16_t* s, int h, int w, float* out);
/* save_labels (:245-259): RPD_EDEGENERATE outside [0, 65535]. */
rpd_status rpd_encode_labels_u16(rpd_ctx* ctx, const int32_t* labels, int h, int w,
                                 uint16_t* out);
/* save_gray_image (:187-199): clamp(round(x), 0, 255). */
rpd_status rpd_encode_gray_u8(rpd_ctx* ctx, const float* img, int h, int w, uint8_t* out);
/* load_gray_image of an RGB raster (:176-181): 0.299 R + 0.587 G + 0.114 B (float). */
rpd_status rpd_gray_from_rgb8(rpd_ctx* ctx, const uint8_t* rgb, int h, int w, float* out);
/* save_overlay (:291-312): gray background, label k tinted with palette (k-1) mod 12. */
rpd_status rpd_overlay_rgb8(rpd_ctx* ctx, const float* img, const int32_t* labels, int h, int w,
                            uint8_t* rgb);


/* ---- synthetic scenes (synth.hpp:12-60, synth.cpp:94-196) — SURVEY.md
 * §8(f) row 4.  The generator draws from the reference's random streams
 * (std::mt19937 + libstdc++ distributions), so a scene equals the
 * reference's for the same spec. */
typedef struct rpd_pothole_spec {
  double cu, cv; /* centre, px */
  double ru, rv; /* radii, px */
  double depth;  /* disparity deficit at the centre, px */
} rpd_pothole_spec;

typedef struct rpd_scene_spec {
  int32_t width, height;
  rpd_stereo_rig rig;
  double a0, a1, phi_true;           /* true road line */
  uint32_t texture_seed;
  double noise_sigma;                /* additive intensity noise */
  int32_t n_potholes;
  const rpd_pothole_spec* potholes;  /* host array of n_potholes */
} rpd_scene_spec;

typedef struct rpd_batch_ranges {
  double depth_min, depth_max;
  double radius_min, radius_max;
  double a0_min, a0_max;
  double a1_min, a1_max;
  double phi_abs_max;
  double noise_sigma;
  int32_t margin;
} rpd_batch_ranges;

/* SceneSpec / BatchRanges defaults (synth.hpp:20-30, 45-53).  Host only. */
void rpd_scene_spec_default(rpd_scene_spec* spec);
void rpd_batch_ranges_default(rpd_batch_ranges* ranges);
/* The spec of scene `index` of scene_batch(count, base_seed, ranges)
 * (synth.cpp:151-192): seed base_seed + index, 1-3 non-overlapping potholes
 * written to potholes[0..2] and linked from spec->potholes.  Host only. */
rpd_status rpd_scene_batch_spec(uint32_t base_seed, int32_t index, const rpd_batch_ranges* ranges,
                                rpd_scene_spec* spec, rpd_pothole_spec potholes[3]);
/* generate_scene, synth.hpp:43 / synth.cpp:94-149: H*W left, right, truth
 * disparity and pothole mask (index + 1); NULL outputs are skipped.
 * RPD_EINVAL on a bad pothole (depth <= 0, radius < 4), RPD_EDEGENERATE when
 * the truth disparity goes negative. */
rpd_status rpd_generate_scene(rpd_ctx* ctx, const rpd_scene_spec* spec, float* left,
                              float* right, float* gt_disparity, int32_t* gt_mask);
/* Streaming extension (product library only): `count` scenes of one size
 * generated straight into device buffers of count*H*W elements each (scene b
 * at offset b*H*W), in one batch of launches on the context stream; returns
 * after the batch completes (errors as rpd_generate_scene). */
rpd_status rpd_generate_scenes_device(rpd_ctx* ctx, int count, const rpd_scene_spec* specs,
                                      float* d_left, float* d_right, float* d_gt,
                                      int32_t* d_mask);

#ifdef __cplusplus
}
#endif

#endif /* RPD_B200_H */
