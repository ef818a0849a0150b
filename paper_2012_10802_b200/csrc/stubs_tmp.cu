// TEMPORARY: entry points not yet ported to the device (removed when done).
#include "abi_util.hpp"
using namespace rpdg;
#define NYI(...) { if (ctx) ctx->err = "not implemented yet"; return RPD_EINVAL; }
extern "C" {
rpd_status rpd_detect(rpd_ctx* ctx, const float*, const float*, int, int, const rpd_config*, rpd_detect_out*) NYI()
rpd_status rpd_detect_u8(rpd_ctx* ctx, const uint8_t*, const uint8_t*, int, int, const rpd_config*, rpd_detect_out*) NYI()
rpd_status rpd_sample_observations(rpd_ctx* ctx, const float*, int, int, const rpd_rect_roi*, int64_t, double*, double*, double*, int64_t*) NYI()
rpd_status rpd_fit_line(rpd_ctx* ctx, const double*, const double*, const double*, int64_t, double, rpd_line_fit*) NYI()
rpd_status rpd_estimate_roll(rpd_ctx* ctx, const double*, const double*, const double*, int64_t, double, double, double, rpd_road_model*) NYI()
rpd_status rpd_fit_road(rpd_ctx* ctx, const double*, const double*, const double*, int64_t, double, double, rpd_road_fit*) NYI()
rpd_status rpd_transform_disparity(rpd_ctx* ctx, const float*, int, int, const rpd_road_model*, double, float*, int64_t*) NYI()
rpd_status rpd_slic(rpd_ctx* ctx, const float*, int, int, int, double, int, int32_t*, rpd_center*, int, int32_t*, double*) NYI()
rpd_status rpd_pool_superpixels(rpd_ctx* ctx, const float*, const int32_t*, int, int, int, float*) NYI()
rpd_status rpd_build_histogram(rpd_ctx* ctx, const float*, int, int, double, int64_t*, int64_t, int64_t*, double*, int64_t*) NYI()
rpd_status rpd_find_road_threshold(rpd_ctx* ctx, const int64_t*, int64_t, double, double, int64_t, double, double, rpd_threshold*) NYI()
rpd_status rpd_connected_components(rpd_ctx* ctx, const int32_t*, int, int, int, int32_t*) NYI()
rpd_status rpd_detect_potholes(rpd_ctx* ctx, const float*, const int32_t*, double, int, int, const rpd_threshold*, int, int, int, int32_t*) NYI()
}
