// sgm.cuh — semi-global matching on the device (sgm.cpp:13-226 of the reference).
#pragma once

#include "common.cuh"

namespace rpdg {

// Geometry of the fast integer path for one pass.
struct SgmLayout {
  int h = 0, w = 0;
  int levels = 0;   // L = d_max + 1
  int G = 1;        // lanes per scan chain
  int wpl = 1;      // u8 cost words per lane (4 levels per word)
  int lw = 4;       // bytes per pixel in the u8 volumes = 4*wpl*G >= L
  int paths = 8;    // P
  size_t pitch = 0; // bytes per image row in the u8 volumes (16-byte multiple)
  size_t vol_bytes() const { return pitch * size_t(h); }
};
SgmLayout sgm_layout(int h, int w, int levels, int paths);
constexpr int kWplG1Max = 17;  // widest one-lane-per-chain layout (68 levels)

// TMA-staged aggregation of all 2P (volume, direction) chains of one pass
// (sgm_tma.cu).  vol_lr: left- then right-reference u8 cost volumes;
// paths: 2P per-path u8 output volumes, each vol_bytes() apart.
bool sgm_tma_supported(const SgmLayout& L);
// nvols = 1 aggregates only the first (left-reference) volume.
void launch_aggregate_tma(rpd_ctx* ctx, const SgmLayout& L, uint8_t* vol_lr, uint8_t* paths,
                          const int32_t* dirs, int paths_n, uint32_t p1, uint32_t p2,
                          int nvols = 2);

// Which aggregation implementation the last match_pair / aggregate_costs of
// a context ran (rpd_stats.last_agg_kernel).
enum AggImpl { kAggNone = 0, kAggF32 = 1, kAggU8Tma = 2, kAggU8 = 3 };

// aggregate_costs (sgm.cpp:70-110) through the production u8 kernels
// (k_aggregate_tma + the WTA's exact u16 sums) — the ABI entry takes this
// route whenever the result is provably identical to the float recursion:
// integral costs and penalties with max(cost) + lambda2 <= 255, and the
// direction set equal to the first 4 or all 8 of kEightDirections.  Returns
// false (nothing launched) when the volume does not qualify.
bool aggregate_u8_eligible(const float* costs_host, size_t cells, int levels,
                           const int32_t* dirs, int ndirs, float l1, float l2, int* paths);
void aggregate_u8_dev(rpd_ctx* ctx, const float* costs, int h, int w, int levels, int paths,
                      float l1, float l2, float* out);

// Whether the integer u8/u16x2 path reproduces the reference's float
// arithmetic bit-exactly for these penalties (integral lambdas and
// (window^2-1) + lambda2 <= 255); otherwise the generic float path runs.
bool sgm_fast_path_ok(float lambda1, float lambda2, int window);

// Optional materialisation of the fast path's intermediate volumes in the
// reference float layout (v*W+u)*L+d, for parity dumps.
struct MatchDump {
  float* cost = nullptr;       // census_cost_volume
  float* agg_left = nullptr;   // aggregate_costs(cost)
  float* agg_right = nullptr;  // aggregate_costs(swap_reference(cost))
  float* disp_left = nullptr;  // select_disparity(agg_left)
  float* disp_right = nullptr; // select_disparity(agg_right)
  float* cost_right = nullptr; // swap_reference(cost)
};

// ---------------------------------------------------------------- kernels --
void launch_u8_to_f32(const uint8_t* in, float* out, long long n, cudaStream_t st,
                      const uint8_t* in1 = nullptr, float* out1 = nullptr);
void launch_half_image(const float* in, int h, int w, float* out, cudaStream_t st,
                       const float* in1 = nullptr, float* out1 = nullptr);
void launch_row_shifts(const DevModel* model, int h, int w, double delta_pt, double* shifts,
                       cudaStream_t st);
void launch_warp_right(const float* right, const double* shifts, int h, int w, float* out,
                       uint8_t* in_view, cudaStream_t st);
void launch_restore(const float* d0, const double* shifts, int h, int w, float* d1,
                    cudaStream_t st);
void launch_census(const float* img, int h, int w, int window, uint64_t* out, cudaStream_t st);
void launch_census2(const float* img0, const float* img1, int h, int w, int window,
                    uint64_t* out0, uint64_t* out1, cudaStream_t st);
// Float cost volume in the reference layout (census_cost_volume ABI).
void launch_cost_f32(const uint64_t* cl, const uint64_t* cr, const uint8_t* in_view, int h, int w,
                     int levels, int window, float* costs, cudaStream_t st);

// Generic float path (any direction list, any penalties), used by the
// aggregate_costs / select_disparity / swap_reference ABI and as the
// match_pair path for non-integral penalties.
void aggregate_f32(rpd_ctx* ctx, const float* costs, int h, int w, int levels,
                   const int32_t* dirs_host, int ndirs, float l1, float l2, float* out);
void swap_reference_f32(rpd_ctx* ctx, const float* costs, int h, int w, int levels, float* out);
void select_disparity_f32(const float* agg, int h, int w, int levels, float* disp,
                          cudaStream_t st);
void consistency_filter_dev(float* left, const float* right, int h, int w, double thr,
                            cudaStream_t st);

// Full matching pass on device buffers (match_pair, sgm.cpp:172-226).
// model: device pointer.  left/right: float images.  Outputs d0, d1 (H*W)
// and shifts (H doubles) are device pointers.
void match_pair_dev(rpd_ctx* ctx, const float* left, const float* right, int h, int w,
                    const DevModel* model, const rpd_config& cfg, int d_max, float* d0,
                    float* d1, double* shifts, const MatchDump* dump = nullptr);

}  // namespace rpdg
