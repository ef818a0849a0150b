// abi_io.cu — per-pixel transforms of the reference's on-disk formats
// (image_io.cpp:171-339) on the device: the KITTI
// x256 disparity encoding, 16-bit labels, 8-bit gray, RGB luminance and the
// overlay tint.  Pipeline outputs are device-resident, so encoding before
// the copy back halves the bytes of a float raster; the file codecs (PNG /
// PGM containers) stay on the host (paper_2012_10802_b200/image_io.py).
// Each transform uses the reference's float / double expression order.
#include <cmath>

#include "abi_util.hpp"

using namespace rpdg;

namespace {

__constant__ unsigned char c_palette[12][3] = {
    {230, 25, 75},  {60, 180, 75},  {255, 225, 25}, {0, 130, 200},   {245, 130, 48},
    {145, 30, 180}, {70, 240, 240}, {240, 50, 230}, {210, 245, 60},  {250, 190, 190},
    {0, 128, 128},  {170, 110, 40}};  // image_io.cpp:262-267

template <typename F>
__global__ void k_map(long long n, F f) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    f(i);
}

template <typename F>
void launch_map(rpd_ctx* ctx, long long n, F f) {
  const int blocks = int(std::min<long long>((n + 255) / 256, ctx->sm_count * 16));
  k_map<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(n, f);
  RPD_LAUNCH_CHECK();
}

__device__ __forceinline__ unsigned char clamp_round_u8(float x) {
  const float r = roundf(x);  // std::round: half away from zero
  return static_cast<unsigned char>(fminf(fmaxf(r, 0.0f), 255.0f));
}

}  // namespace

extern "C" {

rpd_status rpd_encode_disparity_u16(rpd_ctx* ctx, const float* d, int h, int w, uint16_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const long long n = (long long)h * w;
    const float* dd = upload(ctx, "io_f32", d, size_t(n));
    uint16_t* dout = ctx->ws.get<uint16_t>("io_u16", size_t(n));
    int* bad = ctx->ws.get<int>("io_bad", 1);
    RPD_CK(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    launch_map(ctx, n, [=] __device__(long long i) {
      const float x = dd[i];
      uint16_t s = 0;
      if (x != kInvalid) {
        const double scaled = round(static_cast<double>(x) * 256.0);
        if (scaled < 0 || scaled > 65535)
          atomicOr(bad, 1);
        else
          s = static_cast<uint16_t>(scaled);
      }
      dout[i] = s;
    });
    int hb = 0;
    download(ctx, &hb, bad, sizeof(int));
    if (hb) throw Degenerate("disparity exceeds encoding range");
    download(ctx, out, dout, sizeof(uint16_t) * size_t(n));
  });
}

rpd_status rpd_decode_disparity_u16(rpd_ctx* ctx, const uint16_t* s, int h, int w, float* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const long long n = (long long)h * w;
    const uint16_t* ds = upload(ctx, "io_u16", s, size_t(n));
    float* dout = ctx->ws.get<float>("io_f32", size_t(n));
    launch_map(ctx, n, [=] __device__(long long i) {
      const uint16_t v = ds[i];
      dout[i] = v == 0 ? kInvalid : static_cast<float>(v) / 256.0f;
    });
    download(ctx, out, dout, sizeof(float) * size_t(n));
  });
}

rpd_status rpd_encode_labels_u16(rpd_ctx* ctx, const int32_t* labels, int h, int w,
                                 uint16_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const long long n = (long long)h * w;
    const int32_t* dl = upload(ctx, "io_i32", labels, size_t(n));
    uint16_t* dout = ctx->ws.get<uint16_t>("io_u16", size_t(n));
    int* bad = ctx->ws.get<int>("io_bad", 1);
    RPD_CK(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    launch_map(ctx, n, [=] __device__(long long i) {
      const int k = dl[i];
      if (k < 0 || k > 65535) atomicOr(bad, 1);
      dout[i] = static_cast<uint16_t>(k);
    });
    int hb = 0;
    download(ctx, &hb, bad, sizeof(int));
    if (hb) throw Degenerate("label exceeds encoding range");
    download(ctx, out, dout, sizeof(uint16_t) * size_t(n));
  });
}

rpd_status rpd_encode_gray_u8(rpd_ctx* ctx, const float* img, int h, int w, uint8_t* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const long long n = (long long)h * w;
    const float* di = upload(ctx, "io_f32", img, size_t(n));
    uint8_t* dout = ctx->ws.get<uint8_t>("io_u8", size_t(n));
    launch_map(ctx, n, [=] __device__(long long i) { dout[i] = clamp_round_u8(di[i]); });
    download(ctx, out, dout, size_t(n));
  });
}

rpd_status rpd_gray_from_rgb8(rpd_ctx* ctx, const uint8_t* rgb, int h, int w, float* out) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const long long n = (long long)h * w;
    const uint8_t* dr = upload(ctx, "io_rgb", rgb, size_t(n) * 3);
    float* dout = ctx->ws.get<float>("io_f32", size_t(n));
    launch_map(ctx, n, [=] __device__(long long i) {
      // 0.299f * R + 0.587f * G + 0.114f * B, float, left to right, no FMA
      const float r = __fmul_rn(0.299f, float(dr[3 * i]));
      const float g = __fmul_rn(0.587f, float(dr[3 * i + 1]));
      const float b = __fmul_rn(0.114f, float(dr[3 * i + 2]));
      dout[i] = __fadd_rn(__fadd_rn(r, g), b);
    });
    download(ctx, out, dout, sizeof(float) * size_t(n));
  });
}

rpd_status rpd_overlay_rgb8(rpd_ctx* ctx, const float* img, const int32_t* labels, int h, int w,
                            uint8_t* rgb) {
  return guard(ctx, [&] {
    check_dims(h, w);
    const long long n = (long long)h * w;
    const float* di = upload(ctx, "io_f32", img, size_t(n));
    const int32_t* dl = upload(ctx, "io_i32", labels, size_t(n));
    uint8_t* dout = ctx->ws.get<uint8_t>("io_rgb", size_t(n) * 3);
    launch_map(ctx, n, [=] __device__(long long i) {
      const float gray = di[i];
      const int k = dl[i];
      unsigned char c[3];
      if (k > 0) {  // overlay_tint: round((gray + p) * 0.5f), clamped
        const int q = (k - 1) % 12;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
          c[ch] = clamp_round_u8(__fmul_rn(__fadd_rn(gray, float(c_palette[q][ch])), 0.5f));
      } else {
        const unsigned char g = clamp_round_u8(gray);
        c[0] = c[1] = c[2] = g;
      }
      dout[3 * i] = c[0];
      dout[3 * i + 1] = c[1];
      dout[3 * i + 2] = c[2];
    });
    download(ctx, rgb, dout, size_t(n) * 3);
  });
}

}  // extern "C"
