// int_peak.cu — measured integer-pipe peaks of this B200 for the SGM
// aggregation's instruction mix (the denominator of bench.py's
// roofline.int_ops).  Each op runs as 16 independent dependency chains per
// thread on 148 x 16 CTAs of 256 threads (every SM sub-partition saturated);
// one source op = one SASS instruction (checked with cuobjdump -sass, see
// profiles/int_peak.json "sass").  Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/int_peak tools/int_peak.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kChains = 16;

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b, uint32_t c) {
  if constexpr (OP == 0) return a + b + c;                      // IADD3
  if constexpr (OP == 1) return min(a, b);                      // IMNMX.U32
  if constexpr (OP == 2) return __viaddmin_u16x2(a, b, c);      // VIADDMNMX.U16x2 (fused add+min)
  if constexpr (OP == 3) return __vminu2(a, b);                 // VIMNMX.U16x2
  if constexpr (OP == 4) return __vimin3_u16x2(a, b, c);        // VIMNMX3.U16x2
  if constexpr (OP == 5) return __byte_perm(a, b, 0x5410);      // PRMT
  return a;
}

template <int OP>
__global__ void __launch_bounds__(256) k_peak(uint32_t* out, int iters, uint32_t p,
                                              long long* cycles) {
  uint32_t x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 7u + c * 0x00010001u;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = op<OP>(x[c], x[(c + 1) % kChains], p);
  }
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int OP>
void run(const char* name, const char* sass, double cell_ops_per_lane_op, bool last) {
  const int blocks = 148 * 16, threads = 256, iters = 8192;
  uint32_t* d;
  long long* cyc;
  cudaMalloc(&d, sizeof(uint32_t) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long));
  k_peak<OP><<<blocks, threads>>>(d, iters, 0x00050005u, cyc);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_peak<OP><<<blocks, threads>>>(d, iters, 0x00050005u, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long c0 = 0;
  cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  const double lane_ops = double(blocks) * threads * iters * kChains;
  const double s = ms * 1e-3;
  (void)c0;
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);  // max SM clock
  const double clk_hz = double(khz) * 1e3;
  printf("  \"%s\": {\"sass\": \"%s\", \"lane_ops_per_s\": %.4e, \"warp_inst_per_clk_per_sm\": %.3f, "
         "\"cell_ops_per_lane_op\": %.0f, \"cell_ops_per_s\": %.4e, \"sm_clock_mhz\": %.0f}%s\n",
         name, sass, lane_ops / s, lane_ops / 32.0 / s / clk_hz / 148.0, cell_ops_per_lane_op,
         lane_ops * cell_ops_per_lane_op / s, clk_hz / 1e6, last ? "" : ",");
  cudaFree(d);
  cudaFree(cyc);
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  printf("{\n  \"device\": \"%s\", \"sms\": %d,\n", prop.name, prop.multiProcessorCount);
  run<0>("iadd3", "IADD3", 2, false);           // two adds per instruction
  run<1>("imnmx_u32", "IMNMX.U32", 1, false);
  run<2>("viaddmnmx_u16x2", "VIADDMNMX.U16x2", 4, false);  // 2 halves x (add + min)
  run<3>("vimnmx_u16x2", "VIMNMX.U16x2", 2, false);
  run<4>("vimnmx3_u16x2", "VIMNMX3.U16x2", 4, false);      // 2 halves x 2 mins
  run<5>("prmt", "PRMT", 1, true);
  printf("}\n");
  return 0;
}
