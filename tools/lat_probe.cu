// lat_probe.cu — single-warp issue rate of the aggregation's integer ops:
// one warp (one CTA of 32 threads), K independent dependency chains per
// thread, cycles per warp instruction.  Shows how many warps an SM
// sub-partition needs before the ALU pipe saturates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b, uint32_t c) {
  if constexpr (OP == 0) return a + b + c;
  if constexpr (OP == 1) return __viaddmin_u16x2(a, b, c);
  if constexpr (OP == 2) return __vimin3_u16x2(a, b, c);
  if constexpr (OP == 3) return __byte_perm(a, b, 0x5432);
  if constexpr (OP == 4) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(c), "r"(b));
    return r;
  }
  return a;
}

template <int OP, int K>
__global__ void k_lat(uint32_t* out, int iters, uint32_t p, long long* cyc) {
  uint32_t x[K];
#pragma unroll
  for (int c = 0; c < K; ++c) x[c] = threadIdx.x * 7u + c * 0x00010001u;
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < K; ++c) x[c] = op<OP>(x[c], x[(c + 1) % K] | 1u, p);
  }
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < K; ++c) s ^= x[c];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int OP, int K>
void run(const char* name, int warps_per_smsp) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  // one CTA of 32*4*wps threads per SM -> wps warps per sub-partition
  const int threads = 32 * 4 * warps_per_smsp;
  k_lat<OP, K><<<1, threads>>>(out, iters, 1u, cyc);
  k_lat<OP, K><<<1, threads>>>(out, iters, 1u, cyc);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_inst = double(c) / (double(iters) * K);
  std::printf("%-10s K=%2d warps/smsp=%d: %.2f cycles per warp-instruction per warp\n", name, K,
              warps_per_smsp, per_inst);
  cudaFree(out);
  cudaFree(cyc);
}

template <int OP>
void sweep(const char* name) {
  run<OP, 1>(name, 1);
  run<OP, 4>(name, 1);
  run<OP, 8>(name, 1);
  run<OP, 16>(name, 1);
  run<OP, 16>(name, 2);
  run<OP, 16>(name, 4);
}

int main() {
  sweep<0>("IADD3");
  sweep<1>("VIADDMNMX");
  sweep<2>("VIMNMX3");
  sweep<3>("PRMT");
  sweep<4>("IMAD");
  return 0;
}
