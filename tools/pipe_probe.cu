// pipe_probe.cu — which sm_100a pipes the SGM / SLIC instruction mixes use:
// per-op throughput (lanes/clk/SM) and whether two ops of different pipes
// co-issue (the mixed kernels interleave two independent op streams).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe tools/pipe_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kChains = 16;

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b, uint32_t c) {
  if constexpr (OP == 0) return a + b + c;                                   // IADD3
  if constexpr (OP == 1) {                                                   // IMAD
    uint32_t r;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(c | 1u), "r"(b));
    return r;
  }
  if constexpr (OP == 2) return __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(b)));  // FADD
  if constexpr (OP == 3) return __float_as_uint(fminf(__uint_as_float(a), __uint_as_float(b)));      // FMNMX
  if constexpr (OP == 4) return h2u(__hadd2(u2h(a), u2h(b)));                                        // HADD2
  if constexpr (OP == 5) return h2u(__hmin2(u2h(a), u2h(b)));                                        // HMNMX2
  if constexpr (OP == 6) return h2u(__hfma2(u2h(a), u2h(c), u2h(b)));                                // HFMA2
  if constexpr (OP == 7) return __vimin3_u16x2(a, b, c);                                             // VIMNMX3
  if constexpr (OP == 8) return a ^ b ^ c;                                                           // LOP3
  if constexpr (OP == 9) return __float_as_uint(fminf(fminf(__uint_as_float(a), __uint_as_float(b)), __uint_as_float(c)));  // FMNMX3?
  return a;
}

// MIX: chains alternate between op A and op B (independent streams)
template <int A, int B>
__global__ void __launch_bounds__(256) k_probe(uint32_t* out, int iters, uint32_t p) {
  uint32_t x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 7u + c * 0x00010001u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (c % 2 == 0)
        x[c] = op<A>(x[c], x[(c + 2) % kChains], p);
      else
        x[c] = op<B>(x[c], x[(c + 2) % kChains], p);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int A, int B>
void run(const char* name) {
  const int blocks = 148 * 16, threads = 256, iters = 4096;
  uint32_t* d;
  cudaMalloc(&d, sizeof(uint32_t) * blocks * threads);
  k_probe<A, B><<<blocks, threads>>>(d, iters, 0x3C003C00u);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_probe<A, B><<<blocks, threads>>>(d, iters, 0x3C003C00u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double lane_ops = double(blocks) * threads * iters * kChains;
  printf("%-16s %7.1f lanes/clk/SM (all ops)\n", name,
         lane_ops / (ms * 1e-3) / (khz * 1e3) / 148.0);
  cudaFree(d);
}

int main() {
  run<0, 0>("iadd3");
  run<1, 1>("imad");
  run<2, 2>("fadd");
  run<3, 3>("fmnmx");
  run<4, 4>("hadd2");
  run<5, 5>("hmnmx2");
  run<6, 6>("hfma2");
  run<7, 7>("vimnmx3");
  run<8, 8>("lop3");
  run<9, 9>("fmnmx3");
  run<0, 1>("iadd3+imad");
  run<7, 1>("vimnmx3+imad");
  run<7, 2>("vimnmx3+fadd");
  run<7, 4>("vimnmx3+hadd2");
  run<7, 5>("vimnmx3+hmnmx2");
  run<7, 6>("vimnmx3+hfma2");
  run<0, 3>("iadd3+fmnmx");
  run<4, 5>("hadd2+hmnmx2");
  return 0;
}
