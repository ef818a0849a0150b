// dpx_probe.cu — latency / throughput of the integer ops the SGM recurrence
// uses (VIADDMNMX.U16x2, VIMNMX.U16x2, VIMNMX3.U16x2, PRMT, IADD3) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dpx_probe tools/dpx_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

template <int OP, int CHAINS>
__global__ void k_probe(uint32_t* out, int iters, uint32_t p) {
  uint32_t x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 7u + c;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) x[c] = __viaddmin_u16x2(x[c], p, x[(c + 1) % CHAINS] ^ p);
      if (OP == 1) x[c] = __vminu2(x[c] ^ p, x[(c + 1) % CHAINS]);
      if (OP == 2) x[c] = __vimin3_u16x2(x[c], p, x[(c + 1) % CHAINS] + 1u);
      if (OP == 3) x[c] = __byte_perm(x[c], x[(c + 1) % CHAINS], 0x5432) + p;
      if (OP == 4) x[c] = x[c] + x[(c + 1) % CHAINS] - p;
      if (OP == 5) {  // HMNMX2
        __half2 a = *reinterpret_cast<__half2*>(&x[c]), b = *reinterpret_cast<__half2*>(&x[(c + 1) % CHAINS]);
        __half2 r = __hmin2(a, b);
        x[c] = *reinterpret_cast<uint32_t*>(&r) ^ p;
      }
      if (OP == 6) {  // HADD2
        __half2 a = *reinterpret_cast<__half2*>(&x[c]), b = *reinterpret_cast<__half2*>(&x[(c + 1) % CHAINS]);
        __half2 r = __hadd2(a, b);
        x[c] = *reinterpret_cast<uint32_t*>(&r);
      }
      if (OP == 7) {  // HMNMX2 + HADD2 chain without integer ops
        __half2 a = *reinterpret_cast<__half2*>(&x[c]), b = *reinterpret_cast<__half2*>(&x[(c + 1) % CHAINS]);
        __half2 r = __hmin2(__hadd2(a, b), b);
        x[c] = *reinterpret_cast<uint32_t*>(&r);
      }
      if (OP == 8) x[c] = min(x[c], x[(c + 1) % CHAINS] + p);  // IMNMX (u32)
      if (OP == 9) {  // FMNMX
        float a = __uint_as_float(x[c]), b = __uint_as_float(x[(c + 1) % CHAINS]);
        x[c] = __float_as_uint(fminf(a + 1.0f, b));
      }
    }
  }
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = uint32_t(t1 - t0);
}

template <int OP, int CHAINS>
void run(const char* name, int blocks, int threads) {
  uint32_t* d;
  cudaMalloc(&d, sizeof(uint32_t) * blocks * threads);
  const int iters = 4096;
  k_probe<OP, CHAINS><<<blocks, threads>>>(d, iters, 0x00050005u);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_probe<OP, CHAINS><<<blocks, threads>>>(d, iters, 0x00050005u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  uint32_t cyc;
  cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
  // each inner op is ~2 SASS instructions (the op + the xor/add feeding it)
  const double ops = double(blocks) * threads * iters * CHAINS;
  printf("%-14s chains=%d blocks=%4d thr=%4d: %.1f cycles/op/thread (cta0), %.1f Gop/s, %.2f warp-op/clk/SM\n",
         name, CHAINS, blocks, threads, double(cyc) / (iters * CHAINS), ops / (ms * 1e-3) / 1e9,
         ops / 32.0 / (ms * 1e-3) / 1.965e9 / 148.0);
  cudaFree(d);
}

int main() {
  // latency: one warp, one chain
  run<0, 1>("viaddmin", 1, 32);
  run<1, 1>("vminu2", 1, 32);
  run<2, 1>("vimin3", 1, 32);
  run<3, 1>("prmt+add", 1, 32);
  run<4, 1>("iadd3", 1, 32);
  // throughput: full GPU, 8 chains per thread
  run<0, 8>("viaddmin", 148 * 8, 256);
  run<1, 8>("vminu2", 148 * 8, 256);
  run<2, 8>("vimin3", 148 * 8, 256);
  run<3, 8>("prmt+add", 148 * 8, 256);
  run<4, 8>("iadd3", 148 * 8, 256);
  run<5, 8>("hmnmx2", 148 * 8, 256);
  run<6, 8>("hadd2", 148 * 8, 256);
  run<7, 8>("hadd2+hmnmx2", 148 * 8, 256);
  run<8, 8>("imnmx+add", 148 * 8, 256);
  run<9, 8>("fadd+fmnmx", 148 * 8, 256);
  run<5, 1>("hmnmx2", 1, 32);
  run<7, 1>("hadd2+hmnmx2", 1, 32);
  // one warp per SMSP with 8 chains (the aggregation's regime)
  run<0, 8>("viaddmin", 148, 128);
  run<4, 8>("iadd3", 148, 128);
  return 0;
}
