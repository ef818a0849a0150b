#include <cstdio>
__global__ void k(double* out, int iters, double p) {
  double x = threadIdx.x * 1e-3, y = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = x + p; }
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) { y = fma(y, p, 1e-9); }
  long long t2 = clock64();
  double z = 1.0;
  for (int i = 0; i < iters; ++i) { z = z * p; }
  long long t3 = clock64();
  float f = 1.0f;
  for (int i = 0; i < iters; ++i) { f = f + float(p); }
  long long t4 = clock64();
  out[threadIdx.x] = x + y + z + f;
  if (threadIdx.x == 0) printf("dadd %.1f dfma %.1f dmul %.1f fadd %.1f cycles\n", double(t1 - t0) / iters, double(t2 - t1) / iters, double(t3 - t2) / iters, double(t4-t3)/iters);
}
int main() { double* d; cudaMalloc(&d, 1024 * 8); k<<<1, 32>>>(d, 10000, 1.0000001); cudaDeviceSynchronize(); return 0; }
