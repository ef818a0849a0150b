#include <cstdio>
#include <cstdint>
__global__ void k(const int* keys, const unsigned* vals, unsigned* out, int* ok) {
  const int lane = threadIdx.x & 31;
  const int key = keys[threadIdx.x];
  const unsigned v = vals[threadIdx.x];
  const unsigned grp = __match_any_sync(0xFFFFFFFFu, key);
  const unsigned s = __reduce_add_sync(grp, v);
  // reference: manual
  unsigned r = 0;
  for (int l = 0; l < 32; ++l) {
    const unsigned vv = __shfl_sync(0xFFFFFFFFu, v, l);
    const int kk = __shfl_sync(0xFFFFFFFFu, key, l);
    if (kk == key) r += vv;
  }
  out[threadIdx.x] = s;
  if (s != r) atomicAdd(ok, 1);
}
int main() {
  const int n = 32 * 64;
  int hk[n]; unsigned hv[n];
  unsigned seed = 1;
  for (int i = 0; i < n; ++i) { seed = seed * 1664525u + 1013904223u; hk[i] = (seed >> 28) % (1 + (i / 32) % 6); hv[i] = seed >> 8; }
  int* dk; unsigned* dv; unsigned* o; int* ok;
  cudaMalloc(&dk, sizeof hk); cudaMalloc(&dv, sizeof hv); cudaMalloc(&o, sizeof hv); cudaMalloc(&ok, 4);
  cudaMemcpy(dk, hk, sizeof hk, cudaMemcpyHostToDevice); cudaMemcpy(dv, hv, sizeof hv, cudaMemcpyHostToDevice);
  cudaMemset(ok, 0, 4);
  k<<<n / 256, 256>>>(dk, dv, o, ok);
  int bad; cudaMemcpy(&bad, ok, 4, cudaMemcpyDeviceToHost);
  printf("mismatches: %d (err %s)\n", bad, cudaGetErrorString(cudaGetLastError()));
}
