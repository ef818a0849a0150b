// pdl_probe.cu — per-kernel cost of a captured graph of K dependent kernels on
// ONE stream (the serial frame's launch chain), plain vs programmatic
// dependent launch (griddepcontrol.wait at kernel entry, launch_dependents
// right after it).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_probe tools/pdl_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

template <bool PDL>
__global__ void k_tiny(int* p, int n) {
  if (PDL) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] += 1;
}

template <bool PDL>
float run(int K, int blocks, int* buf, cudaStream_t st) {
  cudaGraph_t g;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < K; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = blocks;
    cfg.blockDim = 256;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = PDL ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_tiny<PDL>, buf, blocks * 256);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphExec_t ex;
  if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
    printf("instantiate failed\n");
    return -1;
  }
  for (int r = 0; r < 3; ++r) cudaGraphLaunch(ex, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 50;
  cudaEventRecord(a, st);
  for (int r = 0; r < reps; ++r) cudaGraphLaunch(ex, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ex);
  cudaGraphDestroy(g);
  return ms * 1e3f / (reps * K);
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* buf;
  cudaMalloc(&buf, sizeof(int) * 4096 * 256);
  cudaMemset(buf, 0, sizeof(int) * 4096 * 256);
  for (int blocks : {1, 148, 1024, 4096}) {
    const float a = run<false>(109, blocks, buf, st);
    const float b = run<true>(109, blocks, buf, st);
    printf("K=109 blocks=%4d: plain %.2f us/kernel, PDL %.2f us/kernel\n", blocks, a, b);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
