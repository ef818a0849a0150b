// launch_probe.cu — ceiling that kernel count alone puts on graph throughput:
// S streams each replaying a captured graph of K dependent kernels (tiny
// grids), graphs/s.  Compare with frames/s of the 107-kernel pipeline graph.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_probe tools/launch_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void k_tiny(int* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] += 1;
}

int main() {
  const int K = 107;
  for (int blocks : {1, 148, 1024}) {
    for (int S : {1, 8, 16, 32}) {
      std::vector<cudaStream_t> st(S);
      std::vector<cudaGraphExec_t> ex(S);
      std::vector<int*> buf(S);
      for (int s = 0; s < S; ++s) {
        cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking);
        cudaMalloc(&buf[s], sizeof(int) * blocks * 256);
        cudaMemset(buf[s], 0, sizeof(int) * blocks * 256);
        cudaGraph_t g;
        cudaStreamBeginCapture(st[s], cudaStreamCaptureModeThreadLocal);
        for (int k = 0; k < K; ++k) k_tiny<<<blocks, 256, 0, st[s]>>>(buf[s], blocks * 256);
        cudaStreamEndCapture(st[s], &g);
        cudaGraphInstantiate(&ex[s], g, 0);
        cudaGraphDestroy(g);
      }
      for (int r = 0; r < 3; ++r)
        for (int s = 0; s < S; ++s) cudaGraphLaunch(ex[s], st[s]);
      cudaDeviceSynchronize();
      const int reps = 64;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      for (int r = 0; r < reps; ++r)
        for (int s = 0; s < S; ++s) cudaGraphLaunch(ex[s], st[s]);
      for (int s = 0; s < S; ++s) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st[s]);
        cudaStreamWaitEvent(0, e, 0);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("K=%d blocks=%4d streams=%2d: %8.0f graphs/s (%.2f us per kernel)\n", K, blocks, S,
             reps * S / (ms * 1e-3), ms * 1e3 / (reps * S * K));
      for (int s = 0; s < S; ++s) {
        cudaGraphExecDestroy(ex[s]);
        cudaStreamDestroy(st[s]);
        cudaFree(buf[s]);
      }
    }
  }
  return 0;
}
