// Minimal TMA load/store probe (debug tool).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
struct Args { CUtensorMap m; int x, y, z; };
#ifndef SX
#define SX 8
#endif
#ifndef SY
#define SY 1
#endif
__device__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ Args a, uint32_t* out, int n) {
  extern __shared__ uint8_t raw[];
  uint32_t* buf = (uint32_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(n * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(sa(buf)), "l"((uint64_t)&a.m), "r"(a.x), "r"(a.y), "r"(a.z), "r"(sa(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" :: "r"(sa(&bar)) : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
      :: "l"((uint64_t)&a.m), "r"(a.x + SX), "r"(a.y + SY), "r"(0), "r"(sa(buf)) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(1) : "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  int W = 140, H = 41, wpp = 1; size_t pitch = ((W * wpp * 4 + 15) / 16) * 16;
  std::vector<uint32_t> h(pitch / 4 * H * 2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = i;
  uint32_t* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  int bx = atoi(getenv("BX") ? getenv("BX") : "8"), by = atoi(getenv("BY") ? getenv("BY") : "32");
  Args a{}; a.x = 0; a.y = 0; a.z = 1;
  cuuint64_t dims[3] = {(cuuint64_t)W * wpp, (cuuint64_t)H, 2}; cuuint64_t str[2] = {pitch, pitch * H};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&a.m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d box %d x %d\n", (int)r, bx, by);
  uint32_t* o; cudaMalloc(&o, 65536 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<1, 32, 2048 + bx * by * 4>>>(a, o, bx * by);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint32_t> ho(bx * by); cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
  printf("first %u %u expect %zu\n", ho[0], ho[bx], pitch / 4 * H);
}
