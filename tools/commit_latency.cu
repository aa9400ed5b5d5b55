// commit_latency.cu -- how long after its MMAs does a tcgen05.commit mbarrier arrive?
// One thread issues K MMAs (M=128, N=96, K=16 bf16, SS), commits, then polls the barrier
// with test_wait and records clock64 deltas; K in {1, 4, 12, 24, 48, 96}.
#include <cuda_bf16.h>
#include <cstdio>
#include "tc_ptx.cuh"
using namespace rc::tc;

__global__ void probe(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x;
  for (int i = tid; i < (16384 + 96 * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async_smem();
  if (tid < 32) tmem_alloc<512>(&tb);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 96);
    const uint64_t da = desc_k_sw128(smem_u32(smem)), db = desc_k_sw128(smem_u32(smem + 16384));
    const int Ks[6] = {1, 4, 12, 24, 48, 96};
    uint32_t ph = 0;
    for (int rep = 0; rep < 2; ++rep)
      for (int j = 0; j < 6; ++j) {
        const long long t0 = clock64();
        for (int m = 0; m < Ks[j]; ++m) mma_bf16_ss(tb, da, db, idesc, m != 0);
        const long long t1 = clock64();
        mma_commit(&bar);
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(ok) : "r"(smem_u32(&bar)), "r"(ph) : "memory");
        const long long t2 = clock64();
        ph ^= 1;
        if (rep == 1) {
          out[j * 3 + 0] = Ks[j];
          out[j * 3 + 1] = t1 - t0;
          out[j * 3 + 2] = t2 - t0;
        }
      }
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<512>(tb);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 64 * 1024>>>(d);
  long long h[18];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int j = 0; j < 6; ++j)
    printf("{\"mmas\":%lld,\"issue_cycles\":%lld,\"commit_arrive_cycles\":%lld,\"per_mma\":%.1f}\n", h[j * 3],
           h[j * 3 + 1], h[j * 3 + 2], (double)h[j * 3 + 2] / h[j * 3]);
  return 0;
}
