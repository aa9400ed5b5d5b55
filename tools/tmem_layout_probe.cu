// tmem_layout_probe.cu -- which TMEM lanes hold which accumulator rows for
//   (a) tcgen05.mma cta_group::1, M=64   and   (b) cta_group::2, M=128 (64 rows per CTA).
// A[m][0] = m + 1 (other k = 0), B[n][k] = (k == 0): D[m][n] = m + 1.  Every warp reads
// its 32-lane quadrant, column 0, with 32x32b.x1; the host prints lane -> value.
#include <cuda_bf16.h>
#include <cstdio>

#include "tc_ptx.cuh"

using namespace rc::tc;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ float ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  return __uint_as_float(r);
}

template <int CG>
__global__ void __launch_bounds__(128, 1) probe(float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(smem);          // 128 x 64
  __nv_bfloat16* sB = reinterpret_cast<__nv_bfloat16*>(smem + 16384);  // 64 x 64
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  for (int i = tid; i < 128 * 64; i += 128) {
    const int m = i / 64, k = i % 64;
    // CG=2: this CTA supplies rows m of its half: global row = rank*64 + m
    const float v = (k == 0) ? (float)(CG == 2 ? rank * 64 + m + 1 : m + 1) : (k == 1 ? 1.f : 0.f);
    sA[sw128_offset(m, k) / 2] = __float2bfloat16(v);
  }
  for (int i = tid; i < 64 * 64; i += 128) sB[sw128_offset(i / 64, i % 64) / 2] = __float2bfloat16(i % 64 == 0 ? 128.f : (i % 64 == 1 ? (float)(i / 64) : 0.f));
  fence_proxy_async_smem();
  if (warp == 0) {
    if (CG == 1) {
      tmem_alloc<128>(&tbase);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t d = tbase;
  if (tid == 0 && rank == 0) {
    if (CG == 1) {
      const uint32_t idesc = idesc_bf16_f32(64, 64);
      mma_bf16_ss(d, desc_k_sw128(smem_u32(sA)), desc_k_sw128(smem_u32(sB)), idesc, 0);
      mma_commit(&bar);
    } else {
      const uint32_t idesc = idesc_bf16_f32(128, 64);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
          "l"(desc_k_sw128(smem_u32(sA))), "l"(desc_k_sw128(smem_u32(sB))), "r"(idesc), "r"(0));
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)3));
    }
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  out[(rank * 128 + warp * 32 + lane) * 2 + 0] = ld1(d + ((uint32_t)(warp * 32) << 16));
  out[(rank * 128 + warp * 32 + lane) * 2 + 1] = ld1(d + ((uint32_t)(warp * 32) << 16) + 31);
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  if (warp == 0) {
    if (CG == 1)
      tmem_dealloc<128>(tbase);
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;\n" ::"r"(tbase));
  }
}

int main() {
  float* out;
  cudaMalloc(&out, 512 * 4);
  const int smem = 16384 + 8192 + 1024;
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int cg = 1; cg <= 2; ++cg) {
    cudaMemset(out, 0, 512 * 4);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cg);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cg;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cg == 1 ? cudaLaunchKernelEx(&cfg, probe<1>, out) : cudaLaunchKernelEx(&cfg, probe<2>, out);
    cudaError_t e2 = cudaDeviceSynchronize();
    float h[512];
    cudaMemcpy(h, out, 512 * 4, cudaMemcpyDeviceToHost);
    printf("cta_group::%d %s %s\n", cg, cudaGetErrorString(e), cudaGetErrorString(e2));
    for (int r = 0; r < cg; ++r) {
      printf(" rank %d lane:value(col0/col5)", r);
      for (int l = 0; l < 128; ++l) printf(" %d:%g/%g", l, h[(r * 128 + l) * 2], h[(r * 128 + l) * 2 + 1]);
      printf("\n");
    }
  }
  return 0;
}
