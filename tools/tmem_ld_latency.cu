// tmem_ld_latency.cu -- does a busy MMA stream delay tcgen05.ld?  One CTA: warp 0 issues a
// continuous stream of tcgen05.mma (M=128, N=96, K=16, SS) into TMEM columns [0, 96) (or
// nothing, mode 0); warps 4-7 (the four lane quadrants) time round trips of
// tcgen05.ld 32x32b.x16 + tcgen05.wait::ld on columns [256, 272).  Prints the mean cycles per
// round trip for each mode.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_08888_b200/csrc
#include <cuda_bf16.h>

#include <cstdio>
#include <vector>

#include "tc_ptx.cuh"

using namespace rc::tc;

__global__ void __launch_bounds__(256, 1) probe(int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < (128 + 96) * 64; i += blockDim.x)
    reinterpret_cast<__nv_bfloat16*>(smem)[i] = __float2bfloat16(0.5f);
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    stop = 0;
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  if (warp == 0) {
    if (mode == 1 && elect_one()) {
      const uint64_t da = desc_k_sw128(smem_u32(smem)), db = desc_k_sw128(smem_u32(smem) + 128 * 128);
      const uint32_t idesc = idesc_bf16_f32(128, 96);
      long long n = 0;
      while (!stop) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(t, da + 2 * kk, db + 2 * kk, idesc, 1);
        ++n;
      }
      out[8] = n;
      mma_commit(&bar);  // drain before the TMEM is freed
    }
    __syncwarp();
    if (mode == 1) mbar_wait(&bar, 0);
  } else if (warp >= 4) {
    const uint32_t a = t + ((uint32_t)((warp % 4) * 32) << 16) + 256;
    float v[16];
    float acc = 0.f;
    for (int i = 0; i < 64; ++i) {  // warm up
      tmem_ld16(a, v);
      tmem_wait_ld();
      acc += v[0];
    }
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      tmem_ld16(a, v);
      tmem_wait_ld();
      acc += v[i & 15];
    }
    const long long t1 = clock64();
    if ((tid & 31) == 0) out[warp - 4] = t1 - t0;
    if (acc == 12345.f) out[9] = 1;
    __syncwarp();
    if (warp == 4 && (tid & 31) == 0) stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  const int smem = (128 + 96) * 128 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d, 0, 16 * sizeof(long long));
    probe<<<1, 256, smem>>>(mode, iters, d);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("{\"mode\":%d,\"error\":\"%s\"}\n", mode, cudaGetErrorString(e));
      return 1;
    }
    long long h[16];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int w = 0; w < 4; ++w) mean += (double)h[w] / iters / 4;
    printf("{\"mode\":\"%s\",\"cycles_per_tmem_ld16_round_trip\":%.1f,\"mma_groups_issued\":%lld}\n",
           mode ? "concurrent MMA stream (M128 N96 K16 SS)" : "idle tensor core", mean, h[8]);
  }
  return 0;
}
