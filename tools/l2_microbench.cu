// l2_microbench.cu -- L2 -> SMEM streaming bandwidth with the TMA engine (cp.async.bulk),
// the rate at which the tensor-core RI kernel can re-stream its weight tiles.
// Every CTA streams TILE-byte tiles from an L2-resident region through a STAGES-deep smem
// ring (producer = one thread, consumer = one warp that just releases the slot).
//   mode 0: CTAs start at staggered tile offsets of a shared region (different tiles in flight)
//   mode 1: all CTAs read the same tile sequence (maximal L2 sharing)
//   mode 2: cluster of 2, each tile multicast to both CTAs of the cluster
// Prints aggregate bytes delivered into shared memory per SM-cycle and TB/s.
#include <cstdio>
#include <cstdlib>

#include "tc_ptx.cuh"

using namespace rc::tc;


__device__ __forceinline__ void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
      "[%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int TILE, int STAGES>
__global__ void __launch_bounds__(64, 1)
    stream_kernel(const uint8_t* __restrict__ src, size_t region, int ntiles, int mode, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x;
  const bool mc = mode >= 2;
  const uint32_t csize = mode == 3 ? 4 : 2;
  const uint32_t crank = mc ? cluster_rank() : 0;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mc ? csize : 1);  // multicast: every CTA must free the slot
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (mc) cluster_sync();
  const size_t tiles_in_region = region / TILE;
  const size_t start = (mode == 0 || mode == 4) ? (size_t)blockIdx.x * 37 : 0;
  long long t0 = clock64();
  if (mode == 4 && tid < 32) {
    // each stage issued as 4 sub-copies from 4 different lanes
    for (int i = 0; i < ntiles; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      if (i >= STAGES) mbar_wait(&empty[s], ph ^ 1);
      if (tid == 0) mbar_arrive_expect_tx(&full[s], TILE);
      __syncwarp();
      const uint8_t* g = src + ((start + i) % tiles_in_region) * TILE;
      if (tid < 4) bulk_g2s(smem + s * TILE + tid * (TILE / 4), g + tid * (TILE / 4), TILE / 4, &full[s]);
      __syncwarp();
    }
  } else if (tid == 0) {
    for (int i = 0; i < ntiles; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      if (i >= STAGES) mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], TILE);
      const uint8_t* g = src + ((start + i) % tiles_in_region) * TILE;
      if (!mc) {
        bulk_g2s(smem + s * TILE, g, TILE, &full[s]);
      } else {
        // each CTA issues 1/csize of the tile, multicast to every CTA of the cluster
        const uint32_t part = TILE / csize;
        bulk_g2s_mc(smem + s * TILE + crank * part, g + crank * part, part, &full[s],
                    (uint16_t)((1u << csize) - 1));
      }
    }
  } else if (tid == 32) {
    for (int i = 0; i < ntiles; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      if (!mc) {
        mbar_arrive(&empty[s]);
      } else {
        // release the slot in both CTAs of the pair (remote arrive through DSMEM)
        for (uint32_t peer = 0; peer < csize; ++peer) {
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(&empty[s])), "r"(peer));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
        }
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (mc) cluster_sync();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int TILE, int STAGES>
void run(const uint8_t* src, size_t region, long long* cyc, int sms, int per_sm, int mode) {
  const int ntiles = 48000000 / TILE * 4;
  auto fn = stream_kernel<TILE, STAGES>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * TILE);
  const int grid = sms * per_sm;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = STAGES * TILE;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = mode == 2 ? 2 : (mode == 3 ? 4 : 1);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, src, region, ntiles, mode, cyc);
    cudaEventRecord(b);
    cudaError_t e2 = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)grid * ntiles * TILE;  // bytes landed in shared memory
    const double l2 = mode >= 2 ? bytes / (mode == 2 ? 2 : 4) : bytes;
    if (rep == 1)
      printf("{\"test\":\"l2_stream\",\"tile\":%d,\"stages\":%d,\"ctas_per_sm\":%d,\"mode\":%d,\"err\":\"%s/%s\","
             "\"ms\":%.3f,\"smem_fill_TBps\":%.2f,\"l2_read_TBps\":%.2f}\n",
             TILE, STAGES, per_sm, mode, cudaGetErrorString(e), cudaGetErrorString(e2), ms, bytes / ms / 1e9,
             l2 / ms / 1e9);
  }
}

int main() {
  const size_t region = 9437184;  // 9 MB: one C3 base kernel set in bf16
  uint8_t* src;
  cudaMalloc(&src, region);
  cudaMemset(src, 1, region);
  long long* cyc;
  cudaMalloc(&cyc, 4096 * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<16384, 4>(src, region, cyc, sms, 1, 0);
  run<65536, 3>(src, region, cyc, sms, 1, 0);
  run<65536, 3>(src, region, cyc, sms, 1, 4);
  run<32768, 6>(src, region, cyc, sms, 1, 4);
  run<16384, 8>(src, region, cyc, sms, 1, 4);
  run<65536, 2>(src, region, cyc, sms, 1, 4);
  return 0;
}
