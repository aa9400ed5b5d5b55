// m64_probe.cu -- tcgen05.mma kind::f16 M=64 vs M=128 throughput (SS, K=16)
#include <cuda_bf16.h>
#include <cstdio>
#include "tc_ptx.cuh"
using namespace rc::tc;
template <int M, int N>
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x;
  for (int i = tid; i < (16384 + 256 * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  fence_proxy_async_smem();
  if (tid < 32) tmem_alloc<512>(&tb);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_f32(M, N);
    const uint64_t da = desc_k_sw128(smem_u32(smem)), db = desc_k_sw128(smem_u32(smem + 16384));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tb, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads();
  if (tid < 32) tmem_dealloc<512>(tb);
}
template <int M, int N> void run() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 2000;
  probe<M, N><<<1, 128, 64 * 1024>>>(d, iters);
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"M\":%d,\"N\":%d,\"err\":\"%s\",\"cycles_per_mma\":%.2f,\"macs_per_cycle\":%.0f}\n", M, N,
         cudaGetErrorString(cudaGetLastError()), h / (4.0 * iters), M * N * 16.0 * 4 * iters / h);
}
int main() { run<128, 96>(); run<64, 96>(); run<64, 128>(); run<64, 256>(); run<128, 256>(); return 0; }
