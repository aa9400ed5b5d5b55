// tc_microbench.cu -- measures, on one B200 SM, the numbers the tensor-core RI kernel
// design depends on:
//   1. tcgen05.mma kind::f16 SS, M=128, N in {32,64,128,256}: correctness of our
//      descriptor encodings + cycles per K=16 MMA (smem-operand bandwidth limit);
//   2. tcgen05.ld 32x32b.x32 throughput with 4/8/16 warps (TMEM -> RF bytes/cycle).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_08888_b200/csrc
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_ptx.cuh"

using namespace rc::tc;

template <int N>
__global__ void __launch_bounds__(128, 1)
    mma_bench(int iters, const __nv_bfloat16* Ag, const __nv_bfloat16* Bg, float* out,
              long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* sB = reinterpret_cast<__nv_bfloat16*>(smem + 16384);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 128 * 64; i += blockDim.x) sA[sw128_offset(i / 64, i % 64) / 2] = Ag[i];
  for (int i = tid; i < N * 64; i += blockDim.x) sB[sw128_offset(i / 64, i % 64) / 2] = Bg[i];
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  const uint32_t idesc = idesc_bf16_f32(128, N);
  const uint64_t da = desc_k_sw128(smem_u32(sA)), db = desc_k_sw128(smem_u32(sB));
  long long t0 = clock64();
  if (tid == 0) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, da + 2 * kk, db + 2 * kk, idesc, (it | kk) != 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  long long t1 = clock64();
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(d + ((uint32_t)(warp * 32) << 16) + c0, v);
    tmem_wait_ld();
    for (int j = 0; j < 32 && c0 + j < N; ++j) out[(warp * 32 + lane) * N + c0 + j] = v[j];
  }
  if (tid == 0) cycles[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int NCOL>
__device__ __forceinline__ float ldtm_sum(uint32_t taddr) {
  uint32_t r[32];
  if constexpr (NCOL == 2)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
  else if constexpr (NCOL == 8)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  else if constexpr (NCOL == 16) {
    float v[16];
    tmem_ld16(taddr, v);
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(v[i]);
  } else {
    float v[32];
    tmem_ld32(taddr, v);
    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(v[i]);
  }
  tmem_wait_ld();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < NCOL; ++i) acc += __uint_as_float(r[i]);
  return acc;
}

// TMEM -> RF: each warp issues LOADS back-to-back loads of NCOL columns, then one wait
template <int NCOL, int LOADS>
__global__ void ld_bench(int reps, float* sink, long long* cycles) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tbase + ((uint32_t)((warp % 4) * 32) << 16);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int l = 0; l < LOADS; ++l) acc += ldtm_sum<NCOL>(base + ((r * LOADS + l) * NCOL + warp * 3) % (512 - NCOL));
  }
  __syncthreads();
  long long t1 = clock64();
  sink[tid] = acc;
  if (tid == 0) cycles[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

template <int N>
void run_mma() {
  std::vector<__nv_bfloat16> A(128 * 64), B(N * 64);
  std::vector<float> Af(128 * 64), Bf(N * 64);
  srand(N);
  for (int i = 0; i < 128 * 64; ++i) { Af[i] = (float)(rand() % 5 - 2); A[i] = __float2bfloat16(Af[i]); }
  for (int i = 0; i < N * 64; ++i) { Bf[i] = (float)(rand() % 5 - 2); B[i] = __float2bfloat16(Bf[i]); }
  __nv_bfloat16 *dA, *dB;
  float* dout;
  long long* dcyc;
  CK(cudaMalloc(&dA, A.size() * 2));
  CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMalloc(&dout, 128 * N * 4));
  CK(cudaMalloc(&dcyc, 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  const int smem = 16384 + N * 128 + 1024;
  CK(cudaFuncSetAttribute(mma_bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  mma_bench<N><<<1, 128, smem>>>(1, dA, dB, dout, dcyc);
  CK(cudaDeviceSynchronize());
  std::vector<float> out(128 * N);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int k = 0; k < 64; ++k) ref += Af[m * 64 + k] * Bf[n * 64 + k];
      if (ref != out[m * N + n]) ++bad;
    }
  const int iters = 2000;
  mma_bench<N><<<1, 128, smem>>>(iters, dA, dB, dout, dcyc);
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
  const double per_mma = (double)cyc / (iters * 4);
  const double macs = 128.0 * N * 16 / per_mma;
  const double bytes = (128.0 * 32 + N * 32) / per_mma;
  printf("{\"test\":\"mma_ss\",\"M\":128,\"N\":%d,\"correct\":%s,\"mismatches\":%d,\"cycles_per_mma_k16\":%.2f,"
         "\"macs_per_cycle\":%.1f,\"smem_operand_bytes_per_cycle\":%.1f}\n",
         N, bad == 0 ? "true" : "false", bad, per_mma, macs, bytes);
  cudaFree(dA); cudaFree(dB); cudaFree(dout); cudaFree(dcyc);
}

template <int NCOL>
void run_ld(int warps) {
  float* sink;
  long long* dcyc;
  CK(cudaMalloc(&sink, 4096 * 4));
  CK(cudaMalloc(&dcyc, 8));
  const int reps = 2000;
  ld_bench<NCOL, 1><<<1, warps * 32>>>(reps, sink, dcyc);
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
  const double bytes = (double)reps * warps * 32 * NCOL * 4;
  printf("{\"test\":\"tmem_ld_roundtrip\",\"cols\":%d,\"warps\":%d,\"cycles_per_load_per_warp\":%.1f,"
         "\"bytes_per_cycle\":%.1f}\n", NCOL, warps, (double)cyc / reps, bytes / cyc);
  cudaFree(sink); cudaFree(dcyc);
}

int main() {
  run_mma<32>();
  run_mma<64>();
  run_mma<128>();
  run_mma<256>();
  run_ld<2>(16);
  run_ld<8>(16);
  run_ld<16>(16);
  run_ld<32>(16);
  run_ld<8>(4);
  run_ld<16>(4);
  return 0;
}
