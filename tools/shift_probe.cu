// shift_probe.cu -- can a tcgen05 SW128 K-major operand start at an arbitrary 128-byte row
// of a 1024-byte-aligned swizzled tile?  (implicit-GEMM convolution: a tap = a row shift)
// A: 256 rows x 64 K (bf16) in SW128 K-major; B: 64 rows x 64 K.  For each shift s the MMA
// uses A rows s .. s+127 (descriptor start = base + 128*s, with the matrix base-offset field
// 0 or (s & 7)) and D is compared with the CPU product.  One JSON line per (s, mode).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_08888_b200/csrc
#include <cuda_bf16.h>

#include <cstdio>
#include <vector>

#include "tc_ptx.cuh"

using namespace rc::tc;

constexpr int AR = 256, N = 64;

__global__ void __launch_bounds__(128, 1)
    probe(int s, int mode, const __nv_bfloat16* Ag, const __nv_bfloat16* Bg, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* sB = reinterpret_cast<__nv_bfloat16*>(smem + AR * 128);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < AR * 64; i += blockDim.x) sA[sw128_offset(i / 64, i % 64) / 2] = Ag[i];
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
  if (tid == 0) {
    uint64_t da = desc_k_sw128(smem_u32(sA) + 128 * s);
    if (mode == 1) da |= (uint64_t)(s & 7) << 49;
    const uint64_t db = desc_k_sw128(smem_u32(sB));
    const uint32_t idesc = idesc_bf16_f32(128, N);
    for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tbase, da + 2 * kk, db + 2 * kk, idesc, kk != 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  for (int c = 0; c < N; c += 32) {
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) out[tid * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

// MN-major B: B stored as [K rows][64 N] (one SW128 row = 64 N-elements of one k), the
// implicit-GEMM X layout.  D[m][n] = sum_k A[m][k] * B[s + k][n] for K = 64 (4 MMAs of
// K = 16, each +16 rows), B descriptor start = base + 128 * s, idesc B-major bit set.
constexpr int BR = 256;
__global__ void __launch_bounds__(128, 1)
    probe_mn(int s, const __nv_bfloat16* Ag, const __nv_bfloat16* Bg, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(smem);            // [128 m][64 k] K-major
  __nv_bfloat16* sB = reinterpret_cast<__nv_bfloat16*>(smem + 128 * 128);  // [BR k][64 n] MN-major
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 128 * 64; i += blockDim.x) sA[sw128_offset(i / 64, i % 64) / 2] = Ag[i];
  for (int i = tid; i < BR * 64; i += blockDim.x) sB[sw128_offset(i / 64, i % 64) / 2] = Bg[i];
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint64_t da = desc_k_sw128(smem_u32(sA));
    const uint64_t db = desc_k_sw128(smem_u32(sB) + 128 * s);
    const uint32_t idesc = idesc_bf16_f32(128, 64) | (1u << 16);  // B MN-major
    for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tbase, da + 2 * kk, db + (uint64_t)(kk * 2048 >> 4), idesc, kk != 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  for (int c = 0; c < 64; c += 32) {
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) out[tid * 64 + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

// MN-major B with N = 128: two 64-wide MN atoms [BR k][64 n] stored `lbo` bytes apart (the
// descriptor's leading-byte offset), row shift s as before.
__global__ void __launch_bounds__(128, 1)
    probe_mn128(int s, int lbo, const __nv_bfloat16* Ag, const __nv_bfloat16* Bg, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(smem);
  uint8_t* sB = smem + 128 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 128 * 64; i += blockDim.x) sA[sw128_offset(i / 64, i % 64) / 2] = Ag[i];
  for (int i = tid; i < BR * 128; i += blockDim.x) {  // Bg [k][128 n]
    const int k = i / 128, n = i % 128;
    reinterpret_cast<__nv_bfloat16*>(sB + (n / 64) * lbo)[sw128_offset(k, n % 64) / 2] = Bg[i];
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint64_t da = desc_k_sw128(smem_u32(sA));
    uint64_t db = desc_k_sw128(smem_u32(sB) + 128 * s);
    db = (db & ~(0x3FFFull << 16)) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16);
    const uint32_t idesc = idesc_bf16_f32(128, 128) | (1u << 16);
    for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tbase, da + 2 * kk, db + (uint64_t)(kk * 2048 >> 4), idesc, kk != 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  for (int c = 0; c < 128; c += 32) {
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) out[tid * 128 + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

int main() {
  std::vector<__nv_bfloat16> A(AR * 64), B(N * 64);
  std::vector<float> Af(AR * 64), Bf(N * 64);
  srand(1);
  for (int i = 0; i < AR * 64; ++i) A[i] = __float2bfloat16(Af[i] = (float)(rand() % 9 - 4));
  for (int i = 0; i < N * 64; ++i) B[i] = __float2bfloat16(Bf[i] = (float)(rand() % 9 - 4));
  __nv_bfloat16 *dA, *dB;
  float* dout;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dout, 128 * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = AR * 128 + N * 128 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> out(128 * N);
  const int shifts[] = {0, 1, 2, 3, 5, 7, 8, 9, 13, 18, 34, 66, 127};
  for (int s : shifts)
    for (int mode = 0; mode < 2; ++mode) {
      probe<<<1, 128, smem>>>(s, mode, dA, dB, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("{\"shift\":%d,\"mode\":%d,\"error\":\"%s\"}\n", s, mode, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0, bad_vs_unshifted_rows = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          float ref = 0;
          for (int k = 0; k < 64; ++k) ref += Af[(s + m) * 64 + k] * Bf[n * 64 + k];
          if (ref != out[m * N + n]) ++bad;
        }
      (void)bad_vs_unshifted_rows;
      printf("{\"shift\":%d,\"mode\":%d,\"mismatches\":%d}\n", s, mode, bad);
    }
  {  // MN-major B row shifts
    std::vector<__nv_bfloat16> A2(128 * 64), B2(BR * 64);
    std::vector<float> A2f(128 * 64), B2f(BR * 64);
    for (int i = 0; i < 128 * 64; ++i) A2[i] = __float2bfloat16(A2f[i] = (float)(rand() % 9 - 4));
    for (int i = 0; i < BR * 64; ++i) B2[i] = __float2bfloat16(B2f[i] = (float)(rand() % 9 - 4));
    __nv_bfloat16 *dA2, *dB2;
    cudaMalloc(&dA2, A2.size() * 2);
    cudaMalloc(&dB2, B2.size() * 2);
    cudaMemcpy(dA2, A2.data(), A2.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB2, B2.data(), B2.size() * 2, cudaMemcpyHostToDevice);
    const int sm2 = 128 * 128 + BR * 128 + 2048;
    cudaFuncSetAttribute(probe_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    std::vector<float> o2(128 * 64);
    for (int s : {0, 1, 3, 7, 8, 9, 19, 37, 100}) {
      probe_mn<<<1, 128, sm2>>>(s, dA2, dB2, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("{\"mn_shift\":%d,\"error\":\"%s\"}\n", s, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(o2.data(), dout, o2.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          float ref = 0;
          for (int k = 0; k < 64; ++k) ref += A2f[m * 64 + k] * B2f[(s + k) * 64 + n];
          if (ref != o2[m * 64 + n]) ++bad;
        }
      printf("{\"mn_shift\":%d,\"mismatches\":%d}\n", s, bad);
    }
  }
  {  // MN-major B, N = 128 (two atoms LBO apart)
    std::vector<__nv_bfloat16> A3(128 * 64), B3(BR * 128);
    std::vector<float> A3f(128 * 64), B3f(BR * 128);
    for (int i = 0; i < 128 * 64; ++i) A3[i] = __float2bfloat16(A3f[i] = (float)(rand() % 9 - 4));
    for (int i = 0; i < BR * 128; ++i) B3[i] = __float2bfloat16(B3f[i] = (float)(rand() % 9 - 4));
    __nv_bfloat16 *dA3, *dB3;
    float* dout3;
    cudaMalloc(&dA3, A3.size() * 2);
    cudaMalloc(&dB3, B3.size() * 2);
    cudaMalloc(&dout3, 128 * 128 * 4);
    cudaMemcpy(dA3, A3.data(), A3.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB3, B3.data(), B3.size() * 2, cudaMemcpyHostToDevice);
    const int lbo = BR * 128;  // second atom right after the first [BR x 128 B] block
    const int sm3 = 128 * 128 + 2 * lbo + 2048;
    cudaFuncSetAttribute(probe_mn128, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3);
    std::vector<float> o3(128 * 128);
    for (int s : {0, 1, 5, 9, 37}) {
      probe_mn128<<<1, 128, sm3>>>(s, lbo, dA3, dB3, dout3);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("{\"mn128_shift\":%d,\"error\":\"%s\"}\n", s, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(o3.data(), dout3, o3.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 128; ++n) {
          float ref = 0;
          for (int k = 0; k < 64; ++k) ref += A3f[m * 64 + k] * B3f[(s + k) * 128 + n];
          if (ref != o3[m * 128 + n]) ++bad;
        }
      printf("{\"mn128_shift\":%d,\"lbo\":%d,\"mismatches\":%d}\n", s, lbo, bad);
    }
  }
  return 0;
}
