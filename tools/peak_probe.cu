// peak_probe.cu -- measured compute peaks of this B200 for the roofline denominators that
// MEASURED_PEAKS.json does not hold (it has HBM and dense bf16 from cuBLAS):
//   ffma   : FP32 FMA on the CUDA cores (scalar FFMA), all SMs, 8 independent chains/thread
//   ffma2  : packed FP32x2 FMA (__ffma2_rn -> FFMA2), the instruction the SIMT kernel uses
//   tf32   : tcgen05.mma kind::tf32, M = 128, N = 256, K = 8, operands in shared memory
//   bf16   : tcgen05.mma kind::f16 (bf16), M = 128, N = 256, K = 16, same loop (cross-check
//            against the cuBLAS number)
// One JSON line per measurement: TFLOP/s over the whole GPU (2 FLOP per FMA / MAC), CUDA-event
// time of a launch after warm-up, SM clock sampled by the caller.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_08888_b200/csrc
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "tc_ptx.cuh"

using namespace rc::tc;

template <bool PAIRED>
__global__ void __launch_bounds__(512) ffma_kernel(int iters, float* out) {
  float a[8], b = 1.0000001f, c = 1e-7f;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  if constexpr (!PAIRED) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
  } else {
    float2* a2 = reinterpret_cast<float2*>(a);
    const float2 b2 = make_float2(b, b), c2 = make_float2(c, c);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 4; ++i) a2[i] = __ffma2_rn(a2[i], b2, c2);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[threadIdx.x] = s;  // keep the chains alive
}

// one CTA per SM; warp 0 allocates TMEM, one thread issues `iters` x 4 MMAs (K = 64 bytes of
// operand per row, 4 K-steps) into one accumulator, then commits
template <bool TF32>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int N = 256;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = TF32 ? 0x3f800000u : 0x3f803f80u;  // 1.0
  fence_proxy_async_smem();
  if (threadIdx.x / 32 == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  // kind::f16 (bf16): a/b format 1; kind::tf32: a/b format 2; D f32
  const uint32_t idesc = (1u << 4) | ((TF32 ? 2u : 1u) << 7) | ((TF32 ? 2u : 1u) << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((128u >> 4) << 24);
  const uint64_t da = desc_k_sw128(smem_u32(smem)), db = desc_k_sw128(smem_u32(smem + 128 * 128));
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (it | kk) != 0;
        if constexpr (TF32)
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(idesc), "r"(acc));
        else
          mma_bf16_ss(d, da + 2 * kk, db + 2 * kk, idesc, acc);
      }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 0) tmem_dealloc<512>(d);
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                  \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

template <typename F>
static float time_ms(F launch) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* out;
  long long* cyc;
  CK(cudaMalloc(&out, 4096 * sizeof(float)));
  CK(cudaMalloc(&cyc, 1024 * sizeof(long long)));
  const int iters = 1 << 16, threads = 512, blocks = sms * 4;
  for (int paired = 0; paired < 2; ++paired) {
    const float ms = time_ms([&] {
      if (paired)
        ffma_kernel<true><<<blocks, threads>>>(iters, out);
      else
        ffma_kernel<false><<<blocks, threads>>>(iters, out);
    });
    const double flop = 2.0 * 8 * (double)iters * threads * blocks;
    printf("{\"test\": \"%s\", \"tflops\": %.2f, \"ms\": %.4f, \"blocks\": %d, \"threads\": %d}\n",
           paired ? "ffma2" : "ffma", flop / (ms * 1e-3) / 1e12, ms, blocks, threads);
  }
  const int smem = (128 + 256) * 128 + 1024;
  CK(cudaFuncSetAttribute(mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int miters = 1 << 14;
  for (int tf = 1; tf >= 0; --tf) {
    const float ms = time_ms([&] {
      if (tf)
        mma_kernel<true><<<sms, 128, smem>>>(miters, cyc);
      else
        mma_kernel<false><<<sms, 128, smem>>>(miters, cyc);
    });
    const int k = tf ? 8 : 16;  // K per instruction
    const double flop = 2.0 * 128 * 256 * k * 4.0 * miters * sms;
    long long c0;
    CK(cudaMemcpy(&c0, cyc, sizeof(long long), cudaMemcpyDeviceToHost));
    printf("{\"test\": \"%s\", \"tflops\": %.1f, \"ms\": %.4f, \"cycles_per_mma\": %.2f, \"M\": 128, \"N\": 256, \"K\": %d}\n",
           tf ? "tcgen05_tf32" : "tcgen05_bf16", flop / (ms * 1e-3) / 1e12, ms, (double)c0 / (4.0 * miters), k);
  }
  return 0;
}
