// tc_microbench2.cu -- tcgen05.mma throughput vs N and operand source on one B200 SM.
//   mma_ss  : A and B from shared memory (SW128 K-major), M=128, N in {64..256}
//   mma_ts  : A from TMEM (loaded with tcgen05.st), B from shared memory
//   pattern : the RI kernel's inner loop (bf16x3: 3 MMAs per K-step over hi/lo tiles of
//             4 ci-chunks), N = 96
// Prints one JSON line per measurement: cycles per K=16 MMA and MACs/cycle (peak 4096).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_08888_b200/csrc
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_ptx.cuh"

using namespace rc::tc;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// MODE 0: SS; MODE 1: TS (A in TMEM cols [256, 256+32)); MODE 2: kernel pattern (SS, 2 A tiles,
// 8 B tiles cycling, 3 MMAs per K step)
template <int N, int MODE>
__global__ void __launch_bounds__(128, 1)
    mma_bench(int iters, const __nv_bfloat16* Ag, const __nv_bfloat16* Bg, float* out, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int ATILE = 128 * 128;   // [128 x 64] bf16
  constexpr int BTILE = N * 128;     // [N x 64] bf16
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(smem);
  uint8_t* sB = smem + 2 * ATILE;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    sA[sw128_offset(i / 64, i % 64) / 2] = Ag[i];
    sA[ATILE / 2 + sw128_offset(i / 64, i % 64) / 2] = Ag[i];
  }
  const int nb = MODE == 8 ? 8 : (MODE >= 2 ? 8 : 1);  // B tiles
  for (int t = 0; t < nb; ++t)
    for (int i = tid; i < N * 64; i += blockDim.x)
      reinterpret_cast<__nv_bfloat16*>(sB + t * BTILE)[sw128_offset(i / 64, i % 64) / 2] = Bg[i];
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
  const uint32_t a_tm = tbase + 256;
  if (MODE == 1) {  // A rows -> TMEM lanes: row m, k pairs packed per 32-bit column
    const int m = tid;
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t r[8];
      for (int j = 0; j < 8; ++j) {
        const __nv_bfloat16 lo = Ag[m * 64 + kk * 16 + 2 * j], hi = Ag[m * 64 + kk * 16 + 2 * j + 1];
        r[j] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      tmem_st8(a_tm + ((uint32_t)(warp * 32) << 16) + kk * 8, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t idesc = idesc_bf16_f32(128, N);
  const uint64_t da = desc_k_sw128(smem_u32(sA)), db = desc_k_sw128(smem_u32(sB));
  __shared__ uint64_t full7[8], empty7[8];
  if (MODE >= 700 && tid == 0) {
    for (int i = 0; i < 8; ++i) {
      mbar_init(&full7[i], 1);
      mbar_init(&empty7[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (MODE >= 700 && tid == 32) {
    // producer warp: stage s may be (re)filled once the MMAs of its previous use completed
    constexpr int DEPTH = (MODE / 10) % 10, SC = MODE % 10;
    const int stages = (iters / 3) / SC;
    for (int st = 0; st < stages; ++st) {
      const int sidx = st % DEPTH;
      if (st >= DEPTH) mbar_wait(&empty7[sidx], ((st / DEPTH) - 1) & 1);
      mbar_arrive(&full7[sidx]);
    }
  }
  if (tid == 0) {
    if (MODE >= 700) {
      constexpr int DEPTH = (MODE / 10) % 10, SC = MODE % 10;
      const uint64_t dal = desc_k_sw128(smem_u32(sA) + ATILE);
      const int stages = (iters / 3) / SC;
      int it = 0;
      for (int st = 0; st < stages; ++st) {
        const int sidx = st % DEPTH;
        mbar_wait(&full7[sidx], (st / DEPTH) & 1);
        for (int q = 0; q < SC; ++q, ++it) {
          const int c = it % 4, tap = (it / 4) % 4;
          const uint32_t dd = d + tap * N;
          const uint64_t bh = db + ((c * BTILE) >> 4), bl = db + (((c + 4) * BTILE) >> 4);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, da + 2 * kk, bh + 2 * kk, idesc, (c | kk) != 0);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, da + 2 * kk, bl + 2 * kk, idesc, 1);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, dal + 2 * kk, bh + 2 * kk, idesc, 1);
        }
        mma_commit(&empty7[sidx]);
      }
    } else if (MODE == 0) {
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, da + 2 * kk, db + 2 * kk, idesc, (it | kk) != 0);
    } else if (MODE == 1) {
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ts(d, a_tm + kk * 8, db + 2 * kk, idesc, (it | kk) != 0);
    } else if (MODE == 8) {
      const uint32_t idesc2 = idesc_bf16_f32(128, 2 * N);
      const uint64_t dal = desc_k_sw128(smem_u32(sA) + ATILE);
      for (int it = 0; it < iters / 3; ++it) {
        const int c = it % 4;
        const uint64_t bhl = db + ((c * 2 * BTILE) >> 4);  // [hi | lo] contiguous, 2N rows
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, da + 2 * kk, bhl + 2 * kk, idesc2, (it | kk) != 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, dal + 2 * kk, bhl + 2 * kk, idesc, 1);
      }
    } else if (MODE >= 100) {
      // ring of DEPTH commit barriers, one commit per stage of SC chunks (12 MMAs each);
      // before committing stage i, wait for the commit of stage i - DEPTH (the kernel's
      // W-ring dependency without any loads)
      constexpr int DEPTH = (MODE / 10) % 10, SC = MODE % 10;  // MODE = 100/200/300 + ...
      const uint64_t dal = desc_k_sw128(smem_u32(sA) + ATILE);
      __shared__ uint64_t rb[8];
      for (int i = 0; i < DEPTH; ++i) mbar_init(&rb[i], 1);
      mbar_init(&rb[7], 1);
      fence_barrier_init();
      mbar_arrive(&rb[7]);  // phase 0 complete
      uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int stage = 0;
      for (int it = 0; it < iters / 3; ++it) {
        const int c = it % 4, tap = (it / 4) % 4;
        const uint32_t dd = d + tap * N;
        const uint64_t bh = db + ((c * BTILE) >> 4), bl = db + (((c + 4) * BTILE) >> 4);
        if (MODE >= 400 && it % SC == 0) {
          // wait on a barrier nobody's MMAs complete: initialised with count 1 and arrived
          // once by this thread, so every try_wait on phase 0 succeeds immediately
          if constexpr (MODE >= 500) {
            uint32_t ok = 0;
            while (!ok) {
              asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                           : "=r"(ok) : "r"(smem_u32(&rb[7])), "r"(0u) : "memory");
            }
          } else {
            while (!mbar_try_wait(&rb[7], 0)) {}
          }
        } else if (it % SC == 0 && stage >= DEPTH) {
          const int sidx = stage % DEPTH;
          if constexpr (MODE >= 300) {  // test_wait (non-blocking probe) in a spin loop
            uint32_t ok = 0;
            while (!ok) {
              asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                           : "=r"(ok) : "r"(smem_u32(&rb[sidx])), "r"(phase[sidx]) : "memory");
            }
          } else if constexpr (MODE >= 200) {  // try_wait without the suspend hint
            mbar_wait_spin(&rb[sidx], phase[sidx]);
          } else {
            while (!mbar_try_wait(&rb[sidx], phase[sidx])) {}
          }
          phase[sidx] ^= 1;
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, da + 2 * kk, bh + 2 * kk, idesc, (c | kk) != 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, da + 2 * kk, bl + 2 * kk, idesc, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, dal + 2 * kk, bh + 2 * kk, idesc, 1);
        if (it % SC == SC - 1) {
          if (MODE < 400) mma_commit(&rb[stage % DEPTH]);
          ++stage;
        }
      }
    } else if (MODE == 5 || MODE == 6) {
      // the RI kernel's stream: 3 MMAs x 4 kk per chunk, commit every 2 chunks (a W stage),
      // D buffer switch every 4 chunks (a tap); MODE 6 adds an mbarrier wait per stage
      const uint64_t dal = desc_k_sw128(smem_u32(sA) + ATILE);
      __shared__ uint64_t cb[4];
      if (true) {
        for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1);
        fence_barrier_init();
      }
      uint32_t phase[4] = {0, 0, 0, 0};
      int used[4] = {0, 0, 0, 0};
      for (int it = 0; it < iters / 3; ++it) {
        const int c = it % 4, tap = (it / 4) % 4;
        const uint32_t dd = d + tap * N;
        const uint64_t bh = db + ((c * BTILE) >> 4), bl = db + (((c + 4) * BTILE) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, da + 2 * kk, bh + 2 * kk, idesc, (c | kk) != 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, da + 2 * kk, bl + 2 * kk, idesc, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(dd, dal + 2 * kk, bh + 2 * kk, idesc, 1);
        if (c % 2 == 1) {
          const int sidx = (it / 2) % 2;
          if (MODE == 6 && used[sidx]) {  // wait the stage's previous commit (ring of 2)
            while (!mbar_try_wait(&cb[sidx], phase[sidx])) {}
            phase[sidx] ^= 1;
          }
          mma_commit(&cb[sidx]);
          used[sidx] = 1;
        }
      }
    } else if (MODE == 3 || MODE == 4) {
      // W_hi (MODE 3) or W_hi and W_lo (MODE 4) staged smem -> TMEM with tcgen05.cp per
      // K-step, consumed by TS MMAs in issue order; double-buffered TMEM A regions
      const uint64_t dal = desc_k_sw128(smem_u32(sA) + ATILE);
      for (int it = 0; it < iters / 3; ++it) {
        const int c = it % 4;
        const uint64_t bh = db + ((c * BTILE) >> 4), bl = db + (((c + 4) * BTILE) >> 4);
        const uint32_t ah = a_tm + (it & 1) * 64, al = ah + 32;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          tmem_cp_128x256b(ah + kk * 8, da + 2 * kk);
          if (MODE == 4) tmem_cp_128x256b(al + kk * 8, dal + 2 * kk);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ts(d, ah + kk * 8, bh + 2 * kk, idesc, (it | kk) != 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ts(d, ah + kk * 8, bl + 2 * kk, idesc, 1);
        if (MODE == 4) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16_ts(d, al + kk * 8, bh + 2 * kk, idesc, 1);
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, dal + 2 * kk, bh + 2 * kk, idesc, 1);
        }
      }
    } else {
      const uint64_t dal = desc_k_sw128(smem_u32(sA) + ATILE);
      for (int it = 0; it < iters / 3; ++it) {
        const int c = it % 4;
        const uint64_t bh = db + ((c * BTILE) >> 4), bl = db + (((c + 4) * BTILE) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, da + 2 * kk, bh + 2 * kk, idesc, (it | kk) != 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, da + 2 * kk, bl + 2 * kk, idesc, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, dal + 2 * kk, bh + 2 * kk, idesc, 1);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  long long t1 = clock64();
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(d + ((uint32_t)(warp * 32) << 16) + c0, v);
    tmem_wait_ld();
    for (int j = 0; j < 16 && c0 + j < N; ++j) out[(warp * 32 + (tid % 32)) * N + c0 + j] = v[j];
  }
  if (tid == 0) cycles[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

template <int N, int MODE>
void run(int grid = 1) {
  std::vector<__nv_bfloat16> A(128 * 64), B(N * 64);
  std::vector<float> Af(128 * 64), Bf(N * 64);
  srand(N + MODE);
  for (int i = 0; i < 128 * 64; ++i) {
    Af[i] = (float)(rand() % 5 - 2);
    A[i] = __float2bfloat16(Af[i]);
  }
  for (int i = 0; i < N * 64; ++i) {
    Bf[i] = (float)(rand() % 5 - 2);
    B[i] = __float2bfloat16(Bf[i]);
  }
  __nv_bfloat16 *dA, *dB;
  float* dout;
  long long* dcyc;
  CK(cudaMalloc(&dA, A.size() * 2));
  CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMalloc(&dout, 128 * N * 4));
  CK(cudaMalloc(&dcyc, 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  const int smem = 2 * 128 * 128 + (MODE >= 2 ? 8 : 1) * N * 128 + 2048;
  CK(cudaFuncSetAttribute(mma_bench<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters_check = MODE >= 2 ? 3 : 1;
  mma_bench<N, MODE><<<1, 128, smem>>>(iters_check, dA, dB, dout, dcyc);
  CK(cudaDeviceSynchronize());
  std::vector<float> out(128 * N);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  const float mult = MODE >= 2 ? 3.f : 1.f;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int k = 0; k < 64; ++k) ref += Af[m * 64 + k] * Bf[n * 64 + k];
      if (ref * mult != out[m * N + n]) ++bad;
    }
  const int iters = grid > 1 ? 30000 : 3000;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  mma_bench<N, MODE><<<grid, 128, smem>>>(iters, dA, dB, dout, dcyc);
  CK(cudaEventRecord(e1));
  CK(cudaDeviceSynchronize());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  long long cyc;
  CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
  const int mmas = MODE >= 2 ? (iters / 3) * 12 : iters * 4;
  const double per = (double)cyc / mmas;
  printf("{\"mode\":%d,\"test\":\"%s\",\"M\":128,\"N\":%d,\"correct\":%s,\"mismatches\":%d,\"cycles_per_mma_k16\":%.2f,"
         "\"macs_per_cycle\":%.1f,\"math_cycles\":%.1f,\"grid\":%d,\"ms\":%.4f,\"eff_mhz\":%.0f}\n",
         MODE, MODE == 0 ? "mma_ss" : MODE == 1 ? "mma_ts" : MODE == 2 ? "pattern_bf16x3_ss" : MODE == 3 ? "pattern_bf16x3_whi_tmem" : MODE == 4 ? "pattern_bf16x3_w_tmem" : MODE == 5 ? "kernel_stream_commits" : MODE == 6 ? "kernel_stream_commits_waits" : "commit_ring_depth_x10_plus_chunks_per_stage", N, bad == 0 ? "true" : "false", bad, per,
         128.0 * N * 16 / per, 128.0 * N * 16 / 4096, grid, ms, cyc / (ms * 1e3));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dout);
  cudaFree(dcyc);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // full-chip runs: clock under sustained tensor load
    const int g = atoi(argv[1]);
    run<96, 0>(1);
    run<96, 0>(g);
    run<96, 2>(g);
    run<96, 0>(g);
    return 0;
  }
  run<96, 2>();
  run<96, 8>();
  run<112, 2>();
  run<112, 8>();
  run<64, 2>();
  run<64, 8>();
  return 0;
}
