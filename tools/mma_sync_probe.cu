// mma_sync_probe.cu -- what does the synchronisation around a tcgen05.mma stream cost?
//
// One CTA, the RI kernel's bf16x3 inner loop (12 MMAs per 64-ci chunk: Ah*Bh, Ah*Bl, Al*Bh,
// M = 128, K = 16 each), operands resident in shared memory (no loads), N configurable.
// The MMA warp (warp 1) walks `chunks` chunks; the modes add the kernel's synchronisation:
//   0  no commit, no wait                                  (the SS issue rate)
//   1  commit to a ring barrier every SC chunks, no waits
//   2  1 + the MMA warp waits the commit of DEPTH stages back (single-warp ring)
//   3  1 + the MMA warp waits a plain barrier (always complete) every stage
//   4  two-warp ring: producer warp 0 waits the stage's commit DEPTH back and arrives the
//      stage's full barrier; the MMA warp waits full (the kernel's W ring, no loads)
//   5  4 + D ring: every TAP chunks the MMA warp commits d_full[db] and, before reusing a
//      D buffer, waits d_empty[db]; 16 epilogue warps wait d_full and arrive d_empty
// Output: one JSON line per (mode, N, SC, DEPTH): cycles per MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_08888_b200/csrc
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "tc_ptx.cuh"

using namespace rc::tc;

constexpr int THREADS = 640;  // 20 warps like the RI kernel
constexpr int TAP = 4;        // chunks per tap (Cin = 256)
constexpr int MAXDB = 4;

template <int N, int MODE, int SC, int DEPTH>
__global__ void __launch_bounds__(THREADS, 1) probe(int chunks, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int ATILE = 128 * 128, BTILE = N * 128;
  constexpr int NDB = 512 / N < MAXDB ? 512 / N : MAXDB;
  __shared__ uint64_t full[8], empty[8], dfull[MAXDB], dempty[MAXDB], triv, done, done2;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < (2 * ATILE + 2 * BTILE) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < NDB; ++i) {
      mbar_init(&dfull[i], 1);
      mbar_init(&dempty[i], 16);
    }
    mbar_init(&triv, 1);
    mbar_init(&done, 1);
    mbar_init(&done2, 1);
    fence_barrier_init();
    mbar_arrive(&triv);  // phase 0 complete forever
  }
  if (warp == 1) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const int stages = chunks / SC;
  const long long t0 = clock64();
  if (warp == 0 && MODE >= 4) {
    for (int st = 0; st < stages; ++st) {
      const int s = st % DEPTH;
      if (st >= DEPTH) mbar_wait(&empty[s], ((st / DEPTH) - 1) & 1);
      if (elect_one()) mbar_arrive(&full[s]);
      __syncwarp();
    }
  } else if (warp == 1 || (MODE == 6 && warp == 2)) {
    // MODE 6: warps 1 and 2 both issue, alternating taps (each commits its own MMAs)
    const int me = warp - 1, nissuers = MODE == 6 ? 2 : 1;
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t ah = desc_k_sw128(smem_u32(smem)), al = desc_k_sw128(smem_u32(smem + ATILE));
    const uint64_t bh = desc_k_sw128(smem_u32(smem + 2 * ATILE)), bl = desc_k_sw128(smem_u32(smem + 2 * ATILE + BTILE));
    int db = 0, taps = 0;
    uint32_t dph = 0;
    for (int st = 0; st < stages; ++st) {
      const int s = st % DEPTH;
      if (((st * SC) / TAP) % nissuers != me) {  // another issuer's tap: keep the D ring index
        if (MODE >= 5)
          for (int q = 0; q < SC; ++q)
            if ((st * SC + q) % TAP == TAP - 1) {
              ++taps;
              if (++db == NDB) {
                db = 0;
                dph ^= 1;
              }
            }
        continue;
      }
      if (MODE == 2 && st >= DEPTH) mbar_wait(&empty[s], ((st / DEPTH) - 1) & 1);
      if (MODE == 3) mbar_wait(&triv, 0);
      if (MODE >= 4) mbar_wait(&full[s], (st / DEPTH) & 1);
      tc_fence_after();
      for (int q = 0; q < SC; ++q) {
        const int c = st * SC + q;
        if (MODE >= 5 && c % TAP == 0) {  // new tap: a free D buffer
          if (taps >= NDB) mbar_wait(&dempty[db], dph ^ 1);
          tc_fence_after();
        }
        const uint32_t d = tm + db * N;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, ah + 2 * kk, bh + 2 * kk, idesc, (c % TAP | kk) != 0);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, ah + 2 * kk, bl + 2 * kk, idesc, 1);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, al + 2 * kk, bh + 2 * kk, idesc, 1);
          if (MODE >= 5 && c % TAP == TAP - 1) mma_commit(&dfull[db]);
        }
        __syncwarp();
        if (MODE >= 5 && c % TAP == TAP - 1) {
          ++taps;
          if (++db == NDB) {
            db = 0;
            dph ^= 1;
          }
        }
      }
      if (MODE >= 1) {
        if (elect_one()) mma_commit(&empty[s]);
        __syncwarp();
      }
    }
    if (me == 0) {
      if (MODE == 6) mbar_wait(&done2, 0);  // the other issuer's MMAs are complete too
      if (elect_one()) mma_commit(&done);
    } else if (elect_one()) {
      mma_commit(&done2);
    }
    __syncwarp();
  } else if (warp >= 4 && MODE >= 5) {
    const int ntaps = chunks / TAP;
    int db = 0;
    uint32_t dph = 0;
    for (int t = 0; t < ntaps; ++t) {
      mbar_wait(&dfull[db], dph);
      tc_fence_after();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&dempty[db]);
      if (++db == NDB) {
        db = 0;
        dph ^= 1;
      }
    }
  }
  if (warp == 1) {
    mbar_wait(&done, 0);
    if ((tid & 31) == 0) cycles[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tm);
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

template <int N, int MODE, int SC, int DEPTH>
void run() {
  long long* dc;
  CK(cudaMalloc(&dc, 8));
  const int smem = 2 * 128 * 128 + 2 * N * 128 + 2048;
  CK(cudaFuncSetAttribute(probe<N, MODE, SC, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int chunks = 4 * 4 * 200;  // multiple of TAP and SC
  probe<N, MODE, SC, DEPTH><<<1, THREADS, smem>>>(chunks, dc);  // warm-up
  CK(cudaDeviceSynchronize());
  probe<N, MODE, SC, DEPTH><<<1, THREADS, smem>>>(chunks, dc);
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  const double per = (double)cyc / (chunks * 12.0);
  printf("{\"mode\":%d,\"N\":%d,\"chunks_per_stage\":%d,\"depth\":%d,\"cycles_per_mma\":%.2f,\"ss_floor\":%.1f}\n", MODE, N,
         SC, DEPTH, per, 32.0 + N / 4.0 > N / 2.0 ? 32.0 + N / 4.0 : N / 2.0);
  cudaFree(dc);
}

template <int N>
void sweep() {
  run<N, 0, 2, 2>();
  run<N, 1, 2, 2>();
  run<N, 1, 4, 2>();
  run<N, 2, 2, 2>();
  run<N, 2, 2, 4>();
  run<N, 2, 4, 4>();
  run<N, 3, 2, 2>();
  run<N, 4, 2, 2>();
  run<N, 4, 2, 4>();
  run<N, 4, 4, 4>();
  run<N, 4, 1, 4>();
  run<N, 5, 2, 2>();
  run<N, 5, 2, 4>();
  run<N, 5, 4, 4>();
  run<N, 6, 2, 2>();
  run<N, 6, 2, 4>();
  run<N, 6, 4, 4>();
  run<N, 6, 1, 4>();
}

// TMEM -> register throughput: W warps (4 per lane quadrant) each load 16 columns per
// tcgen05.ld (x16) -- INFLIGHT loads before one wait::ld -- over the 512 columns, ITERS times.
template <int INFLIGHT>
__global__ void __launch_bounds__(THREADS, 1) tmem_ld_probe(int iters, int nwarps, long long* cycles, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t lane_base = tbase + ((uint32_t)((warp % 4) * 32) << 16);
  float acc = 0.f;
  const long long t0 = clock64();
  if (warp < nwarps) {
    for (int it = 0; it < iters; ++it)
      for (int c = 0; c < 512; c += 16 * INFLIGHT) {
        float v[INFLIGHT][16];
#pragma unroll
        for (int j = 0; j < INFLIGHT; ++j) tmem_ld16(lane_base + c + 16 * j, v[j]);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < INFLIGHT; ++j)
#pragma unroll
          for (int k = 0; k < 16; ++k) acc += v[j][k];
      }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int INFLIGHT>
void run_ld(int nwarps) {
  long long* dc;
  float* sink;
  CK(cudaMalloc(&dc, 8));
  CK(cudaMalloc(&sink, THREADS * 4));
  const int iters = 200;
  tmem_ld_probe<INFLIGHT><<<1, THREADS>>>(iters, nwarps, dc, sink);
  CK(cudaDeviceSynchronize());
  tmem_ld_probe<INFLIGHT><<<1, THREADS>>>(iters, nwarps, dc, sink);
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  const double bytes = (double)iters * 512 * 32 * 4 * nwarps;
  printf("{\"test\":\"tmem_ld_x16\",\"warps\":%d,\"inflight\":%d,\"bytes_per_cycle\":%.1f,\"cycles_per_ld_per_warp\":%.1f}\n",
         nwarps, INFLIGHT, bytes / cyc, cyc / ((double)iters * 512 / 16));
  cudaFree(dc);
  cudaFree(sink);
}

int main() {
  run_ld<1>(4);
  run_ld<1>(16);
  run_ld<2>(16);
  run_ld<4>(16);
  run_ld<4>(4);
  sweep<96>();
  sweep<128>();
  sweep<192>();
  sweep<256>();
  return 0;
}
