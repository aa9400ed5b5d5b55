// ri_tc.cu -- tcgen05 tensor-core fused RI scatter convolution, K = 3, W = 16 (sm_100a).
//
// Same math as ri_simt.cu (convention P1), with the channel contraction on
// the 5th-generation tensor cores:
//   Z_t[co, px] = sum_ci W_{b,t}[co, ci] * X[ci, px]      tcgen05.mma kind::f16, M=128 co,
//                                                         N=64 px (one 4-row band), FP32 in TMEM
//   Y_{b,r}(p) += Z_t(p + delta_{r,t})                    CUDA-core epilogue, reuse over r
// precision "bf16"  : one product, bf16 operands;
// precision "bf16x3": operands split hi+lo (bf16 each), hi*hi + hi*lo + lo*hi, FP32-class.
//
// Layout / dataflow per persistent CTA (1 CTA per SM, 10 warps):
//   warp 0  producer   : 1-D bulk copies (TMA engine) of pre-packed SW128 tiles:
//                        X band [64 px x 64 ci] per ci-chunk (double-buffered per band),
//                        W tap tiles [128 co x 64 ci] through a ring of W_STAGES stages.
//   warp 1  MMA issuer : one elected thread; per (base, band, tap) accumulates K into one
//                        of two 64-column TMEM buffers, commits to mbarriers.
//   warps 2-9 epilogue : TMEM lane = output channel (co); every thread owns full 16-px image
//                        rows, so the spatial scatter is register indexing.  Two warps per
//                        lane quadrant split the band's 4 output rows (2 each); 128 fp32 Y
//                        registers per thread (2 rows x 4 rotations x 16 px).
// Bands lag by one row: band k computes input rows [4k, 4k+4) and completes output rows
// [4k-1, 4k+3); the two input rows above the band (4k-2, 4k-1) are kept in TMEM
// ("kept slots", 2 rows x 9 taps) by the h=0 epilogue warps, so no row is ever
// recomputed.  TMEM: D buffers cols [0,128), kept slots [128, 416).
// Pooling / argmax / bias epilogue identical to the SIMT kernel; 128-bit stores.
#include <cuda_bf16.h>

#include "k3_tables.cuh"
#include "rc_internal.cuh"
#include "tc_ptx.cuh"

namespace rc {
namespace {

using namespace tc;

constexpr int TW = 16;        // image width handled by this kernel
constexpr int BAND_ROWS = 4;  // input rows per band
constexpr int BAND_PX = 64;   // = N of the MMA
constexpr int KC = 64;        // ci per chunk (one 128-byte swizzle row of bf16)
constexpr int XTILE = BAND_PX * KC * 2;  // 8 KB
constexpr int WTILE = 128 * KC * 2;      // 16 KB
constexpr int NUM_EPI = 8;
constexpr int THREADS = 32 * (2 + NUM_EPI);
constexpr uint32_t KEPT0 = 128;

struct TcParams {
  const uint8_t* xh;  // packed X tiles [n][band][chunk] (hi), 8 KB each
  const uint8_t* xl;  // lo plane (3-pass) or null
  const uint8_t* wh;  // packed W tiles [b][ct][t][chunk] (hi), 16 KB each
  const uint8_t* wl;  // lo plane
  const float* bias;
  float* y;
  uint8_t* am;
  int N, H, Cout, NB, NBK, NC, NCT, pool, gf, RO, passes, w_stages, items;
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void store16(float* dst, const float (&v)[16]) {
  float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int k = 0; k < 4; ++k) d4[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
}
__device__ __forceinline__ void store16u8(uint8_t* dst, const uint8_t (&a)[16]) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    w[k] = a[4 * k] | (a[4 * k + 1] << 8) | (a[4 * k + 2] << 16) | ((uint32_t)a[4 * k + 3] << 24);
  *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
}

// max-fold of rotations [R0, R0+G) of this base into Yr[R0] (+ argmax, ties -> smallest
// index); everything in place to keep the epilogue's register footprint at Y + 16.
template <int R0, int G>
__device__ __forceinline__ void fold_max(float (&Yr)[4][16], uint32_t (&arg)[4], int kk0) {
#pragma unroll
  for (int r = R0 + 1; r < R0 + G; ++r)
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (Yr[r][j] > Yr[R0][j]) {
        Yr[R0][j] = Yr[r][j];
        arg[j / 4] = (arg[j / 4] & ~(0xFFu << (8 * (j % 4)))) | ((uint32_t)(kk0 + r - R0) << (8 * (j % 4)));
      }
}
__device__ __forceinline__ void store_row(const TcParams& p, size_t off, float (&v)[16], const uint32_t (&arg)[4],
                                          float bz, bool fin) {
  if (fin) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += bz;
  }
  store16(p.y + off, v);
  if (p.am) *reinterpret_cast<uint4*>(p.am + off) = make_uint4(arg[0], arg[1], arg[2], arg[3]);
}

// pool + bias + store one output row (16 px) of base b; same semantics as ri_simt.cu.
// Fold groups gf in {1, 2, 4} stay inside a base; gf % 4 == 0 spans bases through a
// partial (value, argmax) kept in the output row itself (same thread, program order).
__device__ __forceinline__ void finalize_row(const TcParams& p, float (&Yr)[4][16], int n, int co, int b,
                                             int row) {
  const size_t plane = (size_t)p.H * TW;
  const size_t ybase = ((size_t)n * p.Cout + co) * p.RO * plane + (size_t)row * TW;
  const float bz = p.bias ? p.bias[co] : 0.f;
  if (p.pool == RC_POOL_NONE) {
    const uint32_t z[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 4; ++r) store_row(p, ybase + (size_t)(b * 4 + r) * plane, Yr[r], z, bz, true);
    return;
  }
  if (p.pool == RC_POOL_AVG) {
    if (b > 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) Yr[0][j] = p.y[ybase + j] + Yr[0][j];
    }
#pragma unroll
    for (int r = 1; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 16; ++j) Yr[0][j] += Yr[r][j];
    if (b == p.NB - 1) {
      const float R = (float)(p.NB * 4);
#pragma unroll
      for (int j = 0; j < 16; ++j) Yr[0][j] = Yr[0][j] / R + bz;
    }
    store16(p.y + ybase, Yr[0]);
    return;
  }
  const int gf = p.gf;
  uint32_t arg[4] = {0, 0, 0, 0};
  if (gf == 1) {
#pragma unroll
    for (int r = 0; r < 4; ++r) store_row(p, ybase + (size_t)(b * 4 + r) * plane, Yr[r], arg, bz, true);
  } else if (gf == 2) {
    fold_max<0, 2>(Yr, arg, 0);
    store_row(p, ybase + (size_t)(b * 2) * plane, Yr[0], arg, bz, true);
    arg[0] = arg[1] = arg[2] = arg[3] = 0;
    fold_max<2, 2>(Yr, arg, 0);
    store_row(p, ybase + (size_t)(b * 2 + 1) * plane, Yr[2], arg, bz, true);
  } else {  // gf % 4 == 0
    const int o0 = b * 4, slot = o0 / gf, kk0 = o0 - slot * gf;
    const size_t off = ybase + (size_t)slot * plane;
    arg[0] = arg[1] = arg[2] = arg[3] = (uint32_t)kk0 * 0x01010101u;  // candidate r=0 is index kk0
    fold_max<0, 4>(Yr, arg, kk0);
    if (kk0 > 0) {  // continue the slot begun in an earlier base
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float prev = p.y[off + j];
        const uint32_t pa = p.am ? p.am[off + j] : 0u;
        if (!(Yr[0][j] > prev)) {  // earlier (smaller) index wins ties
          Yr[0][j] = prev;
          arg[j / 4] = (arg[j / 4] & ~(0xFFu << (8 * (j % 4)))) | (pa << (8 * (j % 4)));
        }
      }
    }
    store_row(p, off, Yr[0], arg, bz, kk0 + 4 == gf);
  }
}

// scatter one Z row of tap t into this warp half's 2 output rows (all indices
// compile-time; t is dispatched once per call):
//   row holds input row REL relative to the band start 4k;
//   Y[l] is output row (BASE + l) relative to 4k.  Input row q feeds output q - di.
template <int CONV, int REL, int BASE, int TT>
__device__ __forceinline__ void scatter_row_t(float (&Y)[2][4][16], const float (&row)[16]) {
  constexpr K3Tables TB = make_k3(CONV);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int l = REL - TB.di[r][TT] - BASE;
    if (l < 0 || l > 1) continue;
    const int dj = TB.dj[r][TT];
#pragma unroll
    for (int x = 0; x < 16; ++x) {
      const int src = x + dj;
      if (src < 0 || src > 15) continue;
      if (l == 0)
        Y[0][r][x] += row[src];
      else
        Y[1][r][x] += row[src];
    }
  }
}
template <int CONV, int REL, int BASE>
__device__ __forceinline__ void scatter_row(float (&Y)[2][4][16], const float (&row)[16], int t) {
  switch (t) {
    case 0: scatter_row_t<CONV, REL, BASE, 0>(Y, row); break;
    case 1: scatter_row_t<CONV, REL, BASE, 1>(Y, row); break;
    case 2: scatter_row_t<CONV, REL, BASE, 2>(Y, row); break;
    case 3: scatter_row_t<CONV, REL, BASE, 3>(Y, row); break;
    case 4: scatter_row_t<CONV, REL, BASE, 4>(Y, row); break;
    case 5: scatter_row_t<CONV, REL, BASE, 5>(Y, row); break;
    case 6: scatter_row_t<CONV, REL, BASE, 6>(Y, row); break;
    case 7: scatter_row_t<CONV, REL, BASE, 7>(Y, row); break;
    default: scatter_row_t<CONV, REL, BASE, 8>(Y, row); break;
  }
}
template <int CONV, int REL, int BASE>
__device__ __forceinline__ void load_scatter(float (&Y)[2][4][16], uint32_t taddr, int t) {
  float row[16];
  tmem_ld16(taddr, row);
  tmem_wait_ld();
  scatter_row<CONV, REL, BASE>(Y, row, t);
}
__device__ __forceinline__ void copy_row(uint32_t src, uint32_t dst) {
  float row[16];
  tmem_ld16(src, row);
  tmem_wait_ld();
  tmem_st16(dst, row);
}

// Epilogue of one warp half over all work items.  H = 0: output rows 4k-1, 4k (needs
// input rows -2..1: kept slot + new rows 0,1; also copies new rows 2,3 into the kept
// slot for band k+1).  H = 1: output rows 4k+1, 4k+2 (needs new rows 0..3).
// Z rows are pulled from TMEM one at a time (Y 128 + 16 staging registers).
template <int CONV, int H>
__device__ void epilogue(const TcParams& p, uint32_t tmem, uint64_t* d_full, uint64_t* d_empty) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q = warp % 4;
  const int co_l = q * 32 + lane;
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  constexpr int BASE = H == 0 ? -1 : 1;
  uint32_t gd = 0;
  float Y[2][4][16];
  for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
    const int ct = item / p.N, n = item % p.N;
    const int co = ct * 128 + co_l;
    for (int b = 0; b < p.NB; ++b)
      for (int k = 0; k <= p.NBK; ++k) {  // k == NBK: drain band (no MMA, zero rows)
        const bool have_new = k < p.NBK;
        if (H == 1 && !have_new) continue;  // its rows 4*NBK+1.. are beyond H
#pragma unroll
        for (int l = 0; l < 2; ++l)
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int x = 0; x < 16; ++x) Y[l][r][x] = 0.f;
#pragma unroll 1
        for (int t = 0; t < 9; ++t) {
          const int db = gd & 1;
          const uint32_t dcol = tmem + lane_off + db * BAND_PX;
          const uint32_t kcol = tmem + lane_off + KEPT0 + t * 32;
          if (H == 0) {
            if (k > 0) {  // input rows -2, -1 from the kept slot (zero above the image)
              load_scatter<CONV, -2, BASE>(Y, kcol, t);
              load_scatter<CONV, -1, BASE>(Y, kcol + 16, t);
            }
            if (have_new) {
              mbar_wait(&d_full[db], (gd >> 1) & 1);
              tc_fence_after();
              load_scatter<CONV, 0, BASE>(Y, dcol, t);
              load_scatter<CONV, 1, BASE>(Y, dcol + 16, t);
              copy_row(dcol + 32, kcol);  // rows 2, 3 -> kept slot (rows -2, -1 of band k+1)
              copy_row(dcol + 48, kcol + 16);
              tmem_wait_st();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&d_empty[db]);
              ++gd;
            }
          } else {
            mbar_wait(&d_full[db], (gd >> 1) & 1);
            tc_fence_after();
            load_scatter<CONV, 0, BASE>(Y, dcol, t);
            load_scatter<CONV, 1, BASE>(Y, dcol + 16, t);
            load_scatter<CONV, 2, BASE>(Y, dcol + 32, t);
            float row[16];
            tmem_ld16(dcol + 48, row);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&d_empty[db]);
            scatter_row<CONV, 3, BASE>(Y, row, t);
            ++gd;
          }
        }
        if (n < p.N && co < p.Cout) {
#pragma unroll
          for (int l = 0; l < 2; ++l) {
            const int row = BAND_ROWS * k + BASE + l;
            if (row >= 0 && row < p.H) finalize_row(p, Y[l], n, co, b, row);
          }
        }
      }
  }
}

template <int CONV>
__global__ void __launch_bounds__(THREADS, 1) ri_tc_kernel(const __grid_constant__ TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB alignment for the SW128 atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int parts = p.passes == 3 ? 2 : 1;
  const int xbuf_bytes = parts * p.NC * XTILE;
  uint8_t* xs = smem;                      // 2 X band buffers
  uint8_t* ws = smem + 2 * xbuf_bytes;     // W ring
  __shared__ uint64_t w_full[8], w_empty[8], x_full[2], x_empty[2], d_full[2], d_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int S = p.w_stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], NUM_EPI);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t gw = 0, xc = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        const int ct = item / p.N, n = item % p.N;
        for (int b = 0; b < p.NB; ++b)
          for (int k = 0; k < p.NBK; ++k) {
            const int xb = xc & 1;
            if (xc >= 2) mbar_wait(&x_empty[xb], ((xc >> 1) & 1) ^ 1);
            mbar_arrive_expect_tx(&x_full[xb], xbuf_bytes);
            for (int part = 0; part < parts; ++part)
              for (int c = 0; c < p.NC; ++c) {
                const size_t tile = ((size_t)n * p.NBK + k) * p.NC + c;
                bulk_g2s(xs + xb * xbuf_bytes + (part * p.NC + c) * XTILE,
                         (part ? p.xl : p.xh) + tile * XTILE, XTILE, &x_full[xb]);
              }
            ++xc;
            for (int t = 0; t < 9; ++t)
              for (int c = 0; c < p.NC; ++c)
                for (int part = 0; part < parts; ++part) {
                  const int s = gw % S;
                  if (gw >= (uint32_t)S) mbar_wait(&w_empty[s], ((gw / S) & 1) ^ 1);
                  mbar_arrive_expect_tx(&w_full[s], WTILE);
                  const size_t tile = (((size_t)b * p.NCT + ct) * 9 + t) * p.NC + c;
                  bulk_g2s(ws + s * WTILE, (part ? p.wl : p.wh) + tile * WTILE, WTILE, &w_full[s]);
                  ++gw;
                }
          }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(128, BAND_PX);
      uint32_t gw = 0, xc = 0, gd = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        for (int b = 0; b < p.NB; ++b)
          for (int k = 0; k < p.NBK; ++k) {
            const int xb = xc & 1;
            mbar_wait(&x_full[xb], (xc >> 1) & 1);
            tc_fence_after();
            const uint32_t xaddr = smem_u32(xs + xb * xbuf_bytes);
            for (int t = 0; t < 9; ++t) {
              const int db = gd & 1;
              if (gd >= 2) mbar_wait(&d_empty[db], ((gd >> 1) & 1) ^ 1);
              tc_fence_after();
              const uint32_t d = tmem + db * BAND_PX;
              for (int c = 0; c < p.NC; ++c) {
                const uint64_t bh = desc_k_sw128(xaddr + c * XTILE);
                if (parts == 1) {
                  const int s = gw % S;
                  mbar_wait(&w_full[s], (gw / S) & 1);
                  tc_fence_after();
                  const uint64_t a = desc_k_sw128(smem_u32(ws + s * WTILE));
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, a + 2 * kk, bh + 2 * kk, idesc, (c | kk) != 0);
                  mma_commit(&w_empty[s]);
                  ++gw;
                } else {
                  const uint64_t bl = desc_k_sw128(xaddr + (p.NC + c) * XTILE);
                  const int sh = gw % S, sl = (gw + 1) % S;
                  mbar_wait(&w_full[sh], (gw / S) & 1);
                  mbar_wait(&w_full[sl], ((gw + 1) / S) & 1);
                  tc_fence_after();
                  const uint64_t ah = desc_k_sw128(smem_u32(ws + sh * WTILE));
                  const uint64_t al = desc_k_sw128(smem_u32(ws + sl * WTILE));
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, ah + 2 * kk, bh + 2 * kk, idesc, (c | kk) != 0);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, ah + 2 * kk, bl + 2 * kk, idesc, 1);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, al + 2 * kk, bh + 2 * kk, idesc, 1);
                  mma_commit(&w_empty[sh]);
                  mma_commit(&w_empty[sl]);
                  gw += 2;
                }
              }
              mma_commit(&d_full[db]);
              ++gd;
            }
            mma_commit(&x_empty[xb]);
            ++xc;
          }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    if ((warp - 2) / 4 == 0)
      epilogue<CONV, 0>(p, tmem, d_full, d_empty);
    else
      epilogue<CONV, 1>(p, tmem, d_full, d_empty);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ---- packing kernels ----------------------------------------------------------------
__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// X fp32 NCHW (W = 16) -> SW128 bf16 tiles [n][band][chunk][64 px][64 ci] (hi, lo planes)
__global__ void x_pack_kernel(const float* __restrict__ x, uint8_t* __restrict__ xh,
                              uint8_t* __restrict__ xl, int Cin, int H, int NBK, int NC) {
  __shared__ float tile[KC][BAND_PX + 1];
  const int c = blockIdx.x, k = blockIdx.y, n = blockIdx.z;
  for (int i = threadIdx.x; i < KC * BAND_PX; i += blockDim.x) {
    const int cl = i / BAND_PX, px = i % BAND_PX;
    const int ci = c * KC + cl, row = k * BAND_ROWS + px / TW, col = px % TW;
    tile[cl][px] = (ci < Cin && row < H) ? x[(((size_t)n * Cin + ci) * H + row) * TW + col] : 0.f;
  }
  __syncthreads();
  const size_t tidx = ((size_t)n * NBK + k) * NC + c;
  uint8_t* oh = xh + tidx * XTILE;
  uint8_t* ol = xl ? xl + tidx * XTILE : nullptr;
  for (int i = threadIdx.x; i < BAND_PX * (KC / 8); i += blockDim.x) {
    const int px = i / (KC / 8), g = i % (KC / 8);
    __align__(16) __nv_bfloat16 h8[8], l8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) split_bf16(tile[g * 8 + j][px], h8[j], l8[j]);
    const uint32_t off = sw128_offset(px, g * 8);
    *reinterpret_cast<uint4*>(oh + off) = *reinterpret_cast<const uint4*>(h8);
    if (ol) *reinterpret_cast<uint4*>(ol + off) = *reinterpret_cast<const uint4*>(l8);
  }
}

// base kernels fp32 [B][Cout][Cin][9] -> SW128 bf16 tiles [b][ct][t][chunk][128 co][64 ci]
__global__ void w_pack_kernel(const float* __restrict__ bases, uint8_t* __restrict__ wh,
                              uint8_t* __restrict__ wl, int NB, int Cout, int Cin, int NCT, int NC) {
  const long long total = (long long)NB * NCT * 9 * NC * 128 * (KC / 8);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(i % (KC / 8));
    const int col = (int)((i / (KC / 8)) % 128);
    const long long tile = i / ((KC / 8) * 128);  // ((b*NCT + ct)*9 + t)*NC + c
    const int c = (int)(tile % NC);
    const int t = (int)((tile / NC) % 9);
    const int ct = (int)((tile / ((long long)NC * 9)) % NCT);
    const int b = (int)(tile / ((long long)NC * 9 * NCT));
    const int co = ct * 128 + col;
    __align__(16) __nv_bfloat16 h8[8], l8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int ci = c * KC + g * 8 + j;
      const float v = (co < Cout && ci < Cin) ? bases[(((size_t)b * Cout + co) * Cin + ci) * 9 + t] : 0.f;
      split_bf16(v, h8[j], l8[j]);
    }
    const size_t off = (size_t)tile * WTILE + sw128_offset(col, g * 8);
    *reinterpret_cast<uint4*>(wh + off) = *reinterpret_cast<const uint4*>(h8);
    *reinterpret_cast<uint4*>(wl + off) = *reinterpret_cast<const uint4*>(l8);
  }
}

struct TcGeom {
  int NBK, NC, NCT;
  size_t x_plane, w_plane;
};
TcGeom geom(const rc_desc& d) {
  TcGeom g;
  g.NBK = (d.h + BAND_ROWS - 1) / BAND_ROWS;
  g.NC = (d.c_in + KC - 1) / KC;
  g.NCT = (d.c_out + 127) / 128;
  g.x_plane = (size_t)d.n * g.NBK * g.NC * XTILE;
  g.w_plane = (size_t)num_bases(d) * g.NCT * 9 * g.NC * WTILE;
  return g;
}

}  // namespace

bool tc_supported(const rc_desc& d) {
  const int gf = pool_fold(d);
  const bool fold_ok = d.pool == RC_POOL_NONE || d.pool == RC_POOL_AVG || gf == 1 || gf == 2 || gf % 4 == 0;
  return d.k == 3 && d.w == TW && d.group != RC_GROUP_SINGLE && d.c_in <= 512 && fold_ok &&
         (d.precision == RC_PREC_BF16 || d.precision == RC_PREC_BF16X3 || d.precision == RC_PREC_AUTO);
}
size_t tc_bank_bytes(const rc_desc& d) {
  if (!(d.k == 3 && d.group != RC_GROUP_SINGLE)) return 0;
  return 2 * geom(d).w_plane;
}
size_t tc_workspace_bytes(const rc_desc& d) {
  if (!tc_supported(d)) return 0;
  return 2 * geom(d).x_plane;
}

int launch_tc_wpack(const rc_desc& d, const float* bases, uint8_t* tc_section, cudaStream_t s) {
  const TcGeom g = geom(d);
  const long long total = (long long)num_bases(d) * g.NCT * 9 * g.NC * 128 * (KC / 8);
  long long grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  w_pack_kernel<<<(int)grid, 256, 0, s>>>(bases, tc_section, tc_section + g.w_plane, num_bases(d), d.c_out,
                                         d.c_in, g.NCT, g.NC);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

int launch_tc(const rc_desc& d, const float* x, const void* bank, const float* bias, float* y, uint8_t* am,
              void* ws, size_t ws_bytes, cudaStream_t s, bool dry_run, const char** name) {
  if (!tc_supported(d)) return RC_ERR_UNSUPPORTED;
  if (name) *name = d.precision == RC_PREC_BF16 ? "tc_k3w16_bf16" : "tc_k3w16_bf16x3";
  if (dry_run || d.n == 0) return RC_OK;
  const TcGeom g = geom(d);
  if (ws_bytes < tc_workspace_bytes(d) || ws == nullptr)
    return fail(RC_ERR_WORKSPACE, "ri_conv: workspace too small for the tensor-core path");
  const int passes = d.precision == RC_PREC_BF16 ? 1 : 3;
  uint8_t* xh = static_cast<uint8_t*>(ws);
  uint8_t* xl = passes == 3 ? xh + g.x_plane : nullptr;
  x_pack_kernel<<<dim3(g.NC, g.NBK, d.n), 256, 0, s>>>(x, xh, xl, d.c_in, d.h, g.NBK, g.NC);
  RC_CUDA(cudaGetLastError());
  const BankLayout L = bank_layout(d);
  const uint8_t* tcb = static_cast<const uint8_t*>(bank) + L.tc_off;
  TcParams p;
  p.xh = xh;
  p.xl = xl;
  p.wh = tcb;
  p.wl = tcb + g.w_plane;
  p.bias = bias;
  p.y = y;
  p.am = (d.pool == RC_POOL_MAX || d.pool == RC_POOL_SUBGROUP) ? am : nullptr;
  p.N = d.n;
  p.H = d.h;
  p.Cout = d.c_out;
  p.NB = num_bases(d);
  p.NBK = g.NBK;
  p.NC = g.NC;
  p.NCT = g.NCT;
  p.pool = d.pool;
  p.gf = pool_fold(d);
  p.RO = out_orientations(d);
  p.passes = passes;
  const int parts = passes == 3 ? 2 : 1;
  const size_t xbytes = 2 * (size_t)parts * g.NC * XTILE;
  int stages = (int)((220 * 1024 - xbytes) / WTILE);
  if (stages > 8) stages = 8;
  if (stages < 2 * parts) return fail(RC_ERR_UNSUPPORTED, "ri_conv: Cin too large for the tensor-core path");
  p.w_stages = stages;
  p.items = g.NCT * d.n;
  const size_t smem = xbytes + (size_t)stages * WTILE + 1024;
  int dev, sms;
  RC_CUDA(cudaGetDevice(&dev));
  RC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = p.items < sms ? p.items : sms;
  auto fn = d.convention == RC_CONV_RAW ? ri_tc_kernel<1> : ri_tc_kernel<0>;
  RC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<grid, THREADS, smem, s>>>(p);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

}  // namespace rc
