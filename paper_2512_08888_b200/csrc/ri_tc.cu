// ri_tc.cu -- tcgen05 tensor-core fused RI scatter convolution, K = 3 (sm_100a).
//
// Same math as ri_simt.cu (convention P1), with the channel contraction on
// the 5th-generation tensor cores:
//   Z_t[co, px] = sum_ci W_{b,t}[co, ci] * X[ci, px]      tcgen05.mma kind::f16, M = 128 co,
//                                                         N = band px, FP32 accumulators in TMEM
//   Y_{b,r}(p) += Z_t(p + delta_{r,t})                    CUDA-core epilogue, reused by all 4 r
// precision "bf16"  : one product, bf16 operands;
// precision "bf16x3": operands split hi + lo (bf16 each); hi*hi + hi*lo + lo*hi, FP32-class.
//
// Work item = (co tile of 128, image); the image is swept in bands of 64 output pixels.
//
// 16-wide images (the C3 shape): a band is 4 input rows [4k, 4k+4) and NO halo rows.  The
// MMA computes Z for exactly the band's input pixels; output rows that also depend on the
// neighbouring bands are carried across bands in TMEM: band k completes output rows
// [4k-1, 4k+3); the partial sums of row 4k+3 (input rows 4k+2, 4k+3) and of row 4k+4
// (input row 4k+3) are kept for band k+1.  Bases are the outer loop (the carry is per base).
// bf16x3 runs two MMAs per K-step: Wh x [Xh | Xl] (N = 128, one read of the hi weight tile
// for two products) and Wl x Xh (N = 64, accumulating into the first half); the epilogue
// sums the two halves.  Per K-step the shared-memory port then carries 8 KB of weight
// writes + 8 KB of A reads + 6 KB of B reads (was 8 + 12 + 8.25 with 6-row halo bands).
// Other widths (strips of 4x16, whole 8x8 / 4x4 images) keep halo bands (below).
//
// Persistent CTA (1 per SM), 20 warps:
//   warps 1, 2  MMA       : two issuers, alternating taps (warp 1 the even, warp 2 the odd taps
//                           of the global tap sequence).  An elected lane issues tcgen05.mma
//                           (M = 128, K = 16) into the tap's TMEM buffer and commits to
//                           mbarriers.  The tensor pipe's issue queue is shallow, so every
//                           barrier wait / commit / fence of a single issuer is a pipe bubble;
//                           with two issuers one warp's synchronisation overlaps the other's
//                           MMAs (tools/mma_sync_probe.cu: 67.9 -> 56.1 cycles per N = 96 MMA,
//                           the shared-memory operand floor; profiles/r02/probe/).
//   warps 0, 3  producers : 1-D bulk copies (TMA engine) of pre-packed SW128 tiles, one
//                           producer per MMA warp, each filling that warp's own W ring (stages
//                           of spc ci-chunks of one tap's weights [128 co x 64 ci], hi + lo).
//                           Private rings are consumed strictly in order, so no waiter can
//                           reach for a slot's next mbarrier phase before the current one has
//                           completed (the parity of phase n+1 is that of phase n-1).  Warp 0
//                           also loads the X band (NC tiles of [MMA_N px x 64 ci]).
//   warps 4-19  epilogue  : TMEM lane = output channel co.  The 4 warps of a lane quadrant
//                           own 4 output rows of the band (16-wide: roles, see epi_tap_carry);
//                           a thread holds Y[4 rotations][16 px] = 64 fp32 registers, pulls the
//                           input rows it needs from TMEM (one 16-column load each), scatters
//                           with compile-time offsets (taps unrolled), then pools + stores.
// Pooling / argmax / bias epilogue identical to the SIMT kernel; 128-bit stores.
#include <cuda_bf16.h>

#include <cstdlib>

#include "k3_tables.cuh"
#include "rc_internal.cuh"
#include "tc_ptx.cuh"

namespace rc {
namespace {

using namespace tc;

// Band geometry.  A band is 64 output pixels (the register budget of the epilogue: every
// epilogue thread owns 16 of them):
//   TW = 16 : CARRY -- 4 full rows of a 16-wide image, input rows = output rows, the
//             rows that need the neighbouring bands are carried in TMEM (N = 64; 128 for
//             the bf16x3 [Xh | Xl] concatenation)
//   TW = 0  : strip of 4 rows x 16 columns of a wider image (W % 16 == 0, W >= 32) from
//             6 input rows x 18 columns incl. the halo                  (N = 112, 108 used)
//   TW = 8, 4 (H == W): small images, whole images per band and no halo rows at all (the
//             window rows outside an image are the zero padding): 1 image of 8x8 or 4
//             images of 4x4 per band (N = 64); a thread owns TR = 16/W full rows.
// RS is the TMEM / operand row stride (pixels per input row of the band).
// (Measured and rejected in round 1, not shipped: 2-row bands for W = 32, CTA pairs, the hi
// weight tile staged in TMEM -- DESIGN.md 3.1.)
#ifndef RC_TC_ABLATE_W  // experiment switches (compile time, profiling builds only)
#define RC_TC_ABLATE_W 0
#endif
#ifndef RC_TC_ABLATE_X
#define RC_TC_ABLATE_X 0
#endif
#ifndef RC_TC_CAT  // experiment switch (compile time): 0 = CARRY bf16x3 as three N = 64 MMAs
#define RC_TC_CAT 1
#endif
template <int TW>
struct Geo {
  static constexpr bool STRIP = TW == 0;
  static constexpr bool SMALL = TW == 4 || TW == 8;
  static constexpr bool CARRY = TW == 16 || TW == 0;          // rows carried across bands (no row halo)
  static constexpr bool CAT = TW == 16 && RC_TC_CAT;          // bf16x3 as Wh x [Xh | Xl] + Wl x Xh
  static constexpr int OUT_ROWS = STRIP ? 4 : 64 / TW;        // 4 | 4 | 8 | 16
  static constexpr int IN_ROWS = (SMALL || CARRY) ? OUT_ROWS : OUT_ROWS + 2;
  static constexpr int RS = STRIP ? 18 : TW;                  // pixels per band row
  static constexpr int BAND_PX = IN_ROWS * RS;                // 64 | 72 | 64 | 64
  static constexpr int MMA_N = STRIP ? (BAND_PX + 7) / 8 * 8 : (BAND_PX + 15) / 16 * 16;  // strips: N = 72
  static constexpr int XTILE = MMA_N * 64 * 2;                // bytes of one [MMA_N x 64 ci] bf16 tile
  // TMEM: columns [0, D0) hold the carried rows (CARRY: [0, 64) row 4k-1 of the band, [64,
  // 128) row 4k+4) or keep the 1-column-left halo load of a band's first pixel inside the
  // allocation (strips, small images); D buffers from D0.  A CARRY D buffer is [Z of Xh |
  // Z of Xl] (the bf16 one-pass kernel uses the first half).
  static constexpr uint32_t D0 = CARRY ? 128 : 16;
  static constexpr int DCOLS = CAT ? 2 * MMA_N : MMA_N;       // TMEM columns per D buffer
  static constexpr int NDB = (512 - D0) / DCOLS < 6 ? (512 - D0) / DCOLS : 6;
  static constexpr int TR = SMALL ? 16 / TW : 1;              // output rows per epilogue thread
  static constexpr int IMGS = SMALL ? 64 / (TW * TW) : 1;     // images per band
};
constexpr int KC = 64;                  // ci per chunk (one 128-byte swizzle row of bf16)
constexpr int WTILE = 128 * KC * 2;      // 16 KB
constexpr int EPI_WARP0 = 4;             // warps 0-3: producer warpgroup (TMA, 2 x MMA, idle)
constexpr int NUM_MMA = 2;               // MMA-issuing warps (1 and 2)
// Warps and setmaxnreg budgets.  Halo bands: 16 epilogue warps (one 16-px row of 4
// rotations each) x 104 registers, warps 0-3 at 64 (the MMA warp's loop spills at 32: -2..5%,
// profiles/r01/regsplit_ab.txt).  CARRY bands: 8 epilogue warps x 224 (two rows each: the
// [Xh | Xl] row sums and the carried rows need more than 112 registers per one-row thread),
// warps 0-3 at 56.  setmaxnreg.inc only redistributes the CTA's launch allocation (THREADS x
// the kernel's register count R0: 96 at 640 threads, 168 at 384), so 128 x PROD + 32 x WARPS
// x REGS must not exceed THREADS x R0 -- a larger budget would block setmaxnreg.inc forever;
// launch_tc checks it: 640 x 96 = 128 x 64 + 512 x 104;  384 x 168 = 128 x 56 + 256 x 224.
template <int TW>
struct Epi {
  static constexpr bool CARRY = Geo<TW>::CARRY;
  static constexpr int WARPS = CARRY ? 8 : 16;
  static constexpr int REGS = CARRY ? 224 : 104;
  static constexpr int PROD = CARRY ? 56 : 64;
  static constexpr int THREADS = 32 * (EPI_WARP0 + WARPS);
};
constexpr int MAX_NDB = 6;
constexpr int MAX_NC = 8;                // ci chunks of 64 (Cin <= 512)
constexpr int MAX_STAGES = 8;
constexpr int XH = 16;                   // output columns per epilogue thread

// In-kernel cycle accounting for experiments (tools/tc_kernel_profile.py builds a variant of
// the library with -DRC_TC_PROF=1; the shipped build compiles it out).  Per CTA, 32 slots:
//   MMA warp w (w = 0, 1) at 5w: total, wait D buffer, wait X band, wait W stage, issue
//   10 epilogue warp 4: total, 11 wait D full, 12 finalize; 13 producer 0 wait W slot,
//   14 producer 0 wait X slot, 15 producer 1 wait W slot; 16-18 as 10-12 for epilogue
//   warp 8 (CARRY: the second half of a lane quadrant)
#ifndef RC_TC_PROF
#define RC_TC_PROF 0
#endif
#if RC_TC_PROF
__device__ unsigned long long g_tc_prof[1024 * 32];
#define PROF_T(v) const long long v = clock64()
#define PROF_ADD(slot, t0) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_tc_prof[blockIdx.x * 32 + (slot)], (unsigned long long)(clock64() - (t0)))
#else
#define PROF_T(v)
#define PROF_ADD(slot, t0)
#endif

struct TcParams {
  const uint8_t* xh;  // packed X tiles [n][band][chunk] (hi), XTILE bytes each
  const uint8_t* xl;  // lo plane (3-pass) or null
  const uint8_t* w;   // packed W tiles: bf16x3 [b][ct][t][chunk][part], bf16 [b][ct][t][chunk]
  const float* bias;
  float* y;
  uint8_t* am;
  int N, H, W, Cout, NB, NBK, NC, NCT, pool, gf, RO, passes, w_stages, spc, items;
  int xstream;  // 1: X chunks travel with the W stages (the X band does not fit in smem)
  float inv_r;  // 1/R for average pooling (R a power of two)
  int act;      // rc_activation applied after the bias (last op of the epilogue)
};

// ---- TMEM -> registers ----------------------------------------------------------------
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- pooling epilogue ------------------------------------------------------------------
// Generic in NX, the pixels of one row segment (16 from registers, 4 for a carried row read
// back from TMEM in chunks).
// max-fold of rotations [R0, R0+G) of this base into Yr[R0] (+ argmax a[] per pixel, ties ->
// smallest index); in place to keep the register footprint at Y + staging.  Branch-free
// selects: data-dependent branches here cost several times the compares.
template <int R0, int G, int NX, int RPB>
__device__ __forceinline__ void fold_max(float (&Yr)[RPB][NX], uint32_t (&a)[NX], int kk0) {
#pragma unroll
  for (int r = R0 + 1; r < R0 + G; ++r)
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      const bool gt = Yr[r][j] > Yr[R0][j];
      Yr[R0][j] = gt ? Yr[r][j] : Yr[R0][j];
      a[j] = gt ? (uint32_t)(kk0 + r - R0) : a[j];
    }
}
template <int NX>
__device__ __forceinline__ void store_vec(float* dst, const float (&v)[NX]) {
  float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int k = 0; k < NX / 4; ++k) d4[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
}
template <int NX>
__device__ __forceinline__ void store_row(const TcParams& p, size_t off, float (&v)[NX], const uint32_t (&a)[NX],
                                          float bz, bool fin) {
  if (fin) {
#pragma unroll
    for (int j = 0; j < NX; ++j) v[j] += bz;
    if (p.act == RC_ACT_RELU) {
#pragma unroll
      for (int j = 0; j < NX; ++j) v[j] = fmaxf(v[j], 0.f);
    }
  }
  uint32_t arg[NX / 4];  // argmax bytes, little-endian: pixel j in byte j % 4 of word j / 4
#pragma unroll
  for (int k = 0; k < NX / 4; ++k) arg[k] = a[4 * k] | (a[4 * k + 1] << 8) | (a[4 * k + 2] << 16) | (a[4 * k + 3] << 24);
#if RC_TC_ABLATE_FIN == 2  // experiment: pooled, but one float stored per row (wrong results)
  {
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < NX; ++j) acc += v[j] + (float)arg[j / 4];
    p.y[off] = acc;
    return;
  }
#endif
  store_vec<NX>(p.y + off, v);
  if (p.am) {
    if constexpr (NX % 16 == 0) {
#pragma unroll
      for (int k = 0; k < NX / 16; ++k)
        reinterpret_cast<uint4*>(p.am + off)[k] = make_uint4(arg[4 * k], arg[4 * k + 1], arg[4 * k + 2], arg[4 * k + 3]);
    } else {
#pragma unroll
      for (int k = 0; k < NX / 4; ++k) reinterpret_cast<uint32_t*>(p.am + off)[k] = arg[k];
    }
  }
}

// pool + bias + store NX output pixels [x0, x0+NX) of one row of base b; same semantics
// as ri_simt.cu.  Fold groups gf in {1, 2, 4} stay inside a base; gf % 4 == 0 spans bases
// through a partial (value, argmax) kept in the output row itself (same thread, program
// order).
// bz = bias[co] (0 without bias), loaded once per work item by the caller
#ifndef RC_TC_ABLATE_FIN  // experiment: 1 = no pooling (one float per row stored; wrong results)
#define RC_TC_ABLATE_FIN 0
#endif
template <int TW, int RPB, int NX>
__device__ __forceinline__ void finalize_row(const TcParams& p, float (&Yr)[RPB][NX], int n, int co, int b,
                                             int row, int x0, float bz) {
  const int wimg = TW ? TW : p.W;
  const size_t plane = (size_t)p.H * wimg;
  const size_t ybase = ((size_t)n * p.Cout + co) * p.RO * plane + (size_t)row * wimg + x0;
#if RC_TC_ABLATE_FIN == 1
  {
    float acc = bz;
#pragma unroll
    for (int r = 0; r < RPB; ++r)
#pragma unroll
      for (int j = 0; j < NX; ++j) acc += Yr[r][j];
    p.y[ybase] = acc;
    return;
  }
#endif
  uint32_t arg[NX];  // per-pixel argmax (orientation index within the fold group)
#pragma unroll
  for (int j = 0; j < NX; ++j) arg[j] = 0;
  if constexpr (RPB == 1) {  // single orientation: every reduction of one slice is the slice
    store_row<NX>(p, ybase, Yr[0], arg, bz, true);
    return;
  } else {
  if (p.pool == RC_POOL_NONE) {
#pragma unroll
    for (int r = 0; r < 4; ++r) store_row<NX>(p, ybase + (size_t)(b * 4 + r) * plane, Yr[r], arg, bz, true);
    return;
  }
  if (p.pool == RC_POOL_AVG) {
    if (b > 0) {
#pragma unroll
      for (int j = 0; j < NX; ++j) Yr[0][j] = p.y[ybase + j] + Yr[0][j];
    }
#pragma unroll
    for (int r = 1; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < NX; ++j) Yr[0][j] += Yr[r][j];
    if (b == p.NB - 1) {  // R is a power of two here (tc_supported): x * (1/R) == x / R exactly
#pragma unroll
      for (int j = 0; j < NX; ++j) Yr[0][j] = __fadd_rn(__fmul_rn(Yr[0][j], p.inv_r), bz);
      if (p.act == RC_ACT_RELU) {
#pragma unroll
        for (int j = 0; j < NX; ++j) Yr[0][j] = fmaxf(Yr[0][j], 0.f);
      }
    }
    store_vec<NX>(p.y + ybase, Yr[0]);
    return;
  }
  const int gf = p.gf;
  if (gf == 1) {
#pragma unroll
    for (int r = 0; r < 4; ++r) store_row<NX>(p, ybase + (size_t)(b * 4 + r) * plane, Yr[r], arg, bz, true);
  } else if (gf == 2) {
    fold_max<0, 2, NX>(Yr, arg, 0);
    store_row<NX>(p, ybase + (size_t)(b * 2) * plane, Yr[0], arg, bz, true);
#pragma unroll
    for (int j = 0; j < NX; ++j) arg[j] = 0;
    fold_max<2, 2, NX>(Yr, arg, 0);
    store_row<NX>(p, ybase + (size_t)(b * 2 + 1) * plane, Yr[2], arg, bz, true);
  } else {  // gf % 4 == 0
    const int o0 = b * 4, slot = o0 / gf, kk0 = o0 - slot * gf;
    const size_t off = ybase + (size_t)slot * plane;
#pragma unroll
    for (int j = 0; j < NX; ++j) arg[j] = (uint32_t)kk0;  // candidate r = 0 is index kk0
    fold_max<0, 4, NX>(Yr, arg, kk0);
    if (kk0 > 0) {  // continue the slot begun in an earlier base
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        const float prev = p.y[off + j];
        const uint32_t pa = p.am ? p.am[off + j] : 0u;
        const bool keep = !(Yr[0][j] > prev);  // earlier (smaller) index wins ties
        Yr[0][j] = keep ? prev : Yr[0][j];
        arg[j] = keep ? pa : arg[j];
      }
    }
    store_row<NX>(p, off, Yr[0], arg, bz, kk0 + 4 == gf);
  }
  }
}

// ---- scatter ------------------------------------------------------------------------
// A thread's 16 output columns [x0, x0+16) of output row o read input rows o-1 .. o+1
// (D-buffer rows s .. s+2).  z[c] holds input column x0 - 1 + c (c = 0..17); columns
// outside the image are zero in the band (strips) or are skipped at compile time (TW = 16:
// the thread's 16 columns are the whole row).  Y_r(p) += Z_t(p + (di, dj)): for tap T and
// rotation r the single contributing row is I = 1 + di.
template <int TW, int RPB, int CONV, int T, int I>
__device__ __forceinline__ void scatter_row(float (&Y)[RPB][XH], const float (&z)[18]) {
#pragma unroll
  for (int r = 0; r < RPB; ++r) {
    const int di = make_k3(CONV).di[r][T];
    const int dj = make_k3(CONV).dj[r][T];
    if (1 + di != I) continue;
#pragma unroll
    for (int x = 0; x < XH; ++x) {
      const int src = x + dj + 1;
      if (TW == 16 && (src < 1 || src > 16)) continue;
      Y[r][x] += z[src];
    }
  }
}

// one input row of a strip thread's window: the two halo columns after its 16
__device__ __forceinline__ void tmem_ld2f(uint32_t taddr, float& a, float& b) {
  uint32_t r0, r1;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(taddr));
  a = __uint_as_float(r0);
  b = __uint_as_float(r1);
}

// one input row of the thread's window: 16 columns + (strips) the halo columns.
// issue_row only issues the TMEM loads; the caller waits (tcgen05.wait::ld).
template <int TW>
__device__ __forceinline__ void issue_row(uint32_t a, float (&z)[18]) {
  if constexpr (TW == 0) {  // strip: the band row holds the halo columns (zero at image edges)
    tmem_ld16(a, *reinterpret_cast<float(*)[16]>(&z[0]));
    tmem_ld2f(a + 16, z[16], z[17]);
  } else {
    tmem_ld16(a, *reinterpret_cast<float(*)[16]>(&z[1]));
  }
}
template <int TW>
__device__ __forceinline__ void load_row(uint32_t a, float (&z)[18]) {
  issue_row<TW>(a, z);
  tmem_wait_ld();
}

// small images: window row I (input row o0 - 1 + I) feeds output row i of the thread's TR
// rows when I == i + 1 + di; z[c] = input column c - 1 (z[0], z[TW+1] are the zero edges).
template <int TW, int RPB, int CONV, int T, int I>
__device__ __forceinline__ void scatter_small(float (&Y)[RPB][XH], const float (&z)[10]) {
  constexpr int TR = Geo<TW>::TR;
#pragma unroll
  for (int r = 0; r < RPB; ++r) {
    const int di = make_k3(CONV).di[r][T];
    const int dj = make_k3(CONV).dj[r][T];
#pragma unroll
    for (int i = 0; i < TR; ++i) {
      if (I != i + 1 + di) continue;
#pragma unroll
      for (int j = 0; j < TW; ++j) {
        const int src = j + 1 + dj;
        if (src < 1 || src > TW) continue;
        Y[r][i * TW + j] += z[src];
      }
    }
  }
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}

template <int TW, int RPB, int CONV, int T, int I>
__device__ __forceinline__ void small_row(uint32_t a, int o0, float (&Y)[RPB][XH]) {
  const int row = o0 - 1 + I;  // image row of window row I
  if (row < 0 || row >= TW) return;  // the zero padding (warp-uniform)
  float z[10];
  const uint32_t ra = a + (uint32_t)(I * TW) - (uint32_t)TW;  // window row I = image row o0 - 1 + I
  if constexpr (TW == 8)
    tmem_ld8(ra, z + 1);
  else
    tmem_ld4(ra, z + 1);
  tmem_wait_ld();
  scatter_small<TW, RPB, CONV, T, I>(Y, z);
}

struct EpiState {
  uint32_t row_base;  // TMEM address of D-buffer 0, first input row of the thread, its columns
  int db;
  uint32_t dph;
  int lane;
  int o0;  // small images: first output row of the thread (within its image)
};

__device__ __forceinline__ void release_d(EpiState& e, int ndb, uint64_t* d_empty) {
  tc_fence_before();
  __syncwarp();
  if (e.lane == 0) mbar_arrive(&d_empty[e.db]);  // D buffer free: an MMA warp may refill it
  if (++e.db == ndb) {
    e.db = 0;
    e.dph ^= 1;
  }
}

// one tap (compile-time T) of the halo-band geometries (strips, small images): the window
// rows from TMEM, D released after the last load
template <int TW, int RPB, int CONV, int T>
__device__ __forceinline__ void epi_tap(EpiState& e, float (&Y)[RPB][XH], uint64_t* d_full, uint64_t* d_empty) {
  constexpr int NDB = Geo<TW>::NDB;
  const uint32_t a = e.row_base + e.db * Geo<TW>::DCOLS;
  float z[18];
  PROF_T(t_df);
  mbar_wait(&d_full[e.db], e.dph);
  if (threadIdx.x / 32 == EPI_WARP0) PROF_ADD(11, t_df);
  tc_fence_after();
  if constexpr (Geo<TW>::SMALL) {
    constexpr int TR = Geo<TW>::TR;
    small_row<TW, RPB, CONV, T, 0>(a, e.o0, Y);
    small_row<TW, RPB, CONV, T, 1>(a, e.o0, Y);
    if constexpr (TR >= 2) small_row<TW, RPB, CONV, T, 2>(a, e.o0, Y);
    if constexpr (TR >= 2) small_row<TW, RPB, CONV, T, 3>(a, e.o0, Y);
    if constexpr (TR >= 4) small_row<TW, RPB, CONV, T, 4>(a, e.o0, Y);
    if constexpr (TR >= 4) small_row<TW, RPB, CONV, T, 5>(a, e.o0, Y);
    release_d(e, NDB, d_empty);
    return;
  } else {  // strips: rows 0 and 1 in flight together
    float z1[18];
    issue_row<TW>(a, z);
    issue_row<TW>(a + Geo<TW>::RS, z1);
    tmem_wait_ld();
    scatter_row<TW, RPB, CONV, T, 0>(Y, z);
    scatter_row<TW, RPB, CONV, T, 1>(Y, z1);
    load_row<TW>(a + 2 * Geo<TW>::RS, z);
    release_d(e, NDB, d_empty);
    scatter_row<TW, RPB, CONV, T, 2>(Y, z);
  }
}

// ---- 16-wide carry bands ---------------------------------------------------------------
// D-row i of a CARRY D buffer (input row 4k + i): the thread's 16 columns of Z(Xh) (+ Z(Xl),
// bf16x3 concatenation) into z[1..16]; strips also the halo columns 16j-1, 16j+16 (z[0], z[17])
template <bool cat, int TW>
__device__ __forceinline__ void load_row_cat(uint32_t a, float (&z)[18]) {
  if constexpr (TW == 0) {
    issue_row<0>(a, z);
    tmem_wait_ld();
  } else {
    float(&zz)[16] = *reinterpret_cast<float(*)[16]>(&z[1]);
    tmem_ld16(a, zz);
    if constexpr (cat) {
      float t[16];
      tmem_ld16(a + Geo<16>::MMA_N, t);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) zz[j] += t[j];
    } else {
      tmem_wait_ld();
    }
  }
}

// scatter one input row into a row state kept in TMEM (carry + r*16 = rotation r, 16 px):
// read-modify-write of each rotation that takes this row (I = 1 + di, as scatter_row)
template <int RPB, int CONV, int T, int I, int TW>
__device__ __forceinline__ void rmw_row(uint32_t carry, const float (&z)[18]) {
  bool wrote = false;
#pragma unroll
  for (int r = 0; r < RPB; ++r) {
    const int di = make_k3(CONV).di[r][T];
    const int dj = make_k3(CONV).dj[r][T];
    if (1 + di != I) continue;
    float c[16];
    tmem_ld16(carry + r * 16, c);
    tmem_wait_ld();
#pragma unroll
    for (int x = 0; x < 16; ++x) {
      const int src = x + dj + 1;
      if (TW == 16 && (src < 1 || src > 16)) continue;  // strips: z[0], z[17] are the halo columns
      c[x] += z[src];
    }
    tmem_st16(carry + r * 16, c);
    wrote = true;
  }
  if (wrote) tmem_wait_st();
}

// One tap of a 16-wide carry band k.  The 2 warps of a lane quadrant (half h) each own two
// output rows in registers (Y0, Y1) and one carried row in TMEM:
//   h = 0: Y0 = row 4k   (D-rows 0, 1; its input row 4k-1 came in as carry B),
//          Y1 = row 4k+1 (D-rows 0, 1, 2), TMEM carry B = row 4k+4 (D-row 3)
//   h = 1: Y0 = row 4k+2 (D-rows 1, 2, 3), Y1 = row 4k+3 (D-rows 2, 3),
//          TMEM carry A = row 4k-1 (D-row 0; k > 0)
// Each thread reads the 4 D-rows once per tap.  I = 1 + di selects the rotations of tap T
// that read the row (scatter_row).
template <int TW, int RPB, int CONV, int H, int T, bool cat>
__device__ __forceinline__ void epi_tap_carry(EpiState& e, float (&Y0)[RPB][XH], float (&Y1)[RPB][XH],
                                              bool first_band, uint32_t carry, uint64_t* d_full,
                                              uint64_t* d_empty) {
  using G = Geo<TW>;
  constexpr uint32_t RS = G::RS;
  const uint32_t a = e.row_base + e.db * G::DCOLS;
  float z[18];
  PROF_T(t_df);
  mbar_wait(&d_full[e.db], e.dph);
  if (threadIdx.x / 32 == EPI_WARP0) PROF_ADD(11, t_df);
  if (threadIdx.x / 32 == EPI_WARP0 + 4) PROF_ADD(17, t_df);
  tc_fence_after();
  if constexpr (H == 0) {
    load_row_cat<cat, TW>(a, z);
    scatter_row<TW, RPB, CONV, T, 1>(Y0, z);
    scatter_row<TW, RPB, CONV, T, 0>(Y1, z);
    load_row_cat<cat, TW>(a + RS, z);
    scatter_row<TW, RPB, CONV, T, 2>(Y0, z);
    scatter_row<TW, RPB, CONV, T, 1>(Y1, z);
    load_row_cat<cat, TW>(a + 2 * RS, z);
    scatter_row<TW, RPB, CONV, T, 2>(Y1, z);
    load_row_cat<cat, TW>(a + 3 * RS, z);
    release_d(e, G::NDB, d_empty);
    rmw_row<RPB, CONV, T, 0, TW>(carry, z);
  } else {
    load_row_cat<cat, TW>(a + RS, z);
    scatter_row<TW, RPB, CONV, T, 0>(Y0, z);
    load_row_cat<cat, TW>(a + 2 * RS, z);
    scatter_row<TW, RPB, CONV, T, 1>(Y0, z);
    scatter_row<TW, RPB, CONV, T, 0>(Y1, z);
    load_row_cat<cat, TW>(a + 3 * RS, z);
    scatter_row<TW, RPB, CONV, T, 2>(Y0, z);
    scatter_row<TW, RPB, CONV, T, 1>(Y1, z);
    if (first_band) {
      release_d(e, G::NDB, d_empty);
    } else {
      load_row_cat<cat, TW>(a, z);
      release_d(e, G::NDB, d_empty);
      rmw_row<RPB, CONV, T, 2, TW>(carry, z);
    }
  }
}

// h = 1 at the end of band k > 0: output row 4k-1 lives in TMEM carry A; pool + store it
// in chunks of 4 pixels
// (the TMEM loads are warp-collective, .sync.aligned: every lane loads, only live lanes,
// co < Cout, store)
template <int TW, int RPB>
__device__ __forceinline__ void finalize_carried(const TcParams& p, uint32_t carry, int n, int co, int b, int row,
                                                 int x0, bool live, float bz) {
#pragma unroll 1
  for (int c4 = 0; c4 < 4; ++c4) {
    float Yc[RPB][4];
#pragma unroll
    for (int r = 0; r < RPB; ++r) tmem_ld4(carry + r * 16 + c4 * 4, Yc[r]);
    tmem_wait_ld();
    if (live) finalize_row<TW, RPB, 4>(p, Yc, n, co, b, row, x0 + c4 * 4, bz);
  }
}

template <int TW, int RPB, int CONV, int H, bool P3>
__device__ __forceinline__ void epilogue_carry_half(const TcParams& p, uint32_t tmem, uint64_t* d_full,
                                                    uint64_t* d_empty) {
  using G = Geo<TW>;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q = warp % 4;
  const int co_l = q * 32 + lane;
  const uint32_t lanes = tmem + ((uint32_t)(q * 32) << 16);
  const uint32_t carry = lanes + (H == 1 ? 0u : 64u);  // TMEM columns [0, 64): carry A, [64, 128): carry B
  constexpr bool cat = G::CAT && P3;
  EpiState e{lanes + G::D0, 0, 0, lane, 0};
  const int nrb = G::STRIP ? (p.H + 3) / 4 : p.NBK;  // row bands (per strip)
  float Y0[RPB][XH], Y1[RPB][XH];
  PROF_T(t_epi0);
  for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
    const int n = item / p.NCT, ct = item % p.NCT;
    const int co = ct * 128 + co_l;
    const bool live = co < p.Cout;
    const float bz = (live && p.bias) ? p.bias[co] : 0.f;
    // units (base b, band kk): strips are strip-major, kk = j * nrb + k (k = row band)
    for (int b = 0; b < p.NB; ++b)
      for (int kk = 0; kk < p.NBK; ++kk) {
        const int k = G::STRIP ? kk % nrb : kk, x0 = G::STRIP ? (kk / nrb) * 16 : 0;
        const bool first = k == 0, last = k == nrb - 1;
        if (H == 0 && !first) {  // row 4k: its input row 4k-1 was scattered in band k-1
#pragma unroll
          for (int r = 0; r < RPB; ++r) tmem_ld16(carry + r * 16, Y0[r]);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int r = 0; r < RPB; ++r)
#pragma unroll
            for (int x = 0; x < XH; ++x) Y0[r][x] = 0.f;
        }
#pragma unroll
        for (int r = 0; r < RPB; ++r)
#pragma unroll
          for (int x = 0; x < XH; ++x) Y1[r][x] = 0.f;
        if (H == 0) {  // carry B restarts for row 4k+4
#pragma unroll
          for (int r = 0; r < RPB; ++r) tmem_st16_zero(carry + r * 16);
          tmem_wait_st();
        }
        epi_tap_carry<TW, RPB, CONV, H, 0, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        epi_tap_carry<TW, RPB, CONV, H, 1, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        epi_tap_carry<TW, RPB, CONV, H, 2, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        epi_tap_carry<TW, RPB, CONV, H, 3, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        epi_tap_carry<TW, RPB, CONV, H, 4, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        epi_tap_carry<TW, RPB, CONV, H, 5, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        epi_tap_carry<TW, RPB, CONV, H, 6, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        epi_tap_carry<TW, RPB, CONV, H, 7, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        epi_tap_carry<TW, RPB, CONV, H, 8, cat>(e, Y0, Y1, first, carry, d_full, d_empty);
        PROF_T(t_fin);
        // Rows to store: h = 0 rows 4k, 4k+1; h = 1 the carried row 4k-1 (k > 0), row 4k+2 and,
        // in the last band (input row 4k+4 is padding), row 4k+3 -- otherwise row 4k+3
        // continues in band k+1 through carry A.  One finalize call site per half (a rolled
        // loop moving Y1 into Y0): the pooling code is large and runs once per band, so
        // inlined copies would only evict the tap loop from the instruction cache.
        int nrows = 2;
        if constexpr (H == 1) {
          if (!first && 4 * k - 1 < p.H) finalize_carried<TW, RPB>(p, carry, n, co, b, 4 * k - 1, x0, live, bz);
          if (!last) {
#pragma unroll
            for (int r = 0; r < RPB; ++r) tmem_st16(carry + r * 16, Y1[r]);
            tmem_wait_st();
            nrows = 1;
          }
        }
#pragma unroll 1
        for (int i = 0; i < nrows; ++i) {
          const int row = 4 * k + 2 * H + i;
          if (live && row < p.H) finalize_row<TW, RPB, XH>(p, Y0, n, co, b, row, x0, bz);
          if (i == 0) {
#pragma unroll
            for (int r = 0; r < RPB; ++r)
#pragma unroll
              for (int x = 0; x < XH; ++x) Y0[r][x] = Y1[r][x];
          }
        }
        if (warp == EPI_WARP0) PROF_ADD(12, t_fin);
        if (warp == EPI_WARP0 + 4) PROF_ADD(18, t_fin);
      }
  }
  if (warp == EPI_WARP0) PROF_ADD(10, t_epi0);
  if (warp == EPI_WARP0 + 4) PROF_ADD(16, t_epi0);
}

// the 8 epilogue warps of a carry kernel: half h = (warp - 4) / 4 of its lane quadrant
// (compile time below the dispatch: each half's band loop is straight-line code)
template <int TW, int RPB, int CONV, bool P3>
__device__ __forceinline__ void epilogue_carry(const TcParams& p, uint32_t tmem, uint64_t* d_full, uint64_t* d_empty) {
  if ((threadIdx.x / 32 - EPI_WARP0) / 4 == 0)
    epilogue_carry_half<TW, RPB, CONV, 0, P3>(p, tmem, d_full, d_empty);
  else
    epilogue_carry_half<TW, RPB, CONV, 1, P3>(p, tmem, d_full, d_empty);
}

// Epilogue warp of the halo-band geometries: lane quadrant q (co = q*32 + lane); sub-tile
// sub = output row of the band.  Work schedule: CTA i walks items i, i + grid, ...; item ->
// (image n, co tile ct) = (item / NCT, item % NCT).
template <int TW, int RPB, int CONV>
__device__ __forceinline__ void epilogue(const TcParams& p, uint32_t tmem, uint64_t* d_full, uint64_t* d_empty) {
  using G = Geo<TW>;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q = warp % 4;
  const int sub = (warp - EPI_WARP0) / 4;
  const int srow = sub;
  const int co_l = q * 32 + lane;
  // small images: sub = image of the band (4x4) or row pair (8x8); row_base -> its first row
  const int s_img = G::SMALL ? (G::IMGS > 1 ? sub : 0) : 0;
  const int o0 = G::SMALL ? (G::IMGS > 1 ? 0 : sub * G::TR) : 0;
  const uint32_t rb = G::SMALL ? (uint32_t)((s_img * TW + o0) * G::RS) : (uint32_t)(srow * G::RS);
  EpiState e{tmem + ((uint32_t)(q * 32) << 16) + G::D0 + rb, 0, 0, lane, o0};
  const int nstrip = G::STRIP ? p.W / 16 : 1;
  float Y[RPB][XH];
  PROF_T(t_epi0);
  for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
    const int n = item / p.NCT, ct = item % p.NCT;
    const int co = ct * 128 + co_l;
    const float bz = (co < p.Cout && p.bias) ? p.bias[co] : 0.f;
    for (int k = 0; k < p.NBK; ++k)
      for (int b = 0; b < p.NB; ++b) {
#pragma unroll
        for (int r = 0; r < RPB; ++r)
#pragma unroll
          for (int x = 0; x < XH; ++x) Y[r][x] = 0.f;
        epi_tap<TW, RPB, CONV, 0>(e, Y, d_full, d_empty);
        epi_tap<TW, RPB, CONV, 1>(e, Y, d_full, d_empty);
        epi_tap<TW, RPB, CONV, 2>(e, Y, d_full, d_empty);
        epi_tap<TW, RPB, CONV, 3>(e, Y, d_full, d_empty);
        epi_tap<TW, RPB, CONV, 4>(e, Y, d_full, d_empty);
        epi_tap<TW, RPB, CONV, 5>(e, Y, d_full, d_empty);
        epi_tap<TW, RPB, CONV, 6>(e, Y, d_full, d_empty);
        epi_tap<TW, RPB, CONV, 7>(e, Y, d_full, d_empty);
        epi_tap<TW, RPB, CONV, 8>(e, Y, d_full, d_empty);
        const int row = G::SMALL ? o0 : G::OUT_ROWS * (k / nstrip) + srow;
        const int x0 = G::SMALL ? 0 : (k % nstrip) * 16;
        const int img = G::SMALL ? n * G::IMGS + s_img : n;  // small: n indexes bands of IMGS images
        PROF_T(t_fin);
        if (img < p.N && co < p.Cout && row < p.H) finalize_row<TW, RPB, XH>(p, Y, img, co, b, row, x0, bz);
        if (warp == EPI_WARP0) PROF_ADD(12, t_fin);
      }
  }
  if (warp == EPI_WARP0) PROF_ADD(10, t_epi0);
}

// smem ring position: stage index + phase parity, advanced without division
struct Ring {
  uint32_t s = 0, ph = 0;
  bool used = false;
  __device__ __forceinline__ void adv(int S) {
    if (++s == (uint32_t)S) {
      s = 0;
      ph ^= 1;
      used = true;
    }
  }
};

// P3: bf16x3 (three products) -- compile time for the CARRY epilogue's [Xh | Xl] row sums
template <int TW, int RPB, int CONV, bool P3>
__global__ void __launch_bounds__(Epi<TW>::THREADS, 1) ri_tc_kernel(const __grid_constant__ TcParams p) {
  using G = Geo<TW>;
  constexpr int NDB = G::NDB;
  constexpr int XS = G::XTILE;                        // bytes of a band tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB alignment for the SW128 atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int parts = p.passes == 3 ? 2 : 1;
  uint8_t* xs = smem;                           // X band: [part][chunk] tiles of XS bytes
  uint8_t* ws = smem + (p.xstream ? 0 : parts * p.NC * XS);  // W (+ X when streamed) ring
  // per-chunk X barriers: chunk c of band k+1 is reloaded as soon as both MMA warps' last taps
  // of band k on chunk c complete, so band transitions overlap the last taps' MMAs
  __shared__ uint64_t w_full[MAX_STAGES], w_empty[MAX_STAGES], x_full[MAX_NC], x_empty[MAX_NC], d_full[MAX_NDB],
      d_empty[MAX_NDB];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32;
  const int S = p.w_stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int i = 0; i < p.NC; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], NUM_MMA);  // one commit per MMA warp per band
    }
    for (int i = 0; i < NDB; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], Epi<TW>::WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  // W stage = spc consecutive ci-chunks of one tap (hi, or hi+lo interleaved), ONE bulk
  // copy of >= 32 KB: the TMA engine's per-copy cost makes small copies the bottleneck
  // (profiles/r01/l2_microbench.jsonl).
  const int stage_w = p.spc * parts * WTILE;                      // W bytes of a stage
  const int stage_bytes = stage_w + (p.xstream ? p.spc * parts * XS : 0);
  const int stages_per_tap = p.NC / p.spc;
  // ring 0 (MMA warp 1): slots [0, S0); ring 1 (MMA warp 2): [S0, S).  The odd slot goes to ring 1:
  // producer 0 also loads the X bands, so ring 0 runs fuller anyway (C3 -1.3%, C4 -2.5%,
  // profiles/r02/c3_carry/variants_ab.txt)
  const int S0 = S / 2;
  // X chunk c of a region of `cnt` chunks (the resident band: NC; a streamed stage: spc).
  // CARRY: [Xh rows | Xl rows] of a chunk are adjacent (one N = 128 B operand, one copy);
  // otherwise [hi chunks][lo chunks].
  // (lambdas capture scalars by value: a by-reference capture of the __grid_constant__ params
  // would turn every later p.field read into a generic memory load)
  auto xh_off = [=](int c, int cnt) -> uint32_t { return (uint32_t)(G::CARRY ? c * parts * XS : c * XS); };
  auto xl_off = [=](int c, int cnt) -> uint32_t {
    return (uint32_t)(G::CARRY ? c * parts * XS + XS : (cnt + c) * XS);
  };
  // Band schedule of a work item: units u = (band k, base b).  CARRY bands walk the bases
  // outermost (the carried rows belong to one base) and reload X per unit; halo bands keep X
  // resident across the bases of a band.
  const int NB = p.NB, NBK = p.NBK;
  const int units = NB * NBK;
  auto unit_k = [=](int u) { return G::CARRY ? u % NBK : u / NB; };
  auto unit_b = [=](int u) { return G::CARRY ? u / NBK : u % NB; };
  auto x_first = [=](int u) { return G::CARRY || unit_b(u) == 0; };      // unit loads a new X band
  auto x_last = [=](int u) { return G::CARRY || unit_b(u) == NB - 1; };  // last unit on this X band
  const int taps_per_band = G::CARRY ? 9 : p.NB * 9;                          // taps per X band
  if (warp < EPI_WARP0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Epi<TW>::PROD));
  if (warp == 0 || warp == 3) {
    // ------------------------------------------------------------ producers (whole warp
    // walks the schedule in MMA consumption order; one elected lane issues the copies).
    // Producer i = warp / 3 fills ring i for the taps of MMA warp i + 1.
    const uint32_t me = warp == 0 ? 0u : 1u;
    const int S_me = me == 0 ? S0 : S - S0, base = me == 0 ? 0 : S0;
    Ring wr;
    uint32_t xc = 0, gd = 0;  // bands loaded so far (phase of the per-chunk X barriers), global tap
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      const int n = item / p.NCT, ct = item % p.NCT;
      for (int u = 0; u < units; ++u) {
        const int k = unit_k(u), b = unit_b(u);
        const size_t tile = ((size_t)n * p.NBK + k) * p.NC;
        if (me == 0 && !p.xstream && x_first(u)) {  // new band: its X chunks (both MMA warps read them)
          for (int c = 0; c < p.NC; ++c) {
            PROF_T(t_xe);
            if (xc > 0) mbar_wait(&x_empty[c], (xc - 1) & 1);
            PROF_ADD(14, t_xe);
            if (elect_one()) {
#if RC_TC_ABLATE_X  // experiment: X loaded once per CTA (stale bands later; wrong results)
              if (xc > 0) {
                mbar_arrive(&x_full[c]);
              } else
#endif
              {
              mbar_arrive_expect_tx(&x_full[c], parts * XS);
              if (G::CARRY) {
                bulk_g2s(xs + xh_off(c, p.NC), p.xh + (tile + c) * parts * XS, parts * XS, &x_full[c]);
              } else {
                bulk_g2s(xs + xh_off(c, p.NC), p.xh + (tile + c) * XS, XS, &x_full[c]);
                if (parts == 2) bulk_g2s(xs + xl_off(c, p.NC), p.xl + (tile + c) * XS, XS, &x_full[c]);
              }
              }
            }
            __syncwarp();
          }
        }
        const uint8_t* wsrc = p.w + (((size_t)b * p.NCT + ct) * 9) * p.NC * parts * WTILE;
        for (int t = 0; t < 9; ++t, ++gd) {
          if ((gd & 1u) != me) continue;
          for (int sp = 0; sp < stages_per_tap; ++sp) {
            const int st = t * stages_per_tap + sp;
            PROF_T(t_we);
            if (wr.used) mbar_wait(&w_empty[base + wr.s], wr.ph ^ 1);
            PROF_ADD(me == 0 ? 13 : 15, t_we);
            if (elect_one()) {
              uint64_t* full = &w_full[base + wr.s];
              uint8_t* dst = ws + (base + wr.s) * stage_bytes;
#if RC_TC_ABLATE_W  // experiment: no weight traffic (stale stage contents; wrong results)
              mbar_arrive(full);
#else
              mbar_arrive_expect_tx(full, stage_bytes);
              bulk_g2s(dst, wsrc + (size_t)st * stage_w, stage_w, full);
#endif
              if (p.xstream) {  // the stage's X chunks travel with it (re-read from L2 per tap)
                const int c0 = sp * p.spc;
                for (int cl = 0; cl < p.spc; ++cl) {
                  if (G::CARRY) {
                    bulk_g2s(dst + stage_w + xh_off(cl, p.spc), p.xh + (tile + c0 + cl) * parts * XS, parts * XS,
                             full);
                  } else {
                    bulk_g2s(dst + stage_w + xh_off(cl, p.spc), p.xh + (tile + c0 + cl) * XS, XS, full);
                    if (parts == 2)
                      bulk_g2s(dst + stage_w + xl_off(cl, p.spc), p.xl + (tile + c0 + cl) * XS, XS, full);
                  }
                }
              }
            }
            __syncwarp();
            wr.adv(S_me);
          }
        }
        if (x_last(u)) ++xc;
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ------------------------------------------------------------ MMA issuers.  Both warps
    // walk the whole schedule (ring / buffer / phase state stays in lockstep); warp 1 issues
    // the even taps of the global tap sequence, warp 2 the odd ones.  Each tap has its own
    // D buffer and W stages, so the two streams never touch the same accumulator; each warp
    // commits its own MMAs (tcgen05.commit tracks the issuing thread's operations).
    const uint32_t me = (uint32_t)(warp - 1);
    const int S_me = me == 0 ? S0 : S - S0, base = me == 0 ? 0 : S0;
    // CAT bf16x3: Wh x [Xh | Xl] (N = 2 * MMA_N) then Wl x Xh (N = MMA_N) into its first half
    const uint32_t idesc = idesc_bf16_f32(128, (G::CAT && parts == 2) ? 2 * G::MMA_N : G::MMA_N);
    const uint32_t idesc_n = idesc_bf16_f32(128, G::MMA_N);
    const uint32_t xaddr = smem_u32(xs);
    Ring wr;
    uint32_t xc = 0, gd = 0;  // gd: global tap index
    int db = 0;
    uint32_t dph = 0;
    PROF_T(t_mma0);
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      for (int u = 0; u < units; ++u) {
        const int b = unit_b(u);
        for (int t = 0; t < 9; ++t) {
          const int tb = (G::CARRY ? 0 : b * 9) + t;      // tap index within the X band
          const bool mine = (gd & 1u) == me;
          const bool first_mine = tb < 2;                 // this warp's first tap of the X band
          const bool last_mine = tb + 2 >= taps_per_band;  // ... and its last one
          if (mine) {
            PROF_T(t_d);
            if (gd >= (uint32_t)NDB) mbar_wait(&d_empty[db], dph ^ 1);
            PROF_ADD(5 * me + 1, t_d);
            tc_fence_after();
            const uint32_t d = tmem + G::D0 + db * G::DCOLS;
            for (int sp = 0; sp < stages_per_tap; ++sp) {
              PROF_T(t_x);
              if (first_mine && !p.xstream)
                for (int cl = 0; cl < p.spc; ++cl) mbar_wait(&x_full[sp * p.spc + cl], xc & 1);
              PROF_ADD(5 * me + 2, t_x);
              PROF_T(t_w);
              mbar_wait(&w_full[base + wr.s], wr.ph);
              PROF_ADD(5 * me + 3, t_w);
              tc_fence_after();
              PROF_T(t_i);
              if (elect_one()) {
                const uint32_t wbase = smem_u32(ws + (base + wr.s) * stage_bytes);
                // descriptors are linear in the smem address (14-bit field, smem < 256 KB): one
                // base per stage, constant strides per chunk
                const uint32_t xbase = p.xstream ? wbase + stage_w : xaddr;
                const int cbase = p.xstream ? 0 : sp * p.spc, cnt = p.xstream ? p.spc : p.NC;
                const uint64_t a0 = desc_k_sw128(wbase);
                for (int cl = 0; cl < p.spc; ++cl) {
                  const int c = sp * p.spc + cl;
                  const uint64_t bh = desc_k_sw128(xbase + xh_off(cbase + cl, cnt));
                  const uint64_t ah = a0 + (uint32_t)((cl * parts * WTILE) >> 4);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, ah + 2 * kk, bh + 2 * kk, idesc, (c | kk) != 0);
                  if (parts == 2) {
                    const uint64_t al = desc_k_sw128(wbase + (cl * parts + 1) * WTILE);
                    if (!G::CAT) {
                      const uint64_t bl = desc_k_sw128(xbase + xl_off(cbase + cl, cnt));
#pragma unroll
                      for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, ah + 2 * kk, bl + 2 * kk, idesc_n, 1);
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, al + 2 * kk, bh + 2 * kk, idesc_n, 1);
                  }
                  if (last_mine && !p.xstream) mma_commit(&x_empty[c]);  // chunk c done by this warp
                }
                mma_commit(&w_empty[base + wr.s]);
                if (sp == stages_per_tap - 1) mma_commit(&d_full[db]);
              }
              __syncwarp();
              PROF_ADD(5 * me + 4, t_i);
              wr.adv(S_me);
            }
          }
          ++gd;
          if (++db == NDB) {
            db = 0;
            dph ^= 1;
          }
        }
        if (x_last(u)) ++xc;
      }
    }
    PROF_ADD(5 * me, t_mma0);
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Epi<TW>::REGS));
    if constexpr (G::CARRY)
      epilogue_carry<TW, RPB, CONV, P3>(p, tmem, d_full, d_empty);
    else
      epilogue<TW, RPB, CONV>(p, tmem, d_full, d_empty);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}


// ---- packing kernels ------------------------------------------------------------------
__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// X fp32 NCHW -> SW128 bf16 tiles [n][band][chunk][MMA_N px][64 ci] (hi, lo planes).  Band
// pixel px is (r = px / RS, cc = px % RS) -> image row k*OUT_ROWS - 1 + r (k*OUT_ROWS + r
// for CARRY bands) and column cc (full rows) or j*16 - 1 + cc (strip j); pixels outside the
// image (the padding) and the MMA_N - BAND_PX filler pixels are zero.
template <int TW>
__global__ void x_pack_kernel(const float* __restrict__ x, uint8_t* __restrict__ xh,
                              uint8_t* __restrict__ xl, int Cin, int H, int W, int NBK, int NC, int Nimg) {
  using G = Geo<TW>;
  __shared__ float tile[KC][G::MMA_N + 1];
  const int c = blockIdx.x, bk = blockIdx.y, n = blockIdx.z;
  const int nstrip = G::STRIP ? W / 16 : 1;
  const int k = bk / nstrip, j = bk % nstrip;
  for (int i = threadIdx.x; i < KC * G::MMA_N; i += blockDim.x) {
    const int cl = i / G::MMA_N, px = i % G::MMA_N;
    const int ci = c * KC + cl;
    int img = n, row, col;
    if constexpr (G::SMALL) {  // band = IMGS whole images, px = (image, row, col), no halo rows
      img = n * G::IMGS + px / (TW * TW);
      row = (px / TW) % TW;
      col = px % TW;
    } else if constexpr (G::CARRY) {  // input rows [4k, 4k+4), no row halo; strips: the columns
                                      // 16j-1 .. 16j+16 of strip j, bands strip-major
      const int nrb = (H + 3) / 4;
      const int kb = G::STRIP ? bk % nrb : bk, js = G::STRIP ? bk / nrb : 0;
      row = kb * G::OUT_ROWS + px / G::RS;
      col = G::STRIP ? js * 16 - 1 + px % G::RS : px % G::RS;
    } else {
      row = k * G::OUT_ROWS - 1 + px / G::RS;
      col = G::STRIP ? j * 16 - 1 + px % G::RS : px % G::RS;
    }
    const bool in = px < G::BAND_PX && ci < Cin && img < Nimg && row >= 0 && row < H && col >= 0 && col < W;
    // cp.async (zero-filled outside): no thread waits on one load before issuing the next
    const float* src = in ? x + (((size_t)img * Cin + ci) * H + row) * W + col : x;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(&tile[cl][px])), "l"(src),
                 "r"(in ? 4 : 0));
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const size_t tidx = ((size_t)n * NBK + bk) * NC + c;
  // CARRY: one tile per chunk of [MMA_N hi rows | MMA_N lo rows] (the N = 128 B operand of
  // Wh x [Xh | Xl]); xl selects the two-part layout.  Otherwise separate hi / lo planes.
  uint8_t* oh = G::CARRY ? xh + tidx * (xl ? 2 : 1) * G::XTILE : xh + tidx * G::XTILE;
  uint8_t* ol = !xl ? nullptr : (G::CARRY ? oh + G::XTILE : xl + tidx * G::XTILE);
  for (int i = threadIdx.x; i < G::MMA_N * (KC / 8); i += blockDim.x) {
    const int px = i / (KC / 8), g = i % (KC / 8);
    __align__(16) __nv_bfloat16 h8[8], l8[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) split_bf16(tile[g * 8 + jj][px], h8[jj], l8[jj]);
    const uint32_t off = sw128_offset(px, g * 8);
    *reinterpret_cast<uint4*>(oh + off) = *reinterpret_cast<const uint4*>(h8);
    if (ol) *reinterpret_cast<uint4*>(ol + off) = *reinterpret_cast<const uint4*>(l8);
  }
}

// base kernels fp32 [B][Cout][Cin][9] -> SW128 bf16 tiles [b][ct][t][chunk][part][128 co][64 ci]
// (part 0 = hi, 1 = lo) for bf16x3, plus a hi-only copy [b][ct][t][chunk] for bf16 so that
// every W stage is one contiguous bulk copy in both precisions.
__global__ void w_pack_kernel(const float* __restrict__ bases, uint8_t* __restrict__ w,
                              uint8_t* __restrict__ whi, int NB, int Cout, int Cin, int NCT, int NC) {
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
    const size_t off = (size_t)tile * 2 * WTILE + sw128_offset(col, g * 8);  // [tile][part]
    *reinterpret_cast<uint4*>(w + off) = *reinterpret_cast<const uint4*>(h8);
    *reinterpret_cast<uint4*>(w + off + WTILE) = *reinterpret_cast<const uint4*>(l8);
    *reinterpret_cast<uint4*>(whi + (size_t)tile * WTILE + sw128_offset(col, g * 8)) =
        *reinterpret_cast<const uint4*>(h8);
  }
}

struct TcGeom {
  int gi;       // geometry: 0 = TW 16, 2 = strips, 3 = 8x8 images, 4 = 4x4 images
  int units;    // band owners: images, or bands of IMGS small images
  int NBK, NC, NCT, xtile;
  size_t x_plane, w_plane;
};
TcGeom geom(const rc_desc& d) {
  TcGeom g;
  // W = 32 runs as two 4x16 strips per 4 rows (N = 112, 1.69 input px per output px); 2-row
  // bands (N = 128, 2.0) were 5-8% slower on C4 (profiles/r01/strip32.txt)
  g.gi = d.w == 16 ? 0 : (d.w == 8 && d.h == 8) ? 3 : (d.w == 4 && d.h == 4) ? 4 : 2;
  static const int out_rows_of[5] = {Geo<16>::OUT_ROWS, 0, Geo<0>::OUT_ROWS, 8, 4};
  static const int xtile_of[5] = {Geo<16>::XTILE, 0, Geo<0>::XTILE, Geo<8>::XTILE, Geo<4>::XTILE};
  g.xtile = xtile_of[g.gi];
  g.units = g.gi == 3 ? d.n : (g.gi == 4 ? (d.n + 3) / 4 : d.n);
  g.NBK = g.gi >= 3 ? 1 : (d.h + out_rows_of[g.gi] - 1) / out_rows_of[g.gi] * (g.gi == 2 ? d.w / 16 : 1);
  g.NC = (d.c_in + KC - 1) / KC;
  g.NCT = (d.c_out + 127) / 128;
  g.x_plane = (size_t)g.units * g.NBK * g.NC * g.xtile;
  g.w_plane = (size_t)num_bases(d) * g.NCT * 9 * g.NC * WTILE;
  return g;
}

struct SmemPlan {
  int spc, stages, xstream;
  size_t bytes;
};
// Preferred: one resident X band (per-chunk barriers overlap its reload with the last taps)
// plus a W ring of single-chunk stages (one chunk = one tap's 64 input channels, hi + lo)
// as deep as shared memory allows: with two MMA warps working on consecutive taps, small
// stages let the next tap's chunks land as the current tap frees its slots.  When the band
// does not fit (large Cin), X chunks are streamed with the W stages instead (X re-read from
// L2 once per tap).
SmemPlan smem_plan(const TcGeom& g, int parts) {
  SmemPlan sp{0, 0, 0, 0};
  const size_t cap = 232448 - 1024 - 1024;  // dynamic smem minus alignment slack / statics
  const size_t xt = g.xtile;
  const size_t xbuf = (size_t)parts * g.NC * xt;
  const size_t chunk = (size_t)parts * WTILE;
  if (g.NC <= MAX_NC && xbuf < cap) {
    const size_t budget = cap - xbuf;
    // the two MMA warps each own a ring of >= 2 stages: the largest stage (the TMA engine's
    // per-copy cost favours big copies, profiles/r01/wstage_ab.txt) for which 4 stages fit,
    // then as many stages as fit; single-chunk stages, >= 1 per ring, at the least
    for (int c = g.NC; c >= 1; --c) {
      if (g.NC % c) continue;
      const size_t sb = c * chunk;
      const size_t n = budget / sb;
      if (n >= 4 || (c == 1 && n >= 2)) {
        sp.spc = c;
        sp.stages = n > MAX_STAGES ? MAX_STAGES : (int)n;
        sp.bytes = xbuf + sp.stages * sb + 1024;
        return sp;
      }
    }
  }
  const size_t schunk = (size_t)parts * (WTILE + xt);
  for (int c = 1; c <= g.NC; ++c) {
    if (g.NC % c) continue;
    const size_t sb = c * schunk;
    if (4 * sb <= cap || (c == 1 && 2 * sb <= cap)) {
      sp.spc = c;
      sp.stages = (int)(cap / sb) > MAX_STAGES ? MAX_STAGES : (int)(cap / sb);
      sp.xstream = 1;
      sp.bytes = sp.stages * sb + 1024;
      return sp;
    }
  }
  return sp;
}

}  // namespace

namespace {
bool band_supported(const rc_desc& d) {
  const int gf = pool_fold(d);
  const int R = d.orientations;
  const bool fold_ok = d.pool == RC_POOL_NONE || (d.pool == RC_POOL_AVG && (R & (R - 1)) == 0) || gf == 1 ||
                       gf == 2 || gf % 4 == 0;
  const bool geom_ok = d.w == 16 || d.w == 32 || (d.w >= 48 && d.w % 16 == 0) || (d.w == 8 && d.h == 8) ||
                       (d.w == 4 && d.h == 4);
  if (!(d.k == 3 && geom_ok && fold_ok &&
        (d.precision == RC_PREC_BF16 || d.precision == RC_PREC_BF16X3 || d.precision == RC_PREC_AUTO)))
    return false;
  const int parts = d.precision == RC_PREC_BF16 ? 1 : 2;
  return smem_plan(geom(d), parts).spc > 0;
}
}  // namespace

// single orientation: implicit GEMM (ri_igemm.cu); otherwise the band kernels of this file
bool tc_supported(const rc_desc& d) { return igemm_supported(d) || band_supported(d); }
size_t tc_bank_bytes(const rc_desc& d) {
  if (d.k != 3) return 0;
  return 3 * geom(d).w_plane;  // interleaved hi/lo + hi-only
}
size_t tc_workspace_bytes(const rc_desc& d) {
  if (igemm_supported(d)) return igemm_workspace_bytes(d);
  if (!band_supported(d)) return 0;
  return 2 * geom(d).x_plane;
}

int launch_tc_wpack(const rc_desc& d, const float* bases, uint8_t* tc_section, cudaStream_t s) {
  const TcGeom g = geom(d);
  const long long total = (long long)num_bases(d) * g.NCT * 9 * g.NC * 128 * (KC / 8);
  long long grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  w_pack_kernel<<<(int)grid, 256, 0, s>>>(bases, tc_section, tc_section + 2 * g.w_plane, num_bases(d), d.c_out,
                                         d.c_in, g.NCT, g.NC);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

int launch_tc(const rc_desc& d, const float* x, const void* bank, const float* bias, float* y, uint8_t* am,
              void* ws, size_t ws_bytes, cudaStream_t s, bool dry_run, const char** name) {
  if (igemm_supported(d)) {
    if (name) *name = d.precision == RC_PREC_BF16 ? "tc_igemm_bf16" : "tc_igemm_bf16x3";
    if (dry_run || d.n == 0) return RC_OK;
    if (ws_bytes < igemm_workspace_bytes(d) || ws == nullptr)
      return fail(RC_ERR_WORKSPACE, "ri_conv: workspace too small for the tensor-core path");
    const uint8_t* tcb = static_cast<const uint8_t*>(bank) + bank_layout(d).tc_off;
    return launch_igemm(d, x, tcb, tcb + 2 * geom(d).w_plane, bias, y, am, ws, s);
  }
  if (!band_supported(d)) return RC_ERR_UNSUPPORTED;
  if (name) {
    static const char* names[5][2] = {{"tc_k3w16_bf16x3", "tc_k3w16_bf16"},
                                      {"", ""},
                                      {"tc_k3strip_bf16x3", "tc_k3strip_bf16"},
                                      {"tc_k3img8_bf16x3", "tc_k3img8_bf16"},
                                      {"tc_k3img4_bf16x3", "tc_k3img4_bf16"}};
    *name = names[geom(d).gi][d.precision == RC_PREC_BF16];
  }
  if (dry_run || d.n == 0) return RC_OK;
  const TcGeom g = geom(d);
  if (ws_bytes < tc_workspace_bytes(d) || ws == nullptr)
    return fail(RC_ERR_WORKSPACE, "ri_conv: workspace too small for the tensor-core path");
  const int passes = d.precision == RC_PREC_BF16 ? 1 : 3;
  const int parts = passes == 3 ? 2 : 1;
  uint8_t* xh = static_cast<uint8_t*>(ws);
  uint8_t* xl = passes == 3 ? xh + g.x_plane : nullptr;
  const int gi = g.gi;
  const dim3 pgrid(g.NC, g.NBK, g.units);
  switch (gi) {
    case 0: x_pack_kernel<16><<<pgrid, 256, 0, s>>>(x, xh, xl, d.c_in, d.h, d.w, g.NBK, g.NC, d.n); break;
    case 2: x_pack_kernel<0><<<pgrid, 256, 0, s>>>(x, xh, xl, d.c_in, d.h, d.w, g.NBK, g.NC, d.n); break;
    case 3: x_pack_kernel<8><<<pgrid, 256, 0, s>>>(x, xh, xl, d.c_in, d.h, d.w, g.NBK, g.NC, d.n); break;
    default: x_pack_kernel<4><<<pgrid, 256, 0, s>>>(x, xh, xl, d.c_in, d.h, d.w, g.NBK, g.NC, d.n); break;
  }
  RC_CUDA(cudaGetLastError());
  const BankLayout L = bank_layout(d);
  const uint8_t* tcb = static_cast<const uint8_t*>(bank) + L.tc_off;
  const SmemPlan plan = smem_plan(g, parts);
  TcParams p;
  p.xh = xh;
  p.xl = xl;
  p.w = passes == 3 ? tcb : tcb + 2 * g.w_plane;
  p.bias = bias;
  p.y = y;
  p.am = (d.pool == RC_POOL_MAX || d.pool == RC_POOL_SUBGROUP) ? am : nullptr;
  p.N = d.n;
  p.H = d.h;
  p.W = d.w;
  p.Cout = d.c_out;
  p.NB = num_bases(d);
  p.NBK = g.NBK;
  p.NC = g.NC;
  p.NCT = g.NCT;
  p.pool = d.pool;
  p.gf = pool_fold(d);
  p.RO = out_orientations(d);
  p.passes = passes;
  p.inv_r = 1.0f / (float)d.orientations;
  p.act = d.activation;
  p.w_stages = plan.stages;
  p.spc = plan.spc;
  p.xstream = plan.xstream;
  p.items = g.NCT * g.units;
  int dev, sms;
  RC_CUDA(cudaGetDevice(&dev));
  RC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // [geometry][single][convention][bf16x3]
#define RC_TC_K(TW, RPB, CONV) {ri_tc_kernel<TW, RPB, CONV, false>, ri_tc_kernel<TW, RPB, CONV, true>}
  static void (*const kernels[5][2][2][2])(TcParams) = {
      {{RC_TC_K(16, 4, 0), RC_TC_K(16, 4, 1)}, {RC_TC_K(16, 1, 0), RC_TC_K(16, 1, 1)}},
      {{{nullptr, nullptr}, {nullptr, nullptr}}, {{nullptr, nullptr}, {nullptr, nullptr}}},
      {{RC_TC_K(0, 4, 0), RC_TC_K(0, 4, 1)}, {RC_TC_K(0, 1, 0), RC_TC_K(0, 1, 1)}},
      {{RC_TC_K(8, 4, 0), RC_TC_K(8, 4, 1)}, {RC_TC_K(8, 1, 0), RC_TC_K(8, 1, 1)}},
      {{RC_TC_K(4, 4, 0), RC_TC_K(4, 4, 1)}, {RC_TC_K(4, 1, 0), RC_TC_K(4, 1, 1)}}};
#undef RC_TC_K
  const int single = d.group == RC_GROUP_SINGLE, raw = d.convention == RC_CONV_RAW;
  void (*fn)(TcParams) = kernels[gi][single][raw][passes == 3];
  RC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.bytes));
  const int grid = p.items < sms ? p.items : sms;
  prof_begin(s);
  static const int threads_of[5] = {Epi<16>::THREADS, 0, Epi<0>::THREADS, Epi<8>::THREADS, Epi<4>::THREADS};
  static const int budget_of[5] = {128 * Epi<16>::PROD + 32 * Epi<16>::WARPS * Epi<16>::REGS, 0,
                                   128 * Epi<0>::PROD + 32 * Epi<0>::WARPS * Epi<0>::REGS,
                                   128 * Epi<8>::PROD + 32 * Epi<8>::WARPS * Epi<8>::REGS,
                                   128 * Epi<4>::PROD + 32 * Epi<4>::WARPS * Epi<4>::REGS};
  cudaFuncAttributes fa;
  RC_CUDA(cudaFuncGetAttributes(&fa, fn));
  if (fa.numRegs * threads_of[gi] < budget_of[gi])  // setmaxnreg.inc would never be granted
    return fail(RC_ERR_CUDA, "ri_conv: tensor-core kernel register budget exceeds its launch allocation");
  fn<<<grid, threads_of[gi], plan.bytes, s>>>(p);
  prof_end(s);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

#if RC_TC_PROF
extern "C" int rc_tc_prof(unsigned long long* host, int n, int reset) {
  if (host && n > 0) RC_CUDA(cudaMemcpyFromSymbol(host, g_tc_prof, sizeof(unsigned long long) * (size_t)n));
  if (reset) {
    static unsigned long long zeros[1024 * 32];
    RC_CUDA(cudaMemcpyToSymbol(g_tc_prof, zeros, sizeof(zeros)));
  }
  return RC_OK;
}
#endif

}  // namespace rc
