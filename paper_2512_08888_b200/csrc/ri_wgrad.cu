// ri_wgrad.cu -- weight gradient of the K=3 RI layer on tcgen05 (SPEC backward, Eq. 13-16).
//
// The backward pass needs, per unpooled slice m = (co, o) and per input channel ci and
// gather position pos = (i, j) of the 3x3 window,
//   dF[m][ci*9 + pos] = sum_n sum_p  G[n][m][p] * X[n][ci][p + (i-1, j-1)]
// (G = the pool/ReLU-backward gradient of the slices; then backward.cu's param_grad_kernel
// applies the inverse rotations, Eq. 16, and the mirror / steer chain rule).  The previous
// path was im2col + an FP32 SGEMM per image.  Here it is one implicit GEMM over all pixels
// of the batch (K = padded pixels q), with the 3x3 shift applied as a ROW offset of an
// MN-major operand:
//   A = G tile  [128 m x 64 q]  K-major SW128 (packed here from G, zero at the pad ring)
//   B = X rows  [64 q (+halo) x 64 ci]  MN-major SW128 -- exactly the implicit-GEMM forward's
//       padded X planes (ri_igemm.cu); tap pos reads rows shifted by (i-1)*(W+2) + (j-1)
//   D = [128 m x 64 ci] per tap, 5 or 4 taps per work item (TMEM 320 columns)
// A descriptor may start at any 128-byte row of an SW128 tile in K-major AND MN-major form
// (tools/shift_probe.cu, profiles/r01/igemm/).  bf16x3 (hi/lo of both operands, 3 products)
// keeps the FP32-class tolerance of the layer's precision; "bf16" uses one product.
//
// Work item = (m tile, ci chunk, tap group, K split).  Small layers (few m tiles) split K
// and reduce the partial dF deterministically in a second kernel.
#include <cuda_bf16.h>

#include <cstdlib>

#include "rc_internal.cuh"
#include "tc_ptx.cuh"

namespace rc {
namespace {

using namespace tc;

constexpr int KQ = 64;                  // q per K chunk (one SW128 K-major row of A)
constexpr int ATILE = 128 * KQ * 2;     // 16 KB: [128 m x 64 q] bf16
constexpr int EPI_WARPS = 4;
constexpr int THREADS = 32 * (4 + EPI_WARPS);
constexpr int MAX_STAGES = 6;

struct WgParams {
  const uint8_t* gp;  // packed G: [mt][kc][part][128 m][64 q]
  const uint8_t* xh;  // padded X planes [c][rows][64 ci] (hi)
  const uint8_t* xl;  // lo plane or null
  float* out;         // dF, or the split partials [split][M][Ncol]
  long long xrows_plane;
  int M, MT, Cin, NCc, KC, splits, per, items, parts, passes, stages, xr, G, Wp;
  int nci;            // X planes (64 ci each) per work item: 2 -> N = 128 (MN atoms LBO apart)
  int tgs, ntg;       // taps per group, tap groups (N=64: 5 + 4, N=128: 3 + 3 + 3)
  int off[9];         // row offset of gather position pos
};

__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// G [n][M][H][W] fp32 -> Gp[mt][kc][part][128 m][64 q] over the padded pixel grid (pads 0).
// Thread = (m, kc, 8-q group): 8 threads fill one 128-byte row; a warp reads 256
// consecutive q of one m (coalesced), decoding (n, h, w) once and stepping after that.
template <typename IT>  // index type: 32-bit divisions when the packed G allows it
__global__ void __launch_bounds__(256) g_pack_kernel(const float* __restrict__ g, uint8_t* __restrict__ gp, int M,
                                                     int MT, int KC, int H, int W, int Wp, int Pimg, long long QN,
                                                     int parts) {
  const IT total = (IT)((long long)MT * 128 * KC * 8);
  const size_t plane = (size_t)H * W;
  for (IT i = blockIdx.x * (IT)blockDim.x + threadIdx.x; i < total; i += (IT)gridDim.x * blockDim.x) {
    const int grp = (int)(i % 8);
    const IT kc = (i / 8) % (IT)KC;
    const IT m = i / (8 * (IT)KC);
    const int mt = (int)(m / 128), ml = (int)(m % 128);
    const IT q = kc * KQ + grp * 8;
    int n = (int)(q / (IT)Pimg), rem = (int)(q - (IT)n * (IT)Pimg);
    int hp = rem / Wp, wp = rem - hp * Wp;
    // addresses first (the pixel walk is sequential), then 8 independent loads in flight
    long long src[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      src[j] = ((long long)m < M && (long long)q + j < QN && hp >= 1 && hp <= H && wp >= 1 && wp <= W)
                   ? ((long long)n * M + (long long)m) * (long long)plane + (long long)(hp - 1) * W + (wp - 1)
                   : -1;
      if (++wp == Wp) {
        wp = 0;
        if (++hp == H + 2) {
          hp = 0;
          ++n;
        }
      }
    }
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = src[j] >= 0 ? __ldg(g + src[j]) : 0.f;
    __align__(16) __nv_bfloat16 h8[8], l8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) split_bf16(v[j], h8[j], l8[j]);
    const size_t tile = ((size_t)mt * KC + kc) * parts;
    const size_t off = (size_t)ml * 128 + (size_t)((grp ^ (ml & 7)) << 4);
    *reinterpret_cast<uint4*>(gp + tile * ATILE + off) = *reinterpret_cast<const uint4*>(h8);
    if (parts == 2) *reinterpret_cast<uint4*>(gp + (tile + 1) * ATILE + off) = *reinterpret_cast<const uint4*>(l8);
  }
}

__global__ void split_reduce_kernel(const float* __restrict__ part, float* __restrict__ out, long long n, int splits) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < splits; ++s) a += part[(size_t)s * n + i];  // fixed order: deterministic
    out[i] = a;
  }
}

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

struct Item {
  int mt, cc, tg, split, k0, k1, t0, nt;
};
__device__ __forceinline__ Item decode(const WgParams& p, int item) {
  Item it;
  it.split = item % p.splits;
  int r = item / p.splits;
  it.tg = r % p.ntg;
  r /= p.ntg;
  it.cc = r % p.NCc;
  it.mt = r / p.NCc;
  it.k0 = it.split * p.per;  // host: splits = ceil(KC / per), so no split is empty
  it.k1 = min(p.KC, it.k0 + p.per);
  it.t0 = it.tg * p.tgs;
  it.nt = min(p.tgs, 9 - it.t0);
  return it;
}

__global__ void __launch_bounds__(THREADS, 1) wgrad_kernel(const __grid_constant__ WgParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[MAX_STAGES], empty[MAX_STAGES], d_full, d_empty;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t XB = (uint32_t)p.xr * 128;            // bytes of one X plane block per stage
  const uint32_t XP = p.nci * XB;                      // one part (hi or lo): nci plane blocks
  const uint32_t stage = p.parts * (ATILE + XP);
  if (threadIdx.x == 0) {
    for (int i = 0; i < MAX_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&d_full, 1);
    mbar_init(&d_empty, EPI_WARPS);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    Ring r;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      const Item it = decode(p, item);
      for (int kc = it.k0; kc < it.k1; ++kc) {
        if (r.used) mbar_wait(&empty[r.s], r.ph ^ 1);
        if (elect_one()) {
          uint8_t* dst = sm + r.s * stage;
          mbar_arrive_expect_tx(&full[r.s], stage);
          bulk_g2s(dst, p.gp + ((size_t)it.mt * p.KC + kc) * p.parts * ATILE, p.parts * ATILE, &full[r.s]);
          const long long r0 = ((long long)p.G + (long long)kc * KQ - p.Wp - 1) & ~7LL;
          for (int pl = 0; pl < p.nci; ++pl) {
            const size_t src = ((size_t)(it.cc * p.nci + pl) * p.xrows_plane + r0) * 128;
            bulk_g2s(dst + p.parts * ATILE + pl * XB, p.xh + src, XB, &full[r.s]);
            if (p.parts == 2) bulk_g2s(dst + p.parts * ATILE + XP + pl * XB, p.xl + src, XB, &full[r.s]);
          }
        }
        __syncwarp();
        r.adv(p.stages);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t NT = 64 * p.nci;
    const uint32_t idesc = idesc_bf16_f32(128, NT) | (1u << 16);  // B (X rows) MN-major
    // MN-major B: the second 64-ci atom lies XB bytes after the first (leading-byte offset)
    const uint64_t lbo = (uint64_t)(((p.nci == 2 ? XB : 16) >> 4) & 0x3FFF) << 16;
    auto bdesc = [&](uint32_t a) { return (desc_k_sw128(a) & ~(0x3FFFull << 16)) | lbo; };
    Ring r;
    int n_items = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++n_items) {
      const Item it = decode(p, item);
      if (n_items > 0) mbar_wait(&d_empty, (n_items - 1) & 1);
      tc_fence_after();
      for (int kc = it.k0; kc < it.k1; ++kc) {
        mbar_wait(&full[r.s], r.ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t base = smem_u32(sm + r.s * stage);
          const uint64_t gh = desc_k_sw128(base), gl = desc_k_sw128(base + ATILE);
          const long long r0 = ((long long)p.G + (long long)kc * KQ - p.Wp - 1) & ~7LL;
          const uint32_t row0 = (uint32_t)(p.G + (long long)kc * KQ - r0);
          const uint32_t xb = base + p.parts * ATILE;
          for (int tt = 0; tt < it.nt; ++tt) {
            const uint32_t d = tmem + tt * NT;
            const uint32_t xrow = (row0 + p.off[it.t0 + tt]) * 128;
            const uint64_t xh = bdesc(xb + xrow), xl = bdesc(xb + XP + xrow);
            const uint32_t acc0 = kc != it.k0;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, gh + 2 * kk, xh + (uint64_t)(kk * 128), idesc, acc0 | kk);
            if (p.passes == 3) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, gh + 2 * kk, xl + (uint64_t)(kk * 128), idesc, 1);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, gl + 2 * kk, xh + (uint64_t)(kk * 128), idesc, 1);
            }
          }
          mma_commit(&empty[r.s]);
          if (kc == it.k1 - 1) mma_commit(&d_full);
        }
        __syncwarp();
        r.adv(p.stages);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int qd = warp % 4;
    const int Ncol = p.Cin * 9;
    int n_items = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++n_items) {
      const Item it = decode(p, item);
      mbar_wait(&d_full, n_items & 1);
      tc_fence_after();
      const int m = it.mt * 128 + qd * 32 + lane;
      float* dst = p.out + (size_t)it.split * p.M * Ncol + (size_t)m * Ncol;
      const int NT = 64 * p.nci;
      for (int tt = 0; tt < it.nt; ++tt) {
        const int pos = it.t0 + tt;
        for (int c0 = 0; c0 < NT; c0 += 16) {
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + tt * NT + c0, v);
          tmem_wait_ld();
          if (m < p.M) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int ci = it.cc * NT + c0 + j;
              if (ci < p.Cin) dst[(size_t)ci * 9 + pos] = v[j];
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

struct WgGeom {
  int M, MT, NCc, KC, xr, parts, splits, per, stages, nci, tgs, ntg;
  long long QN;
  size_t gp_bytes, x_bytes, part_bytes, smem;
};
WgGeom wg_geom(const rc_desc& d) {
  WgGeom g{};
  const PadGeom pg = pad_geom(d);
  g.M = d.c_out * num_bases(d) * rot_per_base(d);
  g.MT = (g.M + 127) / 128;
  // 128-ci tiles (N = 128: math-bound MMAs, 3 taps x 128 TMEM columns) when the planes pair
  // up, else 64-ci tiles (N = 64: shared-memory bound, 5 + 4 taps); RC_WGRAD_N=64 forces 64
  g.nci = pg.NC % 2 == 0 ? 2 : 1;  // 128-ci tiles where Cin allows (profiles/r01/bwd_wgrad_ab.txt)
  g.parts = d.precision == RC_PREC_BF16 ? 1 : 2;
  g.xr = (KQ + 2 * (pg.Wp + 1) + 7 + 7) / 8 * 8;
  const size_t cap0 = 232448 - 1024 - 512;
  if (g.nci == 2 && cap0 / ((size_t)g.parts * (ATILE + 2 * (size_t)g.xr * 128)) < 2) g.nci = 1;  // wide images
  g.tgs = g.nci == 2 ? 3 : 5;
  g.ntg = (9 + g.tgs - 1) / g.tgs;
  g.NCc = pg.NC / g.nci;
  g.QN = (long long)d.n * pg.Pimg;
  g.KC = (int)((g.QN + KQ - 1) / KQ);
  g.xr = (KQ + 2 * (pg.Wp + 1) + 7 + 7) / 8 * 8;
  g.parts = d.precision == RC_PREC_BF16 ? 1 : 2;
  const int base = g.MT * g.NCc * g.ntg;
  int sp = (296 + base - 1) / base;
  const int maxsp = g.KC / 16 > 1 ? g.KC / 16 : 1;
  sp = sp < 1 ? 1 : (sp > maxsp ? maxsp : sp);
  g.per = g.KC > 0 ? (g.KC + sp - 1) / sp : 1;
  g.splits = g.KC > 0 ? (g.KC + g.per - 1) / g.per : 1;
  const size_t stage = (size_t)g.parts * (ATILE + (size_t)g.nci * g.xr * 128);
  const size_t cap = 232448 - 1024 - 512;
  g.stages = (int)(cap / stage) > MAX_STAGES ? MAX_STAGES : (int)(cap / stage);
  g.smem = (size_t)g.stages * stage + 1024;
  g.gp_bytes = (size_t)g.MT * g.KC * g.parts * ATILE;
  g.x_bytes = pad_planes_bytes(d, g.parts);
  g.part_bytes = g.splits > 1 ? (size_t)g.splits * g.M * d.c_in * 9 * sizeof(float) : 0;
  return g;
}

size_t al256(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace

bool wgrad_supported(const rc_desc& d) {
  if (d.k != 3 || d.precision == RC_PREC_FP32) return false;
  return wg_geom(d).stages >= 2;
}

size_t wgrad_ws_bytes(const rc_desc& d) {
  const WgGeom g = wg_geom(d);
  return al256(g.gp_bytes) + al256(g.x_bytes) + al256(g.part_bytes);
}

int launch_wgrad(const rc_desc& d, const float* x, const float* df, float* dF, void* ws, cudaStream_t s) {
  const WgGeom g = wg_geom(d);
  const PadGeom pg = pad_geom(d);
  uint8_t* gp = static_cast<uint8_t*>(ws);
  uint8_t* xh = gp + al256(g.gp_bytes);
  uint8_t* xl = g.parts == 2 ? xh + (size_t)pg.NC * pg.rows * 128 : nullptr;
  float* part = reinterpret_cast<float*>(xh + al256(g.x_bytes));
  int st = launch_pad_pack(d, x, xh, xl, s);
  if (st != RC_OK) return st;
  {
    const long long total = (long long)g.MT * 128 * g.KC * 8;
    const long long grid = total / 256 + 1 < 148 * 32 ? total / 256 + 1 : 148 * 32;
    if (total < (1LL << 31) && g.QN + KQ < (1LL << 31))
      g_pack_kernel<unsigned><<<(int)grid, 256, 0, s>>>(df, gp, g.M, g.MT, g.KC, d.h, d.w, pg.Wp, pg.Pimg, g.QN, g.parts);
    else
      g_pack_kernel<unsigned long long><<<(int)grid, 256, 0, s>>>(df, gp, g.M, g.MT, g.KC, d.h, d.w, pg.Wp, pg.Pimg,
                                                                  g.QN, g.parts);
    RC_CUDA(cudaGetLastError());
  }
  WgParams p;
  p.gp = gp;
  p.xh = xh;
  p.xl = xl;
  p.out = g.splits > 1 ? part : dF;
  p.xrows_plane = pg.rows;
  p.M = g.M;
  p.MT = g.MT;
  p.Cin = d.c_in;
  p.NCc = g.NCc;
  p.KC = g.KC;
  p.splits = g.splits;
  p.per = g.per;
  p.nci = g.nci;
  p.tgs = g.tgs;
  p.ntg = g.ntg;
  p.items = g.MT * g.NCc * g.ntg * g.splits;
  p.parts = g.parts;
  p.passes = g.parts == 2 ? 3 : 1;
  p.stages = g.stages;
  p.xr = g.xr;
  p.G = pg.G;
  p.Wp = pg.Wp;
  for (int pos = 0; pos < 9; ++pos) p.off[pos] = (pos / 3 - 1) * pg.Wp + (pos % 3 - 1);
  int dev, sms;
  RC_CUDA(cudaGetDevice(&dev));
  RC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RC_CUDA(cudaFuncSetAttribute(wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
  const int grid = p.items < sms ? p.items : sms;
  wgrad_kernel<<<grid, THREADS, g.smem, s>>>(p);
  RC_CUDA(cudaGetLastError());
  if (g.splits > 1) {
    const long long n = (long long)g.M * d.c_in * 9;
    const long long blocks = n / 256 + 1 < 148 * 8 ? n / 256 + 1 : 148 * 8;
    split_reduce_kernel<<<(int)blocks, 256, 0, s>>>(part, dF, n, g.splits);
    RC_CUDA(cudaGetLastError());
  }
  return RC_OK;
}

}  // namespace rc
