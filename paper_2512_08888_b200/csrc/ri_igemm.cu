// ri_igemm.cu -- single-orientation K=3 convolution (group "single", R = 1) as an implicit
// GEMM on tcgen05 (sm_100a).
//
// R = 1 has no rotation reuse to exploit (SPEC:274-282 degenerates to one slice), so the
// scatter-epilogue design of ri_tc.cu (Z per tap in TMEM, CUDA-core scatter, 1.5x halo
// recompute) is the wrong shape for it.  Here every tap is a SHIFTED VIEW of one operand:
//   Y[px, co] = sum_t sum_ci X[px + off_t, ci] * K_t[co, ci]       off_t = di_t * Wp + dj_t
// with X stored zero-padded, (H+2) x (W+2) pixels per image, images back to back, one
// 128-byte SW128 row per pixel (64 ci of bf16).  A tcgen05 shared-memory descriptor may start
// at ANY 128-byte row of a 1024-byte-aligned SW128 tile (the swizzle follows the absolute
// address; measured, tools/shift_probe.cu), so the 9 taps are 9 descriptor offsets into one
// staged X tile and all 9 x Cin/16 (x3 for bf16x3) MMAs accumulate into the same TMEM tile.
// The epilogue reads the finished tile once: bias + activation + store.  No halo recompute
// (only the zero pad rows / columns of the padded grid: 6% at 64x64, 27% at 16x16).
//
//   A = X tile   [128 padded pixels x 64 ci]  (M = 128)
//   B = K_t tile [N co x 64 ci]               (N = Cout rounded to 32, <= 256)
//   D = 128 lanes (pixels) x N columns (co), double-buffered in TMEM (2 x N <= 512)
// The weights are ri_tc.cu's packed tiles (bank tc section, [ct][t][c][part] of 128 co);
// the tap -> (di, dj) map is convention P1's for rotation 0 (slice_tap_offsets).
//
// Persistent CTA, 12 warps: warp 0 producer (bulk copies: X chunk tiles incl. the +-(Wp+1)
// row halo, K_t stages), warp 1 MMA issuer, warps 4-11 epilogue (TMEM lane quadrant
// warp % 4 = pixels, column half (warp - 4) / 4).  Work item = (pixel tile, co tile).
#include <cuda_bf16.h>

#include <cstdlib>

#include "k3_tables.cuh"
#include "rc_internal.cuh"
#include "tc_ptx.cuh"

namespace rc {
namespace {

using namespace tc;

constexpr int KC = 64;                 // ci per chunk
constexpr int WTILE = 128 * KC * 2;    // packed weight tile [128 co x 64 ci] bf16 (ri_tc.cu)
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 32 * (4 + EPI_WARPS);
constexpr int MAX_WSTAGES = 8;

struct IgParams {
  const uint8_t* xh;  // padded X planes [c][rows][128 B] (hi), SW128 rows
  const uint8_t* xl;  // lo plane (bf16x3) or null
  const uint8_t* w;   // packed weights: [tile][part] (bf16x3) or [tile] (bf16, hi plane)
  const float* bias;
  float* y;
  uint8_t* am;        // argmax (R = 1: all zero) or null
  long long rows;     // rows per chunk plane
  int N, H, W, Cout, NC, NCTW, NN, NCTN, tiles, items;
  int Wp, G, Pimg, xrows, parts, passes, x_stages, w_stages, act;
  int off[9];         // A row shift of base tap t
  int seg;            // ci chunks per TMEM accumulation segment
};

__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// fp32 NCHW -> padded SW128 planes.  A block owns PACK_ROWS consecutive plane rows of one
// ci chunk: phase 1 reads [64 ci x PACK_ROWS px] with consecutive threads on consecutive
// pixels (coalesced fp32 reads, zero for pad / guard rows) into shared memory; phase 2
// writes whole 128-byte rows (8 threads per row, 16 B each: coalesced, swizzled).
constexpr int PACK_ROWS = 64;
__global__ void __launch_bounds__(256) ig_pack_kernel(const float* __restrict__ x, uint8_t* __restrict__ xh,
                                                      uint8_t* __restrict__ xl, int N, int Cin, int H, int W, int Wp,
                                                      int G, int Pimg, long long rows, int NC) {
  __shared__ float tile[PACK_ROWS][KC + 1];
  const long long blocks_per_chunk = (rows + PACK_ROWS - 1) / PACK_ROWS;
  for (long long blk = blockIdx.x; blk < blocks_per_chunk * NC; blk += gridDim.x) {
    const int c = (int)(blk / blocks_per_chunk);
    const long long g0 = (blk % blocks_per_chunk) * PACK_ROWS;
    {  // thread = one pixel row r of the block (its source pixel decoded once), 16 channels
      const int r = threadIdx.x % PACK_ROWS;
      const long long q = g0 + r - G;
      const float* src = nullptr;
      if (q >= 0 && q < (long long)N * Pimg) {
        const int n = (int)(q / Pimg), rem = (int)(q - (long long)n * Pimg);
        const int hp = rem / Wp, h = hp - 1, w = rem - hp * Wp - 1;
        if (h >= 0 && h < H && w >= 0 && w < W) src = x + ((size_t)n * Cin + c * KC) * H * W + (size_t)h * W + w;
      }
      const size_t cs = (size_t)H * W;
      const int cl0 = threadIdx.x / PACK_ROWS, nval = Cin - c * KC;  // 256 threads: 4 x 16 channels
      float v[KC / 4];
#pragma unroll
      for (int i = 0; i < KC / 4; ++i) {  // all 16 loads in flight before the smem stores
        const int cl = cl0 + 4 * i;
        v[i] = (src && cl < nval) ? __ldg(src + cl * cs) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < KC / 4; ++i) tile[r][cl0 + 4 * i] = v[i];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < PACK_ROWS * 8; e += blockDim.x) {
      const int r = e / 8, grp = e % 8;
      const long long g = g0 + r;
      if (g < rows) {
        __align__(16) __nv_bfloat16 h8[8], l8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) split_bf16(tile[r][grp * 8 + j], h8[j], l8[j]);
        const size_t off = ((size_t)c * rows + g) * 128 + (size_t)((grp ^ (int)(g & 7)) << 4);
        *reinterpret_cast<uint4*>(xh + off) = *reinterpret_cast<const uint4*>(h8);
        if (xl) *reinterpret_cast<uint4*>(xl + off) = *reinterpret_cast<const uint4*>(l8);
      }
    }
    __syncthreads();
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

__global__ void __launch_bounds__(THREADS, 1) igemm_kernel(const __grid_constant__ IgParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t x_full[2], x_empty[2], w_full[MAX_WSTAGES], w_empty[MAX_WSTAGES];
  __shared__ __align__(8) uint64_t d_full[2], d_empty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t XS = (uint32_t)p.xrows * 128;   // bytes per part of an X stage
  const uint32_t xstage = p.parts * XS;
  const uint32_t WS = (uint32_t)p.NN * 128;      // bytes per part of a weight stage
  const uint32_t wstage = p.parts * WS;
  uint8_t* xs = sm;
  uint8_t* ws = sm + p.x_stages * xstage;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], EPI_WARPS);
    }
    for (int i = 0; i < MAX_WSTAGES; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const int S = p.w_stages;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    Ring xr, wr;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      const int tile = item / p.NCTN, ct = item % p.NCTN;
      const long long r0 = ((long long)p.G + (long long)tile * 128 - p.Wp - 1) & ~7LL;
      const int wt0 = ct * p.NN / 128;             // first packed 128-co weight tile
      const int rows0 = p.NN < 128 ? p.NN : 128;   // rows taken from it
      const int rows1 = (p.NN > 128 && wt0 + 1 < p.NCTW) ? p.NN - 128 : 0;
      for (int c = 0; c < p.NC; ++c) {
        if (xr.used) mbar_wait(&x_empty[xr.s], xr.ph ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&x_full[xr.s], p.parts * XS);
          const size_t src = ((size_t)c * p.rows + r0) * 128;
          bulk_g2s(xs + xr.s * xstage, p.xh + src, XS, &x_full[xr.s]);
          if (p.parts == 2) bulk_g2s(xs + xr.s * xstage + XS, p.xl + src, XS, &x_full[xr.s]);
        }
        __syncwarp();
        xr.adv(p.x_stages);
        for (int t = 0; t < 9; ++t) {
          if (wr.used) mbar_wait(&w_empty[wr.s], wr.ph ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&w_full[wr.s], p.parts * (rows0 + rows1) * 128);
            uint8_t* dst = ws + wr.s * wstage;
            for (int part = 0; part < p.parts; ++part) {
              const size_t t0 = ((size_t)wt0 * 9 + t) * p.NC + c;
              const size_t t1 = ((size_t)(wt0 + 1) * 9 + t) * p.NC + c;
              const size_t s0 = p.parts == 2 ? (t0 * 2 + part) * WTILE : t0 * WTILE;
              const size_t s1 = p.parts == 2 ? (t1 * 2 + part) * WTILE : t1 * WTILE;
              bulk_g2s(dst + part * WS, p.w + s0, rows0 * 128, &w_full[wr.s]);
              if (rows1) bulk_g2s(dst + part * WS + 128 * 128, p.w + s1, rows1 * 128, &w_full[wr.s]);
            }
          }
          __syncwarp();
          wr.adv(S);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = idesc_bf16_f32(128, p.NN);
    Ring xr, wr;
    uint32_t gd = 0, dph = 0;
    int db = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      const int tile = item / p.NCTN;
      const long long q0 = (long long)tile * 128;
      const long long r0 = ((long long)p.G + q0 - p.Wp - 1) & ~7LL;
      const uint32_t arow0 = (uint32_t)(p.G + q0 - r0);  // A row of pixel q0 in the X stage
      uint32_t d = 0;
      for (int c = 0; c < p.NC; ++c) {
        if (c % p.seg == 0) {  // a new accumulation segment: the next D buffer
          if (gd >= 2) mbar_wait(&d_empty[db], dph ^ 1);
          tc_fence_after();
          d = tmem + db * p.NN;
        }
        const bool seg_end = c % p.seg == p.seg - 1 || c == p.NC - 1;
        mbar_wait(&x_full[xr.s], xr.ph);
        const uint32_t xa = smem_u32(xs + xr.s * xstage);
        for (int t = 0; t < 9; ++t) {
          mbar_wait(&w_full[wr.s], wr.ph);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t wa = smem_u32(ws + wr.s * wstage);
            const uint32_t arow = (arow0 + p.off[t]) * 128;
            const uint64_t ah = desc_k_sw128(xa + arow), bh = desc_k_sw128(wa);
            const uint32_t acc = (c % p.seg != 0) || t != 0;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, ah + 2 * kk, bh + 2 * kk, idesc, acc | kk);
            if (p.passes == 3) {
              const uint64_t al = desc_k_sw128(xa + XS + arow), bl = desc_k_sw128(wa + WS);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, al + 2 * kk, bh + 2 * kk, idesc, 1);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(d, ah + 2 * kk, bl + 2 * kk, idesc, 1);
            }
            mma_commit(&w_empty[wr.s]);
            if (t == 8) mma_commit(&x_empty[xr.s]);
            if (t == 8 && seg_end) mma_commit(&d_full[db]);
          }
          __syncwarp();
          wr.adv(S);
        }
        xr.adv(p.x_stages);
        if (seg_end) {
          ++gd;
          if (++db == 2) {
            db = 0;
            dph ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int qd = warp % 4, eh = (warp - 4) / 4;
    const int half = p.NN / 2;
    int db = 0;
    uint32_t dph = 0;
    const size_t plane = (size_t)p.H * p.W;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      const int tile = item / p.NCTN, ct = item % p.NCTN;
      const long long q = (long long)tile * 128 + qd * 32 + lane;
      bool ok = q < (long long)p.N * p.Pimg;
      int n = 0, h = 0, w = 0;
      if (ok) {
        n = (int)(q / p.Pimg);
        const int rem = (int)(q % p.Pimg);
        h = rem / p.Wp - 1;
        w = rem % p.Wp - 1;
        ok = h >= 0 && h < p.H && w >= 0 && w < p.W;
      }
      const size_t pix = (size_t)n * p.Cout * plane + (size_t)h * p.W + w;
      const int nseg = (p.NC + p.seg - 1) / p.seg;
      for (int sg = 0; sg < nseg; ++sg) {
        // long reductions (Cin > 8*64) are cut into segments of <= 4608 K: each segment is a
        // fresh TMEM accumulation, added here in FP32 (same thread, program order); the
        // tensor-core accumulation error grows with the K of one accumulator
        // (profiles/r01/igemm/acc_probe.txt), the sum of segments only with its square root
        const bool first = sg == 0, last = sg == nseg - 1;
        mbar_wait(&d_full[db], dph);
        tc_fence_after();
        const uint32_t a = tmem + ((uint32_t)(qd * 32) << 16) + db * p.NN + eh * half;
        for (int c0 = 0; c0 < half; c0 += 16) {
          float v[16];
          tmem_ld16(a + c0, v);
          tmem_wait_ld();
          if (ok) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int co = ct * p.NN + eh * half + c0 + j;
              if (co < p.Cout) {
                float* yp = p.y + pix + (size_t)co * plane;
                float r = first ? v[j] : *yp + v[j];
                if (last) {
                  r += p.bias ? p.bias[co] : 0.f;
                  if (p.act == RC_ACT_RELU) r = fmaxf(r, 0.f);
                  if (p.am) p.am[pix + (size_t)co * plane] = 0;
                }
                *yp = r;
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[db]);
        if (++db == 2) {
          db = 0;
          dph ^= 1;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

struct IgGeom {
  int Wp, G, Pimg, xrows, NC, NCTW, NN, NCTN, tiles;
  long long rows;
};
IgGeom ig_geom(const rc_desc& d) {
  IgGeom g;
  g.Wp = d.w + 2;
  g.G = (g.Wp + 1 + 7) / 8 * 8;
  g.Pimg = (d.h + 2) * g.Wp;
  g.tiles = (int)(((long long)d.n * g.Pimg + 127) / 128);
  // the last tile's rows [r0, r0 + xrows) must lie inside the plane
  g.xrows = (128 + 2 * (g.Wp + 1) + 7 + 7) / 8 * 8;
  g.rows = ((long long)g.G + (long long)g.tiles * 128 + g.Wp + 1 + g.xrows + 7) / 8 * 8;
  g.NC = (d.c_in + KC - 1) / KC;
  g.NCTW = (d.c_out + 127) / 128;
  g.NN = d.c_out >= 256 ? 256 : (d.c_out + 31) / 32 * 32;
  g.NCTN = (d.c_out + g.NN - 1) / g.NN;
  // small layers: 128-channel N tiles when 256-channel tiles would leave SMs idle (the C2
  // appendix cells: 81 pixel tiles at 16x16, N = 32)
  if (g.NN == 256 && (long long)g.tiles * g.NCTN < 148) {
    g.NN = 128;
    g.NCTN = (d.c_out + 127) / 128;
  }
  return g;
}

struct IgPlan {
  int x_stages, w_stages;
  size_t bytes;
};
IgPlan ig_plan(const IgGeom& g, int parts) {
  const size_t cap = 232448 - 1024 - 512;
  const size_t xst = (size_t)parts * g.xrows * 128, wst = (size_t)parts * g.NN * 128;
  for (int xsn = 2; xsn >= 1; --xsn) {
    if (xsn * xst + 2 * wst > cap) continue;
    const size_t ws = (cap - xsn * xst) / wst;
    const int wsn = ws > MAX_WSTAGES ? MAX_WSTAGES : (int)ws;
    return IgPlan{xsn, wsn, xsn * xst + wsn * wst + 1024};
  }
  return IgPlan{0, 0, 0};
}

}  // namespace

bool igemm_supported(const rc_desc& d) {
  // whole 8x8 / 4x4 images: the band kernels' small-image geometry has neither halo nor pad
  // (the padded grid here would be 1.56x / 2.25x the pixels); C1: 16.5 vs 31.5 us
  if ((d.w == 8 && d.h == 8) || (d.w == 4 && d.h == 4)) return false;
  if (!(d.group == RC_GROUP_SINGLE && d.k == 3 &&
        (d.precision == RC_PREC_BF16 || d.precision == RC_PREC_BF16X3 || d.precision == RC_PREC_AUTO)))
    return false;
  const int parts = d.precision == RC_PREC_BF16 ? 1 : 2;
  return ig_plan(ig_geom(d), parts).x_stages > 0;
}

size_t igemm_workspace_bytes(const rc_desc& d) {
  const IgGeom g = ig_geom(d);
  const int parts = d.precision == RC_PREC_BF16 ? 1 : 2;
  return (size_t)parts * g.NC * g.rows * 128;
}

PadGeom pad_geom(const rc_desc& d) {
  const IgGeom g = ig_geom(d);
  return PadGeom{g.Wp, g.G, g.Pimg, g.NC, g.rows};
}

size_t pad_planes_bytes(const rc_desc& d, int parts) {
  const IgGeom g = ig_geom(d);
  return (size_t)parts * g.NC * g.rows * 128;
}

int launch_pad_pack(const rc_desc& d, const float* x, uint8_t* xh, uint8_t* xl, cudaStream_t s) {
  const IgGeom g = ig_geom(d);
  const long long total = (long long)g.NC * ((g.rows + PACK_ROWS - 1) / PACK_ROWS);
  const long long grid = total < 148 * 16 ? total : 148 * 16;
  ig_pack_kernel<<<(int)grid, 256, 0, s>>>(x, xh, xl, d.n, d.c_in, d.h, d.w, g.Wp, g.G, g.Pimg, g.rows, g.NC);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

// bank: the tc section of the bank (ri_tc.cu's packed weights; whi = its hi-only plane)
int launch_igemm(const rc_desc& d, const float* x, const uint8_t* wpk, const uint8_t* whi, const float* bias,
                 float* y, uint8_t* am, void* ws, cudaStream_t s) {
  const IgGeom g = ig_geom(d);
  const int passes = d.precision == RC_PREC_BF16 ? 1 : 3;
  const int parts = passes == 3 ? 2 : 1;
  const IgPlan plan = ig_plan(g, parts);
  uint8_t* xh = static_cast<uint8_t*>(ws);
  uint8_t* xl = parts == 2 ? xh + (size_t)g.NC * g.rows * 128 : nullptr;
  {
    const int st = launch_pad_pack(d, x, xh, xl, s);
    if (st != RC_OK) return st;
  }
  IgParams p;
  p.xh = xh;
  p.xl = xl;
  p.w = passes == 3 ? wpk : whi;
  p.bias = bias;
  p.y = y;
  p.am = (d.pool == RC_POOL_MAX || d.pool == RC_POOL_SUBGROUP) ? am : nullptr;
  p.rows = g.rows;
  p.N = d.n;
  p.H = d.h;
  p.W = d.w;
  p.Cout = d.c_out;
  p.NC = g.NC;
  p.NCTW = g.NCTW;
  p.NN = g.NN;
  p.NCTN = g.NCTN;
  p.tiles = g.tiles;
  p.items = g.tiles * g.NCTN;
  p.Wp = g.Wp;
  p.G = g.G;
  p.Pimg = g.Pimg;
  p.xrows = g.xrows;
  p.parts = parts;
  p.passes = passes;
  p.x_stages = plan.x_stages;
  p.w_stages = plan.w_stages;
  p.act = d.activation;
  {
    p.seg = 8;  // chunks per accumulation segment (profiles/r01/igemm/acc_probe.txt)
  }
  TapOffsets to;
  slice_tap_offsets(3, d.convention, &to);
  for (int t = 0; t < 9; ++t) p.off[t] = to.di[0][t] * g.Wp + to.dj[0][t];
  int dev, sms;
  RC_CUDA(cudaGetDevice(&dev));
  RC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RC_CUDA(cudaFuncSetAttribute(igemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.bytes));
  const int grid = p.items < sms ? p.items : sms;
  prof_begin(s);
  igemm_kernel<<<grid, THREADS, plan.bytes, s>>>(p);
  prof_end(s);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

}  // namespace rc
