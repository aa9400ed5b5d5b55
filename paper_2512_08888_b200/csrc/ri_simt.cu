// ri_simt.cu -- CUDA-core FP32 fused RI scatter convolution for K = 3 (sm_100a).
//
// What it computes (one launch = the whole layer): for every image n, output channel
// co and base kernel b (SPEC:274-282 group_conv_scatter_reuse):
//   Z_t(q) = sum_ci K_b[co, ci, t] * X[n, ci, q]           (one channel dot per tap t)
//   Y_{b,r}(p) += Z_t(p + delta_{r,t})                     (reused by all 4 rotations r)
// then orientation pooling and the bias epilogue, straight to HBM.
// delta_{r,t} are the slice index maps of convention P1 (slice (b,r) ==
// scatter_conv_multi(X, rot90^r K_b), scatter_conv.hpp:189-193), compile-time here.
//
// Dataflow (output-stationary, no global atomics):
//  * thread = (image, co, x-segment of SW columns); S = W/SW segments per image row
//    sit in adjacent lanes, so the one-column halo of Z is a warp shuffle.
//  * the image is swept row by row (the reference's row-locality): input row q
//    produces Z for 9 taps x SW columns in registers (72 FFMA chains over ci) and
//    scatters them into a 3-row ring of 4-rotation accumulators (96 registers); output
//    row q-1 is then complete and is pooled + stored with 128-bit stores.
//  * X rows and the co-block's weights stream through a 2-stage cp.async ring in shared
//    memory, CC input channels per stage; IMG images share each weight stage.
// Each channel dot accumulates in ascending ci with FFMA; each output adds its 9 taps in
// a fixed order, so dyadic inputs reproduce the oracle bit-for-bit (tests/test_gpu_parity).
#include <algorithm>
#include <cstdlib>

#include "k3_tables.cuh"
#include "rc_internal.cuh"

#ifndef RC_SIMT_ROT
#define RC_SIMT_ROT 1  // 1: one step body + register ring rotation; 0: three unrolled ring phases
#endif

namespace rc {
namespace {

constexpr int CC = 32;  // input channels per shared-memory stage (32: half the CTA barriers of 16, C3 fp32 -5.6%)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src_size = valid ? 16 : 0;  // 0 -> zero-fill (ragged Cin / Cout / N)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_size));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct Params {
  const float* x;     // [N][Cin][H][W]
  const float* wk;    // [B][Cin][Cout][12]
  const float* bias;  // [Cout] or null
  float* y;           // [N][Cout][RO][H][W]
  uint8_t* am;        // [N][Cout][RO][H][W] or null
  int N, Cin, H, Cout, NB, pool, gf, RO, COB, IMG;
  int act;  // rc_activation, applied after the bias
  int resident;  // small Cin (<= CC): the CTA's images and all weights are loaded into shared
                 // memory once; the row sweep then runs without copies or CTA barriers
};

template <int SW, int S, int RPB, int CONV>
struct SimtK3 {
  static constexpr int W = SW * S;
  // register pairs: the channel dots and the scatter run as packed FP32x2 (FFMA2 / FADD2,
  // one instruction per two columns; per-lane IEEE fma / add, so results are unchanged)
  float2 Z2[9][SW / 2];
  float2 Y2[3][RPB][SW / 2];
  __device__ __forceinline__ float& Y(int s, int r, int j) { return (j & 1) ? Y2[s][r][j >> 1].y : Y2[s][r][j >> 1].x; }
  __device__ __forceinline__ float& Z(int t, int j) { return (j & 1) ? Z2[t][j >> 1].y : Z2[t][j >> 1].x; }

  const Params& p;
  float* smem;
  int tid, seg, co_l, img_l, co, n, x0, nchunks, stage_x, stage_floats;

  __device__ SimtK3(const Params& pp, float* sm) : p(pp), smem(sm) {
    tid = threadIdx.x;
    seg = tid % S;
    co_l = (tid / S) % p.COB;
    img_l = tid / (S * p.COB);
    co = blockIdx.x * p.COB + co_l;
    n = blockIdx.y * p.IMG + img_l;
    x0 = seg * SW;
    nchunks = (p.Cin + CC - 1) / CC;
    stage_x = p.IMG * CC * W;
    stage_floats = stage_x + CC * p.COB * 12;
  }

  // cooperative cp.async of chunk gi = ((b*H)+q)*nchunks + c into stage gi&1
  __device__ void issue(int gi, int total) {
    if (gi < total) {
      const int c = gi % nchunks;
      const int q = (gi / nchunks) % p.H;
      const int b = gi / (nchunks * p.H);
      float* st = smem + (gi & 1) * stage_floats;
      const int xq = W / 4;  // 16-byte pieces per image row
      const int nx = p.IMG * CC * xq;
      const int n0 = blockIdx.y * p.IMG;
      for (int i = tid; i < nx; i += blockDim.x) {
        const int img = i / (CC * xq), rem = i % (CC * xq);
        const int cl = rem / xq, x4 = rem % xq;
        const int gn = n0 + img, gci = c * CC + cl;
        const bool ok = gn < p.N && gci < p.Cin;
        const float* src =
            p.x + ((((size_t)(ok ? gn : 0) * p.Cin + (ok ? gci : 0)) * p.H + q) * W + x4 * 4);
        cp_async16(st + (img * CC + cl) * W + x4 * 4, src, ok);
      }
      const int nw = CC * p.COB * 3;
      const int co0 = blockIdx.x * p.COB;
      float* sw = st + stage_x;
      for (int i = tid; i < nw; i += blockDim.x) {
        const int cl = i / (p.COB * 3), rem = i % (p.COB * 3);
        const int cc = rem / 3, part = rem % 3;
        const int gci = c * CC + cl, gco = co0 + cc;
        const bool ok = gci < p.Cin && gco < p.Cout;
        const float* src =
            p.wk + ((((size_t)b * p.Cin + (ok ? gci : 0)) * p.Cout + (ok ? gco : 0)) * 12 + part * 4);
        cp_async16(sw + (cl * p.COB + cc) * 12 + part * 4, src, ok);
      }
    }
    cp_async_commit();
  }

  // ncl = channels of this chunk (CC, fewer for the last chunk of a small / ragged Cin:
  // the zero-filled tail channels are skipped instead of multiplied)
  __device__ __forceinline__ void compute_stage(const float* st, int ncl) {
    compute_rows(st + img_l * CC * W + x0, W, reinterpret_cast<const float4*>(st + stage_x) + co_l * 3, ncl);
  }
  // resident mode: X [img][ci][H][W], then weights [b][ci][COB][12] for all bases
  __device__ __forceinline__ void compute_resident(int b, int q) {
    const float* sx = smem + ((size_t)img_l * p.Cin * p.H + q) * W + x0;
    const float* swf = smem + (size_t)p.IMG * p.Cin * p.H * W;
    compute_rows(sx, p.H * W, reinterpret_cast<const float4*>(swf) + ((size_t)b * p.Cin * p.COB + co_l) * 3, p.Cin);
  }
  __device__ void load_resident() {
    const int xq = W / 4;
    const int per_img = p.Cin * p.H * xq;
    const int n0 = blockIdx.y * p.IMG;
    for (int i = tid; i < p.IMG * per_img; i += blockDim.x) {
      const int img = i / per_img, rem = i % per_img;
      const bool ok = n0 + img < p.N;
      cp_async16(smem + (size_t)i * 4, p.x + ((size_t)(ok ? n0 + img : 0) * per_img + rem) * 4, ok);
    }
    float* sw = smem + (size_t)p.IMG * p.Cin * p.H * W;
    const int nw = p.NB * p.Cin * p.COB * 3;
    const int co0 = blockIdx.x * p.COB;
    for (int i = tid; i < nw; i += blockDim.x) {
      const int b = i / (p.Cin * p.COB * 3), r1 = i % (p.Cin * p.COB * 3);
      const int ci = r1 / (p.COB * 3), r2 = r1 % (p.COB * 3);
      const int cc = r2 / 3, part = r2 % 3;
      const bool ok = co0 + cc < p.Cout;
      const float* src = p.wk + ((((size_t)b * p.Cin + ci) * p.Cout + (ok ? co0 + cc : 0)) * 12 + part * 4);
      cp_async16(sw + (size_t)i * 4, src, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
  }
  // channel dots of ncl channels (channel stride cs floats; weights 3 float4 per channel,
  // COB*3 float4 apart), accumulated in ascending ci
  __device__ __forceinline__ void compute_rows(const float* sx, int cs, const float4* sw, int ncl) {
#pragma unroll 4
    for (int cl = 0; cl < ncl; ++cl) {
      float xv[SW];
#pragma unroll
      for (int v = 0; v < SW / 4; ++v) {
        const float4 t4 = *reinterpret_cast<const float4*>(sx + (size_t)cl * cs + v * 4);
        xv[v * 4 + 0] = t4.x;
        xv[v * 4 + 1] = t4.y;
        xv[v * 4 + 2] = t4.z;
        xv[v * 4 + 3] = t4.w;
      }
      const float4 a = sw[cl * p.COB * 3 + 0];
      const float4 bq = sw[cl * p.COB * 3 + 1];
      const float4 cq = sw[cl * p.COB * 3 + 2];
      const float wv[9] = {a.x, a.y, a.z, a.w, bq.x, bq.y, bq.z, bq.w, cq.x};
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const float2 w2 = make_float2(wv[t], wv[t]);
#pragma unroll
        for (int k = 0; k < SW / 2; ++k)
          Z2[t][k] = __ffma2_rn(w2, make_float2(xv[2 * k], xv[2 * k + 1]), Z2[t][k]);
      }
    }
  }

  __device__ __forceinline__ void store_vec(float* dst, const float (&v)[SW]) {
#pragma unroll
    for (int k = 0; k < SW / 4; ++k)
      reinterpret_cast<float4*>(dst)[k] = make_float4(v[k * 4], v[k * 4 + 1], v[k * 4 + 2], v[k * 4 + 3]);
  }
  __device__ __forceinline__ void store_arg(uint8_t* dst, const uint8_t (&a)[SW]) {
    uint32_t w[SW / 4];
#pragma unroll
    for (int k = 0; k < SW / 4; ++k)
      w[k] = a[k * 4] | (a[k * 4 + 1] << 8) | (a[k * 4 + 2] << 16) | ((uint32_t)a[k * 4 + 3] << 24);
    if constexpr (SW == 8)
      *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
    else
      *reinterpret_cast<uint32_t*>(dst) = w[0];
  }

  __device__ __forceinline__ float activate(float v) const { return p.act == RC_ACT_RELU ? fmaxf(v, 0.f) : v; }

  // pool + bias + store of one finished output row (slot), base b
  template <int SLOT>
  __device__ void finalize(int b, int row) {
    if (n >= p.N || co >= p.Cout) return;
    const size_t plane = (size_t)p.H * W;
    const size_t ybase = ((size_t)n * p.Cout + co) * p.RO * plane + (size_t)row * W + x0;
    const float bz = p.bias ? p.bias[co] : 0.f;
    const int R = p.NB * RPB;
    if (p.pool == RC_POOL_NONE) {
#pragma unroll
      for (int r = 0; r < RPB; ++r) {
        float v[SW];
#pragma unroll
        for (int j = 0; j < SW; ++j) v[j] = activate(Y(SLOT, r, j) + bz);
        store_vec(p.y + ybase + (size_t)(b * RPB + r) * plane, v);
      }
      return;
    }
    if (p.pool == RC_POOL_AVG) {
      float acc[SW];
      if (b == 0) {
#pragma unroll
        for (int j = 0; j < SW; ++j) acc[j] = Y(SLOT, 0, j);
      } else {
#pragma unroll
        for (int j = 0; j < SW; ++j) acc[j] = p.y[ybase + j] + Y(SLOT, 0, j);
      }
#pragma unroll
      for (int r = 1; r < RPB; ++r)
#pragma unroll
        for (int j = 0; j < SW; ++j) acc[j] += Y(SLOT, r, j);
      if (b == p.NB - 1) {
#pragma unroll
        for (int j = 0; j < SW; ++j) acc[j] = activate(acc[j] / (float)R + bz);
      }
      store_vec(p.y + ybase, acc);
      return;
    }
    // max / subgroup max with argmax (ties -> smallest orientation index)
    const int gf = p.gf;
    float best[SW];
    uint8_t arg[SW];
#pragma unroll
    for (int r = 0; r < RPB; ++r) {
      const int o = b * RPB + r;
      const int slot = o / gf, kk = o - slot * gf;
      const size_t off = ybase + (size_t)slot * plane;
      if (kk == 0) {
#pragma unroll
        for (int j = 0; j < SW; ++j) {
          best[j] = Y(SLOT, r, j);
          arg[j] = 0;
        }
      } else {
        if (r == 0) {  // this slot started in the previous base: reload its partial state
#pragma unroll
          for (int j = 0; j < SW; ++j) {
            best[j] = p.y[off + j];
            arg[j] = p.am ? p.am[off + j] : 0;
          }
        }
#pragma unroll
        for (int j = 0; j < SW; ++j)
          if (Y(SLOT, r, j) > best[j]) {
            best[j] = Y(SLOT, r, j);
            arg[j] = (uint8_t)kk;
          }
      }
      if (kk == gf - 1 || r == RPB - 1) {
        float v[SW];
        const bool final_ = kk == gf - 1;
#pragma unroll
        for (int j = 0; j < SW; ++j) v[j] = final_ ? activate(best[j] + bz) : best[j];
        store_vec(p.y + off, v);
        if (p.am) store_arg(p.am + off, arg);
      }
    }
  }

  template <int P>
  __device__ void step(int b, int q, int& gi, int total) {
    // slot (P+1)%3 held output row q-2 (finalised last step); it now receives row q+1.
    // At q == 0 (start of a base) slot P (row 0) is fresh too; slot (P+2)%3 collects the
    // clipped row -1 and is zeroed before reuse at q == 1.
#pragma unroll
    for (int r = 0; r < RPB; ++r)
#pragma unroll
      for (int k = 0; k < SW / 2; ++k) Y2[(P + 1) % 3][r][k] = make_float2(0.f, 0.f);
    if (P == 0 && q == 0) {
#pragma unroll
      for (int r = 0; r < RPB; ++r)
#pragma unroll
        for (int k = 0; k < SW / 2; ++k) Y2[0][r][k] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int k = 0; k < SW / 2; ++k) Z2[t][k] = make_float2(0.f, 0.f);
    if (q < p.H && p.resident) {
      compute_resident(b, q);
    } else if (q < p.H) {
      for (int c = 0; c < nchunks; ++c, ++gi) {
        issue(gi + 1, total);
        cp_async_wait<1>();
        __syncthreads();
        compute_stage(smem + (gi & 1) * stage_floats, min(CC, p.Cin - c * CC));
        __syncthreads();
      }
    }
    // one-column halo from the neighbouring segments (zero at the image border)
    float Zl[9], Zr[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      if constexpr (S > 1) {
        const float l = __shfl_up_sync(0xffffffffu, Z2[t][SW / 2 - 1].y, 1, S);
        const float rr = __shfl_down_sync(0xffffffffu, Z2[t][0].x, 1, S);
        Zl[t] = seg == 0 ? 0.f : l;
        Zr[t] = seg == S - 1 ? 0.f : rr;
      } else {
        Zl[t] = 0.f;
        Zr[t] = 0.f;
      }
    }
    // reuse scatter: each Z_t feeds all RPB rotations (PAPER Eq. 8).
    // Y[j] += Z[j + dj]: dj = 0 adds the aligned pairs Z2[k]; dj = -1 / +1 add the odd-aligned
    // pairs B[k] = (Z[2k-1], Z[2k]) / B[k+1], built once per tap (halo columns included).
    constexpr K3Tables TB = make_k3(CONV);
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      float2 B[SW / 2 + 1];
      B[0] = make_float2(Zl[t], Z2[t][0].x);
#pragma unroll
      for (int k = 1; k < SW / 2; ++k) B[k] = make_float2(Z2[t][k - 1].y, Z2[t][k].x);
      B[SW / 2] = make_float2(Z2[t][SW / 2 - 1].y, Zr[t]);
#pragma unroll
      for (int r = 0; r < RPB; ++r) {
        const int di = TB.di[r][t], dj = TB.dj[r][t];
        const int slot = (P - di + 3) % 3;
#pragma unroll
        for (int k = 0; k < SW / 2; ++k) {
          const float2 v = dj == 0 ? Z2[t][k] : (dj < 0 ? B[k] : B[k + 1]);
          if (slot == 0) Y2[0][r][k] = __fadd2_rn(Y2[0][r][k], v);
          else if (slot == 1) Y2[1][r][k] = __fadd2_rn(Y2[1][r][k], v);
          else Y2[2][r][k] = __fadd2_rn(Y2[2][r][k], v);
        }
      }
    }
    if (q >= 1) finalize<(P + 2) % 3>(b, q - 1);
  }

  __device__ void run() {
    const int total = p.NB * p.H * nchunks;
    int gi = 0;
    if (p.resident)
      load_resident();
    else
      issue(0, total);
    for (int b = 0; b < p.NB; ++b) {
#if RC_SIMT_ROT
      // one step body (a third of the code of three ring phases, for the instruction cache):
      // slot 0 = row q, 1 = row q+1, 2 = row q-1; the ring is rotated by register moves
      for (int q = 0; q <= p.H; ++q) {
        step<0>(b, q, gi, total);
#pragma unroll
        for (int r = 0; r < RPB; ++r)
#pragma unroll
          for (int k = 0; k < SW / 2; ++k) {
            Y2[2][r][k] = Y2[0][r][k];
            Y2[0][r][k] = Y2[1][r][k];
          }
      }
#else
      for (int q0 = 0; q0 <= p.H; q0 += 3) {
        step<0>(b, q0, gi, total);
        if (q0 + 1 <= p.H) step<1>(b, q0 + 1, gi, total);
        if (q0 + 2 <= p.H) step<2>(b, q0 + 2, gi, total);
      }
#endif
    }
    cp_async_wait<0>();
  }
};

#ifndef RC_SIMT_MINB
#define RC_SIMT_MINB 1  // resident CTAs per SM the register allocation targets (A/B builds)
#endif
template <int SW, int S, int RPB, int CONV>
__global__ void __launch_bounds__(256, RC_SIMT_MINB) simt_k3_kernel(Params p) {
  extern __shared__ __align__(16) float smem[];
  SimtK3<SW, S, RPB, CONV> k(p, smem);
  k.run();
}

template <int SW, int S, int RPB, int CONV>
int launch_t(const Params& p, int grid_x, int grid_y, int threads, size_t smem, cudaStream_t s) {
  auto fn = simt_k3_kernel<SW, S, RPB, CONV>;
  RC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  prof_begin(s);
  fn<<<dim3(grid_x, grid_y), threads, smem, s>>>(p);
  prof_end(s);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

template <int SW, int S>
int launch_rc(const rc_desc& d, const Params& p, int gx, int gy, int threads, size_t smem,
              cudaStream_t s) {
  const bool single = d.group == RC_GROUP_SINGLE;
  const bool raw = d.convention == RC_CONV_RAW;
  if (single) return raw ? launch_t<SW, S, 1, 1>(p, gx, gy, threads, smem, s)
                         : launch_t<SW, S, 1, 0>(p, gx, gy, threads, smem, s);
  return raw ? launch_t<SW, S, 4, 1>(p, gx, gy, threads, smem, s)
             : launch_t<SW, S, 4, 0>(p, gx, gy, threads, smem, s);
}

}  // namespace

int launch_simt_k3(const rc_desc& d, const float* x, const void* bank, const float* bias,
                   float* y, uint8_t* argmax, cudaStream_t s, bool dry_run, const char** name) {
  if (d.k != 3) return RC_ERR_UNSUPPORTED;
  int SW, S;
  // SW columns per thread: 8 keeps more work per thread, 4 halves the register state
  // (3-row x 4-rotation accumulators) so more warps fit per SM; RC_SIMT_SW selects (A/B)
  const int sw_pref = 8;  // 8-column segments for 8-wide images (profiles/r01/simt_sw_ab.txt)
  switch (d.w) {
    case 4: SW = 4; S = 1; break;
    case 8: SW = sw_pref == 4 ? 4 : 8; S = 8 / SW; break;
    case 16: SW = sw_pref == 4 ? 4 : 8; S = 16 / SW; break;
    case 32: SW = sw_pref == 4 ? 4 : 8; S = 32 / SW; break;
    case 64: SW = sw_pref == 4 ? 4 : 8; S = 64 / SW; break;
    default: return RC_ERR_UNSUPPORTED;
  }
  // CTA shape: threads = COB * S * IMG <= 256; prefer >= 2 waves of CTAs over 148 SMs.
  int COB = std::max(1, std::min(256 / S, 64));
  int IMG = std::max(1, 256 / (COB * S));
  auto ctas = [&](int cob, int img) {
    return (long long)((d.c_out + cob - 1) / cob) * ((d.n + img - 1) / img);
  };
  while (ctas(COB, IMG) < 296 && IMG > 1) IMG /= 2;
  while (ctas(COB, IMG) < 296 && COB * S > 32 && COB > 8) COB /= 2;
  const int threads = COB * S * IMG;
  if (threads % 32 != 0) return RC_ERR_UNSUPPORTED;
  if (name) {
    static thread_local char buf[64];
    snprintf(buf, sizeof buf, "simt_k3<%d,%d,%d>", SW, S, d.group == RC_GROUP_SINGLE ? 1 : 4);
    *name = buf;
  }
  if (dry_run) return RC_OK;
  if (d.n == 0) return RC_OK;
  const BankLayout L = bank_layout(d);
  Params p;
  p.x = x;
  p.wk = reinterpret_cast<const float*>(static_cast<const char*>(bank) + L.simt_off);
  p.bias = bias;
  p.y = y;
  p.am = (d.pool == RC_POOL_MAX || d.pool == RC_POOL_SUBGROUP) ? argmax : nullptr;
  p.N = d.n;
  p.Cin = d.c_in;
  p.H = d.h;
  p.Cout = d.c_out;
  p.NB = num_bases(d);
  p.pool = d.pool;
  p.gf = pool_fold(d);
  p.RO = out_orientations(d);
  p.COB = COB;
  p.IMG = IMG;
  p.act = d.activation;
  size_t smem = 2 * sizeof(float) * ((size_t)IMG * CC * d.w + (size_t)CC * COB * 12);
  const size_t smem_res = sizeof(float) * ((size_t)IMG * d.c_in * d.h * d.w + (size_t)p.NB * d.c_in * COB * 12);
  p.resident = d.c_in <= CC && smem_res <= 200 * 1024;
  if (p.resident) smem = std::max(smem, smem_res);
  const int gx = (d.c_out + COB - 1) / COB, gy = (d.n + IMG - 1) / IMG;
  if (gy > 65535) return RC_ERR_UNSUPPORTED;
  if (SW == 4) {
    switch (d.w) {
      case 4: return launch_rc<4, 1>(d, p, gx, gy, threads, smem, s);
      case 8: return launch_rc<4, 2>(d, p, gx, gy, threads, smem, s);
      case 16: return launch_rc<4, 4>(d, p, gx, gy, threads, smem, s);
      case 32: return launch_rc<4, 8>(d, p, gx, gy, threads, smem, s);
      default: return launch_rc<4, 16>(d, p, gx, gy, threads, smem, s);
    }
  }
  switch (d.w) {
    case 8: return launch_rc<8, 1>(d, p, gx, gy, threads, smem, s);
    case 16: return launch_rc<8, 2>(d, p, gx, gy, threads, smem, s);
    case 32: return launch_rc<8, 4>(d, p, gx, gy, threads, smem, s);
    default: return launch_rc<8, 8>(d, p, gx, gy, threads, smem, s);
  }
}

}  // namespace rc
