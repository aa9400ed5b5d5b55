// ri_direct.cu -- FP32 CUDA-core single-orientation K = 3 conv for small channel counts
// (Cin <= 32; `auto` uses it up to Cin = 16) on small images (W in {4, 8, 16, 32}): the C2
// appendix cells where the layer is a few microseconds of work and the row-sweep SIMT kernel
// (ri_simt.cu) or the tensor-core kernels (K padded to 64 channels per chunk) spend it on
// pipeline set-up.
//
// Same math as scatter_conv_multi (scatter_conv.hpp:189-193) / tiled_scatter_conv
// (:330-368) for R = 1, convention P1 (k3_tables.cuh):
//   y[n, co, h, w] = sum_ci sum_t W[co, ci, t] * X[n, ci, h + di_t, w + dj_t]   (+ bias, ReLU)
// Lane = output channel (32 per warp), warp = (image, TR output rows); the warp's X slab
// (Cin x (TR + 2) x (W + 2), zero-padded) sits in shared memory and is read as broadcasts,
// the CTA's 32-channel weights as [Cin * 9][33] (one conflict-free word per lane).  Each
// thread keeps TR x W accumulators; per input channel it loads the (TR + 2) padded rows into
// registers once and runs the 9 taps as FMA chains from registers.  Accumulation order per
// output: ci ascending, taps ascending -- dyadic inputs are bit-exact vs the oracle.
#include "k3_tables.cuh"
#include "rc_internal.cuh"

namespace rc {
namespace {

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(gmem), "r"(valid ? 4 : 0));
}

constexpr int DCO = 32;      // output channels per CTA (one per lane)
constexpr int WS = DCO + 1;  // weight row stride in shared memory (conflict-free transposed fill)
constexpr int DMAX_CIN = 32;

struct DirectParams {
  const float* x;     // [N][Cin][H][W]
  const float* w;     // base kernels [Cout][Cin][3][3]
  const float* bias;  // [Cout] or null
  float* y;           // [N][Cout][1][H][W]
  uint8_t* am;        // argmax for max / subgroup pooling of R = 1: always orientation 0
  int N, Cin, H, Cout, act, units, row_groups;
};

template <int W, int TR, int RW, int CONV>
__global__ void __launch_bounds__(32 * RW) direct_k3_kernel(const __grid_constant__ DirectParams p) {
  constexpr int PW = W + 2, PR = TR + 2;  // padded slab
  extern __shared__ float sm[];
  float* ws = sm;                                        // [Cin * 9][WS]
  float* xs = sm + p.Cin * 9 * WS + (threadIdx.x / 32) * (p.Cin * PR * PW);  // this warp's slab
  const int lane = threadIdx.x & 31, warp = threadIdx.x / 32;
  const int co0 = blockIdx.x * DCO, co = co0 + lane;
  // weights of the CTA's 32 channels: coalesced reads of [co][ci][t], transposed into
  // [ci * 9 + t][lane] rows of stride 33 (conflict-free both ways)
  // Both fills are cp.async copies (4 bytes, zero-filled outside the image / channel range):
  // no thread waits on one load before issuing the next -- the whole layer is a few
  // microseconds, so serialised load latencies would dominate it.
  const int taps = p.Cin * 9;
  for (int i = threadIdx.x; i < taps * DCO; i += blockDim.x) {
    const int l = i / taps;
    const bool ok = co0 + l < p.Cout;
    cp_async4(&ws[(i - l * taps) * WS + l], ok ? p.w + (size_t)co0 * taps + i : p.w, ok);
  }
  const int unit = blockIdx.y * RW + warp;  // (image, row group) of this warp
  const bool live = unit < p.units;
  const int n = live ? unit / p.row_groups : 0, r0 = live ? (unit % p.row_groups) * TR : 0;
  if (live) {
    const float* xn = p.x + (size_t)n * p.Cin * p.H * W;
    for (int i = lane; i < p.Cin * PR * PW; i += 32) {
      const int c = i % PW, r = (i / PW) % PR, ci = i / (PW * PR);
      const int hh = r0 - 1 + r, ww = c - 1;
      const bool ok = hh >= 0 && hh < p.H && ww >= 0 && ww < W;
      cp_async4(&xs[i], ok ? xn + ((size_t)ci * p.H + hh) * W + ww : xn, ok);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  if (!live) return;
  float acc[TR][W];
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < W; ++j) acc[i][j] = 0.f;
  constexpr K3Tables T = make_k3(CONV);
  for (int ci = 0; ci < p.Cin; ++ci) {
    float xr[PR][PW];
    const float* xc = xs + ci * PR * PW;
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int c = 0; c < PW; ++c) xr[r][c] = xc[r * PW + c];
    const float* wc = ws + ci * 9 * WS + lane;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const float wv = wc[t * WS];
      const int di = T.di[0][t], dj = T.dj[0][t];
#pragma unroll
      for (int i = 0; i < TR; ++i)
#pragma unroll
        for (int j = 0; j < W; ++j) acc[i][j] = fmaf(wv, xr[i + 1 + di][j + 1 + dj], acc[i][j]);
    }
  }
  if (co >= p.Cout) return;
  const float bz = p.bias ? p.bias[co] : 0.f;
  float* yc = p.y + ((size_t)n * p.Cout + co) * p.H * W;
  if (p.am) {  // R = 1: the argmax of a max / subgroup pool over one orientation is 0
    uint8_t* ac = p.am + ((size_t)n * p.Cout + co) * p.H * W;
    for (int i = 0; i < TR && r0 + i < p.H; ++i)
#pragma unroll
      for (int j = 0; j < W; j += 4) *reinterpret_cast<uint32_t*>(ac + (size_t)(r0 + i) * W + j) = 0u;
  }
#pragma unroll
  for (int i = 0; i < TR; ++i) {
    const int row = r0 + i;
    if (row >= p.H) break;
#pragma unroll
    for (int j = 0; j < W; j += 4) {
      float4 v = make_float4(acc[i][j] + bz, acc[i][j + 1] + bz, acc[i][j + 2] + bz, acc[i][j + 3] + bz);
      if (p.act == RC_ACT_RELU) {
        v.x = fmaxf(v.x, 0.f);
        v.y = fmaxf(v.y, 0.f);
        v.z = fmaxf(v.z, 0.f);
        v.w = fmaxf(v.w, 0.f);
      }
      *reinterpret_cast<float4*>(yc + (size_t)row * W + j) = v;
    }
  }
}

template <int W, int TR, int RW>
int launch_rw(const rc_desc& d, const DirectParams& p, cudaStream_t s) {
  const int rg = (d.h + TR - 1) / TR;
  DirectParams q = p;
  q.row_groups = rg;
  q.units = d.n * rg;
  const dim3 grid((d.c_out + DCO - 1) / DCO, (q.units + RW - 1) / RW);
  if (grid.y > 65535) return RC_ERR_UNSUPPORTED;
  const size_t smem = sizeof(float) * ((size_t)d.c_in * 9 * WS + (size_t)RW * d.c_in * (TR + 2) * (W + 2));
  auto fn = d.convention == RC_CONV_RAW ? direct_k3_kernel<W, TR, RW, 1> : direct_k3_kernel<W, TR, RW, 0>;
  if (smem > 48 * 1024) RC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  prof_begin(s);
  fn<<<grid, 32 * RW, smem, s>>>(q);
  prof_end(s);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

// warps per CTA: 4 (the weight stage is shared by more units) unless the grid would then
// leave SMs idle (fewer than 2 x 148 CTAs), then 2 or 1
template <int W, int TR>
int launch_w(const rc_desc& d, const DirectParams& p, cudaStream_t s) {
  const long long units = (long long)d.n * ((d.h + TR - 1) / TR), cob = (d.c_out + DCO - 1) / DCO;
  if (cob * ((units + 3) / 4) >= 296) return launch_rw<W, TR, 4>(d, p, s);
  if (cob * ((units + 1) / 2) >= 296) return launch_rw<W, TR, 2>(d, p, s);
  return launch_rw<W, TR, 1>(d, p, s);
}

}  // namespace

bool direct_supported(const rc_desc& d) {
  return d.group == RC_GROUP_SINGLE && d.k == 3 && d.c_in >= 1 && d.c_in <= DMAX_CIN &&
         (d.w == 4 || d.w == 8 || d.w == 16 || d.w == 32) && d.h >= 1;
}

int launch_direct_k3(const rc_desc& d, const float* x, const void* bank, const float* bias, float* y,
                     uint8_t* am, cudaStream_t s, bool dry_run, const char** name) {
  if (!direct_supported(d)) return RC_ERR_UNSUPPORTED;
  if (name) {
    static thread_local char buf[32];
    snprintf(buf, sizeof buf, "simt_direct_k3<%d>", d.w);
    *name = buf;
  }
  if (dry_run || d.n == 0) return RC_OK;
  DirectParams p;
  p.x = x;
  p.w = reinterpret_cast<const float*>(static_cast<const char*>(bank) + bank_layout(d).bases_off);
  p.bias = bias;
  p.y = y;
  p.am = (d.pool == RC_POOL_MAX || d.pool == RC_POOL_SUBGROUP) ? am : nullptr;
  p.N = d.n;
  p.Cin = d.c_in;
  p.H = d.h;
  p.Cout = d.c_out;
  p.act = d.activation;
  // TR x W = 16 or 32 accumulators per thread
  switch (d.w) {
    case 4: return launch_w<4, 4>(d, p, s);
    case 8: return launch_w<8, 4>(d, p, s);
    case 16: return launch_w<16, 2>(d, p, s);
    default: return launch_w<32, 1>(d, p, s);
  }
}

}  // namespace rc
