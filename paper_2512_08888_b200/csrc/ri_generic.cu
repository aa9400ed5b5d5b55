// ri_generic.cu -- shape-general FP32 kernels (sm_100a): any K <= 11 (odd or even for
// R = 1), any H, W.  Used where the specialised kernels do not apply (SPEC's K in
// {1, 5}, ragged widths).  Output-stationary gather form of the same slice semantics
// (convention P1): slice (b, r) reads base tap t at gather offset delta_{r,t}.  It does
// not reuse the channel dots across rotations (R/B x the FLOPs of the fused kernels).
// Also: the standalone orientation-pooling kernel for materialised
// OrientedFeature batches.
#include "rc_internal.cuh"

namespace rc {
namespace {

__device__ __forceinline__ void fold(int pool, int k, float v, float& best, int& arg) {
  if (pool == RC_POOL_AVG) {
    best = k == 0 ? v : best + v;
  } else if (k == 0 || v > best) {  // ties -> smallest index
    best = v;
    arg = k;
  }
}

__global__ void generic_kernel(const float* __restrict__ x, const float* __restrict__ bases,
                               const float* __restrict__ bias, float* __restrict__ y,
                               uint8_t* __restrict__ am, int N, int Cin, int H, int W, int Cout,
                               int K, int NB, int RPB, int pool, int gf, int RO, int act, TapOffsets T) {
  const long long plane = (long long)H * W;
  const long long total = (long long)N * Cout * plane;
  const int KK = K * K;
  const int R = NB * RPB;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int pix = (int)(idx % plane);
    const int co = (int)((idx / plane) % Cout);
    const int n = (int)(idx / (plane * Cout));
    const int py = pix / W, px = pix % W;
    const float bz = bias ? bias[co] : 0.f;
    const float* xn = x + (size_t)n * Cin * plane;
    float best = 0.f;
    int arg = 0;
    for (int o = 0; o < R; ++o) {
      const int b = o / RPB, r = o % RPB;
      const float* wb = bases + ((size_t)b * Cout + co) * Cin * KK;
      float v = 0.f;
      for (int t = 0; t < KK; ++t) {
        const int sy = py + T.di[r][t], sx = px + T.dj[r][t];
        if (sy < 0 || sy >= H || sx < 0 || sx >= W) continue;
        const float* xp = xn + (size_t)sy * W + sx;
        const float* wp = wb + t;
        for (int ci = 0; ci < Cin; ++ci) v = fmaf(wp[(size_t)ci * KK], xp[(size_t)ci * plane], v);
      }
      const int slot = o / gf, k = o % gf;
      fold(pool == RC_POOL_NONE ? RC_POOL_MAX : pool, k, v, best, arg);
      if (k == gf - 1) {
        float outv = pool == RC_POOL_AVG ? best / (float)R : best;
        const size_t off = (((size_t)n * Cout + co) * RO + slot) * plane + pix;
        const float v = outv + bz;
        y[off] = act == RC_ACT_RELU ? fmaxf(v, 0.f) : v;
        if (am && (pool == RC_POOL_MAX || pool == RC_POOL_SUBGROUP)) am[off] = (uint8_t)arg;
      }
    }
  }
}

__global__ void pool_kernel(const float* __restrict__ f, const float* __restrict__ bias,
                            float* __restrict__ y, uint8_t* __restrict__ am, int N, int Cout,
                            int R, int plane, int pool, int gf, int RO) {
  const long long total = (long long)N * Cout * RO * plane;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int pix = (int)(idx % plane);
    const int slot = (int)((idx / plane) % RO);
    const long long nc = idx / ((long long)plane * RO);  // n * Cout + co
    const int co = (int)(nc % Cout);
    const float* src = f + (nc * R + (long long)slot * gf) * plane + pix;
    float best = 0.f;
    int arg = 0;
    for (int k = 0; k < gf; ++k) fold(pool, k, src[(long long)k * plane], best, arg);
    if (pool == RC_POOL_AVG) best = best / (float)R;
    y[idx] = best + (bias ? bias[co] : 0.f);
    if (am && pool != RC_POOL_AVG) am[idx] = (uint8_t)arg;
  }
}

int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  if (g > 148LL * 32) g = 148LL * 32;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

int launch_generic(const rc_desc& d, const float* x, const void* bank, const float* bias,
                   float* y, uint8_t* argmax, cudaStream_t s, const char** name) {
  if (d.k > kMaxK) return RC_ERR_UNSUPPORTED;
  if (name) *name = "generic";
  const long long total = (long long)d.n * d.c_out * d.h * d.w;
  if (total == 0) return RC_OK;
  TapOffsets T;
  slice_tap_offsets(d.k, d.convention, &T);
  const BankLayout L = bank_layout(d);
  const bool has_arg = d.pool == RC_POOL_MAX || d.pool == RC_POOL_SUBGROUP;
  prof_begin(s);
  generic_kernel<<<grid_for(total, 256), 256, 0, s>>>(
      x, reinterpret_cast<const float*>(static_cast<const char*>(bank) + L.bases_off), bias, y,
      has_arg ? argmax : nullptr, d.n, d.c_in, d.h, d.w, d.c_out, d.k, num_bases(d),
      rot_per_base(d), d.pool, pool_fold(d), out_orientations(d), d.activation, T);
  prof_end(s);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

int launch_pool(int n, int c_out, int r, int h, int w, int pool, int g, const float* f,
                const float* bias, float* y, uint8_t* argmax, cudaStream_t s) {
  const int gf = pool == RC_POOL_NONE ? 1 : (pool == RC_POOL_SUBGROUP ? g : r);
  const int ro = r / gf;
  const long long total = (long long)n * c_out * ro * h * w;
  if (total == 0) return RC_OK;
  pool_kernel<<<grid_for(total, 256), 256, 0, s>>>(
      f, bias, y, (pool == RC_POOL_MAX || pool == RC_POOL_SUBGROUP) ? argmax : nullptr, n, c_out,
      r, h * w, pool == RC_POOL_NONE ? RC_POOL_MAX : pool, gf, ro);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

}  // namespace rc
