// backward.cu -- gradients of the RI layer (SPEC backward module).
//
// Notation (convention P1): slice o = (b, r) of the forward is the gather-"same" conv
//   Y_o[co, p] = sum_{ci, pos} F_o[co, ci, pos] * X[ci, p + off(pos)],
//   F_o[co, ci, pos] = K_b[co, ci, t]  with  pos = pos_r(t)   (slice_tap_offsets: the tap t
//   of base K_b lands at gather offset (di, dj) = off(pos) for rotation r).
// Then, for an upstream gradient D_o = dL/dY_o (after pool backward):
//   dX[ci, q]        = sum_o sum_{co,pos} F_o[co, ci, pos] * D_o[co, q - off(pos)]      (Eq. 13+15)
//                    = conv_gather_same(D as (Cout*R) channels, Wt)  with
//                      Wt[ci, co*R + o, pos'] = F_o[co, ci, K*K-1-pos']  (flip + transpose):
//                      one single-orientation forward of this library (raw convention);
//   dF_o[co,ci,pos]  = sum_{n,p} D_o[co, p] * X[ci, p + off(pos)]                          (Eq. 14)
//                      = one GEMM per image over im2col(X) (cuBLAS SGEMM, FP32);
//   dK_b[co,ci,t]    = sum_r dF_{b,r}[co, ci, pos_r(t)]                                   (Eq. 16)
//   parameters       : W = K_0 (single, p4);  W += mirror(dK_1) (p4m);
//                      f_x = sum_b sin(theta_b) dK_b, f_y = sum_b cos(theta_b) dK_b (steer).
// Pool backward (Eq. 11/12): avg spreads G/R, max / subgroup route G to the stored argmax
// (the forward tie rule, smallest index); bias and ReLU backward are elementwise.
#include <cublas_v2.h>

#include <cmath>
#include <mutex>
#include <vector>

#include "rc_internal.cuh"

namespace rc {
namespace {

int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  if (g > 148LL * 32) g = 148LL * 32;
  return (int)(g < 1 ? 1 : g);
}

// gy (N, Cout, RO, H, W) -> df (N, Cout, R, H, W)
__global__ void pool_backward_kernel(const float* __restrict__ gy, const uint8_t* __restrict__ am,
                                     float* __restrict__ df, long long planes_nc, int R, int RO, int plane,
                                     int pool, int gf) {
  const long long total = planes_nc * R * plane;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int px = (int)(i % plane);
    const int o = (int)((i / plane) % R);
    const long long nc = i / ((long long)plane * R);
    float v;
    if (pool == RC_POOL_NONE) {
      v = gy[(nc * RO + o) * plane + px];
    } else if (pool == RC_POOL_AVG) {
      v = gy[nc * RO * plane + px] / (float)R;
    } else {  // max (gf == R, RO == 1) / subgroup (blocks of gf): the argmax slot gets G
      const int slot = o / gf, kk = o % gf;
      const long long src = (nc * RO + slot) * plane + px;
      v = (am[src] == kk) ? gy[src] : 0.f;
    }
    df[i] = v;
  }
}

// the same, 4 pixels per thread (plane % 4 == 0): one index decode per float4, 128-bit
// loads / stores, uchar4 argmax reads
template <typename IT>  // index type: 32-bit division when the tensor allows it
__global__ void pool_backward_vec_kernel(const float4* __restrict__ gy, const uchar4* __restrict__ am,
                                         float4* __restrict__ df, long long planes_nc, int R, int RO, int plane4,
                                         int pool, int gf, float inv_r) {
  const IT total = (IT)(planes_nc * R * plane4);
  for (IT i = blockIdx.x * (IT)blockDim.x + threadIdx.x; i < total; i += (IT)gridDim.x * blockDim.x) {
    const IT pi = i / (IT)plane4;  // (nc, o) plane
    const int px = (int)(i - pi * (IT)plane4);
    const int o = (int)(pi % (IT)R);
    const long long nc = (long long)(pi / (IT)R);
    float4 v;
    if (pool == RC_POOL_NONE) {
      v = gy[(nc * RO + o) * plane4 + px];
    } else if (pool == RC_POOL_AVG) {
      const float4 g = gy[nc * RO * plane4 + px];
      v = make_float4(g.x * inv_r, g.y * inv_r, g.z * inv_r, g.w * inv_r);
    } else {
      const int slot = o / gf, kk = o % gf;
      const long long src = (nc * RO + slot) * plane4 + px;
      const float4 g = gy[src];
      const uchar4 a = am[src];
      v = make_float4(a.x == kk ? g.x : 0.f, a.y == kk ? g.y : 0.f, a.z == kk ? g.z : 0.f, a.w == kk ? g.w : 0.f);
    }
    df[i] = v;
  }
}

// gy *= (y > 0) in place (ReLU backward from the forward output)
__global__ void relu_backward_kernel(const float* __restrict__ y, float* __restrict__ gy, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!(y[i] > 0.f)) gy[i] = 0.f;
}

// dbias[co] = sum over (n, ro, px) of gy; one CTA per co
__global__ void bias_backward_kernel(const float* __restrict__ gy, float* __restrict__ db, int N, int Cout,
                                     long long per) {
  const int co = blockIdx.x;
  double s = 0.0;
  for (int n = 0; n < N; ++n) {
    const float* p = gy + ((size_t)n * Cout + co) * per;
    for (long long i = threadIdx.x; i < per; i += blockDim.x) s += p[i];
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) db[co] = (float)red[0];
}

// Wt[ci][co*R + o][pos'] = F_o[co][ci][KK-1-pos'] = K_b[co][ci][t] with pos_r(t) = KK-1-pos'
__global__ void bwd_input_weights_kernel(const float* __restrict__ bases, float* __restrict__ wt, int Cout,
                                         int Cin, int K, int NB, int RPB, TapOffsets T) {
  const int KK = K * K, R = NB * RPB, c = K / 2;
  const long long total = (long long)Cin * Cout * R * KK;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(i % KK);  // base tap
    const int o = (int)((i / KK) % R);
    const int co = (int)((i / ((long long)KK * R)) % Cout);
    const int ci = (int)(i / ((long long)KK * R * Cout));
    const int b = o / RPB, r = o % RPB;
    const int pos = (T.di[r][t] + c) * K + (T.dj[r][t] + c);
    wt[(((size_t)ci * Cout + co) * R + o) * KK + (KK - 1 - pos)] =
        bases[(((size_t)b * Cout + co) * Cin + ci) * KK + t];
  }
}

// cols[p][ci*KK + pos] = X[ci, p + off(pos)] (zero padded), one image
__global__ void im2col_kernel(const float* __restrict__ x, float* __restrict__ cols, int Cin, int H, int W, int K) {
  const int KK = K * K, c = K / 2;
  const long long total = (long long)H * W * Cin * KK;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int pos = (int)(i % KK);
    const int ci = (int)((i / KK) % Cin);
    const long long p = i / ((long long)KK * Cin);
    const int py = (int)(p / W), px = (int)(p % W);
    const int sy = py + pos / K - c, sx = px + pos % K - c;
    cols[i] = (sy >= 0 && sy < H && sx >= 0 && sx < W) ? x[((size_t)ci * H + sy) * W + sx] : 0.f;
  }
}

// dF (Cout*R rows ordered (co, o), Cin*KK cols) -> parameter gradients (Eq. 16 + chain rule)
struct SteerCo {
  float s[64], c[64];
};
__global__ void param_grad_kernel(const float* __restrict__ dF, float* __restrict__ dw0, float* __restrict__ dw1,
                                  int Cout, int Cin, int K, int NB, int RPB, int group, TapOffsets T, SteerCo sc) {
  const int KK = K * K, R = NB * RPB, c = K / 2;
  const long long total = (long long)Cout * Cin * KK;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(i % KK);
    const int ci = (int)((i / KK) % Cin);
    const int co = (int)(i / ((long long)KK * Cin));
    float g0 = 0.f, g1 = 0.f;
    for (int b = 0; b < NB; ++b) {
      // dK_b at tap tb; for p4m base 1 the parameter tap t reads mirror(W): tb = mirrored t
      const int tb = (group == RC_GROUP_P4M && b == 1) ? (t / K) * K + (K - 1 - t % K) : t;
      float dk = 0.f;
      for (int r = 0; r < RPB; ++r) {
        const int o = b * RPB + r;
        const int pos = (T.di[r][tb] + c) * K + (T.dj[r][tb] + c);
        dk += dF[((size_t)co * R + o) * ((size_t)Cin * KK) + (size_t)ci * KK + pos];
      }
      if (group == RC_GROUP_STEER) {
        g0 += sc.s[b] * dk;
        g1 += sc.c[b] * dk;
      } else {
        g0 += dk;
      }
    }
    dw0[i] = g0;
    if (group == RC_GROUP_STEER && dw1) dw1[i] = g1;
  }
}

struct CublasHandles {
  std::mutex mu;
  cublasHandle_t h[64] = {};
};
CublasHandles g_cublas;

}  // namespace

// ---- workspace plans -----------------------------------------------------------------
// backward-input: Wt (Cin x Cout*R x KK floats) + the single-orientation bank of Wt + its
// forward workspace
static rc_desc bwd_input_desc(const rc_desc& d) {
  rc_desc s = d;
  s.c_in = d.c_out * num_bases(d) * rot_per_base(d);
  s.c_out = d.c_in;
  s.group = RC_GROUP_SINGLE;
  s.orientations = 1;
  s.pool = RC_POOL_NONE;
  s.pool_group = 1;
  s.convention = RC_CONV_RAW;
  s.activation = RC_ACT_NONE;
  return s;
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

size_t bwd_input_ws(const rc_desc& d) {
  const rc_desc s = bwd_input_desc(d);
  const size_t wt = align256((size_t)s.c_out * s.c_in * d.k * d.k * sizeof(float));
  return wt + align256(bank_layout(s).total) + align256(tc_workspace_bytes(s));
}

size_t bwd_weight_ws(const rc_desc& d) {
  const int R = num_bases(d) * rot_per_base(d);
  const size_t dF = (size_t)d.c_out * R * d.c_in * d.k * d.k * sizeof(float);
  if (wgrad_supported(d)) return align256(dF) + wgrad_ws_bytes(d);  // tensor-core implicit GEMM
  const size_t cols = (size_t)d.h * d.w * d.c_in * d.k * d.k * sizeof(float);
  return align256(cols) + align256(dF);
}

int launch_pool_backward(const rc_desc& d, const float* gy, const uint8_t* am, float* df, cudaStream_t s) {
  const int R = num_bases(d) * rot_per_base(d), RO = out_orientations(d), plane = d.h * d.w;
  const long long work = (long long)d.n * d.c_out * R * plane;
  if (work == 0) return RC_OK;
  const bool pow2 = (R & (R - 1)) == 0;  // x / R == x * (1/R) exactly
  if (plane % 4 == 0 && (d.pool != RC_POOL_AVG || pow2))
  {
    if (work / 4 < (1LL << 31))
      pool_backward_vec_kernel<unsigned><<<grid_for(work / 4, 256), 256, 0, s>>>(
          reinterpret_cast<const float4*>(gy), reinterpret_cast<const uchar4*>(am), reinterpret_cast<float4*>(df),
          (long long)d.n * d.c_out, R, RO, plane / 4, d.pool, pool_fold(d), 1.0f / (float)R);
    else
      pool_backward_vec_kernel<unsigned long long><<<grid_for(work / 4, 256), 256, 0, s>>>(
          reinterpret_cast<const float4*>(gy), reinterpret_cast<const uchar4*>(am), reinterpret_cast<float4*>(df),
          (long long)d.n * d.c_out, R, RO, plane / 4, d.pool, pool_fold(d), 1.0f / (float)R);
  }
  else
    pool_backward_kernel<<<grid_for(work, 256), 256, 0, s>>>(gy, am, df, (long long)d.n * d.c_out, R, RO, plane,
                                                            d.pool, pool_fold(d));
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

int launch_bwd_input(const rc_desc& d, const float* df, const void* bank, float* dx, void* ws, cudaStream_t s) {
  const rc_desc sd = bwd_input_desc(d);
  const size_t wtb = align256((size_t)sd.c_out * sd.c_in * d.k * d.k * sizeof(float));
  float* wt = static_cast<float*>(ws);
  void* sbank = static_cast<char*>(ws) + wtb;
  void* sws = static_cast<char*>(sbank) + align256(bank_layout(sd).total);
  TapOffsets T;
  slice_tap_offsets(d.k, d.convention, &T);
  const BankLayout L = bank_layout(d);
  const long long work = (long long)sd.c_out * sd.c_in * d.k * d.k;
  bwd_input_weights_kernel<<<grid_for(work, 256), 256, 0, s>>>(
      reinterpret_cast<const float*>(static_cast<const char*>(bank) + L.bases_off), wt, d.c_out, d.c_in, d.k,
      num_bases(d), rot_per_base(d), T);
  RC_CUDA(cudaGetLastError());
  int st = launch_bank(sd, wt, nullptr, sbank, s);
  if (st != RC_OK) return st;
  return dispatch_forward(sd, df, sbank, nullptr, dx, nullptr, sws, tc_workspace_bytes(sd), s);
}

static int param_grad(const rc_desc& d, const float* dF, float* dw0, float* dw1, cudaStream_t s);

int launch_bwd_weight(const rc_desc& d, const float* x, const float* df, float* dw0, float* dw1, void* ws,
                      cudaStream_t s) {
  const int R = num_bases(d) * rot_per_base(d), KK = d.k * d.k;
  if (wgrad_supported(d)) {  // bf16 / bf16x3 / auto: one tcgen05 implicit GEMM over the batch
    float* dF = static_cast<float*>(ws);
    const size_t dFb = align256((size_t)d.c_out * R * d.c_in * KK * sizeof(float));
    const int st = launch_wgrad(d, x, df, dF, static_cast<char*>(ws) + dFb, s);
    if (st != RC_OK) return st;
    return param_grad(d, dF, dw0, dw1, s);
  }
  const size_t colsb = align256((size_t)d.h * d.w * d.c_in * KK * sizeof(float));
  float* cols = static_cast<float*>(ws);
  float* dF = reinterpret_cast<float*>(static_cast<char*>(ws) + colsb);
  int dev = 0;
  RC_CUDA(cudaGetDevice(&dev));
  cublasHandle_t h;
  {
    std::lock_guard<std::mutex> lock(g_cublas.mu);
    if (!g_cublas.h[dev] && cublasCreate(&g_cublas.h[dev]) != CUBLAS_STATUS_SUCCESS)
      return fail(RC_ERR_CUDA, "ri_conv_backward: cublasCreate failed");
    h = g_cublas.h[dev];
  }
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return fail(RC_ERR_CUDA, "ri_conv_backward: cublasSetStream");
  cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);  // true FP32 (no TF32): the weight gradient keeps FP32 tolerance
  const int M = d.c_out * R, Kd = d.h * d.w, Ncol = d.c_in * KK;
  const size_t plane = (size_t)d.h * d.w;
  RC_CUDA(cudaMemsetAsync(dF, 0, (size_t)M * Ncol * sizeof(float), s));
  for (int n = 0; n < d.n; ++n) {
    const long long work = (long long)Kd * Ncol;
    im2col_kernel<<<grid_for(work, 256), 256, 0, s>>>(x + (size_t)n * d.c_in * plane, cols, d.c_in, d.h, d.w, d.k);
    RC_CUDA(cudaGetLastError());
    // row-major dF[M x Ncol] += D_n[M x Kd] * cols[Kd x Ncol]  ==  column-major
    // dF^T[Ncol x M] += cols^T[Ncol x Kd] * D_n^T[Kd x M]
    const float one = 1.f;
    const cublasStatus_t cs = cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, Ncol, M, Kd, &one, cols, Ncol,
                                          df + (size_t)n * M * plane, Kd, &one, dF, Ncol);
    if (cs != CUBLAS_STATUS_SUCCESS) return fail(RC_ERR_CUDA, "ri_conv_backward: cublasSgemm failed");
  }
  return param_grad(d, dF, dw0, dw1, s);
}

// dF -> parameter gradients: inverse rotations (Eq. 16) and the mirror / steer chain rule
static int param_grad(const rc_desc& d, const float* dF, float* dw0, float* dw1, cudaStream_t s) {
  const int KK = d.k * d.k;
  TapOffsets T;
  slice_tap_offsets(d.k, d.convention, &T);
  SteerCo sc{};
  for (int b = 0; b < num_bases(d) && b < 64; ++b) {
    const double th = 2.0 * M_PI * (double)b / (double)d.orientations;
    sc.s[b] = (float)std::sin(th);
    sc.c[b] = (float)std::cos(th);
  }
  const long long work = (long long)d.c_out * d.c_in * KK;
  param_grad_kernel<<<grid_for(work, 256), 256, 0, s>>>(dF, dw0, dw1, d.c_out, d.c_in, d.k, num_bases(d),
                                                        rot_per_base(d), d.group, T, sc);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

int launch_relu_backward(const float* y, float* gy, long long n, cudaStream_t s) {
  if (n == 0) return RC_OK;
  relu_backward_kernel<<<grid_for(n, 256), 256, 0, s>>>(y, gy, n);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

int launch_bias_backward(const float* gy, float* db, int n, int cout, long long per, cudaStream_t s) {
  bias_backward_kernel<<<cout, 256, 0, s>>>(gy, db, n, cout, per);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

}  // namespace rc
