// stack.cu -- glue kernels of the multi-layer RI classifier (config C5).
//
// The paper's base block (SPEC train_demo MicroNet) is an
// RI conv (subgroup-4 max pooling) followed by a standard conv; the U-Net around it
// down-samples with 2x2 max pooling and the classifier ends in global average pooling and a
// 1x1 head.  None of these ops is in the reference; they are builder-defined
// and run here as small HBM-bound kernels between the fused conv launches:
//   maxpool2x2_kernel  : (N, C, H, W) -> (N, C, H/2, W/2), float4 reads of two rows
//   gap_linear_kernel  : (N, C, H, W) -> mean over H*W -> logits = feat @ Wc^T + bc
#include "rc_internal.cuh"

namespace rc {
namespace {

// one thread per output pair of pixels (2 outputs from a 4-wide window of two input rows)
__global__ void maxpool2x2_kernel(const float* __restrict__ x, float* __restrict__ y, long long planes, int H,
                                  int W) {
  const int Ho = H / 2, Wo = W / 2;
  const long long total = planes * Ho * (Wo / 2);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int xo = (int)(i % (Wo / 2)) * 2;
    const long long r = i / (Wo / 2);
    const int yo = (int)(r % Ho);
    const long long pl = r / Ho;
    const float* src = x + (pl * H + 2 * yo) * W + 2 * xo;
    const float4 a = *reinterpret_cast<const float4*>(src);
    const float4 b = *reinterpret_cast<const float4*>(src + W);
    float2 o;
    o.x = fmaxf(fmaxf(a.x, a.y), fmaxf(b.x, b.y));
    o.y = fmaxf(fmaxf(a.z, a.w), fmaxf(b.z, b.w));
    *reinterpret_cast<float2*>(y + (pl * Ho + yo) * Wo + xo) = o;
  }
}

// one CTA per image: channel means in shared memory, then the classifier rows
__global__ void gap_linear_kernel(const float* __restrict__ x, const float* __restrict__ wc,
                                  const float* __restrict__ bc, float* __restrict__ out, int C, int HW,
                                  int classes) {
  extern __shared__ float feat[];
  const int n = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const float inv = 1.0f / (float)HW;
  for (int c = warp; c < C; c += nw) {
    const float* p = x + ((size_t)n * C + c) * HW;
    float s = 0.f;
    for (int i = lane; i < HW; i += 32) s += p[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) feat[c] = s * inv;
  }
  __syncthreads();
  for (int k = warp; k < classes; k += nw) {
    const float* wr = wc + (size_t)k * C;
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s = fmaf(wr[c], feat[c], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[(size_t)n * classes + k] = s + (bc ? bc[k] : 0.f);
  }
}

}  // namespace

int launch_maxpool2x2(int n, int c, int h, int w, const float* x, float* y, cudaStream_t s) {
  const long long work = (long long)n * c * (h / 2) * (w / 4);
  if (work == 0) return RC_OK;
  long long grid = (work + 255) / 256;
  if (grid > 148LL * 32) grid = 148LL * 32;
  maxpool2x2_kernel<<<(int)grid, 256, 0, s>>>(x, y, (long long)n * c, h, w);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

int launch_gap_linear(int n, int c, int h, int w, const float* x, const float* wc, const float* bc, int classes,
                      float* out, cudaStream_t s) {
  if (n == 0) return RC_OK;
  gap_linear_kernel<<<n, 256, c * sizeof(float), s>>>(x, wc, bc, out, c, h * w, classes);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

}  // namespace rc

using namespace rc;

extern "C" {

int rc_maxpool2x2(int n, int c, int h, int w, const float* d_x, float* d_y, void* stream) {
  if (n < 0 || c < 1 || h < 2 || w < 4 || h % 2 || w % 4)
    return fail(RC_ERR_INVALID, "maxpool2x2: need n >= 0, c >= 1, even H >= 2, W a multiple of 4");
  if (n > 0 && (!d_x || !d_y)) return fail(RC_ERR_INVALID, "maxpool2x2: null pointer");
  return launch_maxpool2x2(n, c, h, w, d_x, d_y, static_cast<cudaStream_t>(stream));
}

int rc_gap_linear(int n, int c, int h, int w, const float* d_x, const float* d_wc, const float* d_bc, int classes,
                  float* d_out, void* stream) {
  if (n < 0 || c < 1 || h < 1 || w < 1 || classes < 1 || c > 12288)
    return fail(RC_ERR_INVALID, "gap_linear: need n >= 0, 1 <= c <= 12288, h, w, classes >= 1");
  if (n > 0 && (!d_x || !d_wc || !d_out)) return fail(RC_ERR_INVALID, "gap_linear: null pointer");
  return launch_gap_linear(n, c, h, w, d_x, d_wc, d_bc, classes, d_out, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
