// bank.cu -- rotated-filter-bank precompute (SPEC:439-456 steer/build_orientation_bank,
// SPEC:256-264 transform_kernel, tensor.hpp:348-370 rot90/mirror).
//
// The conv kernels never see R rotated banks: rotations are index maps (rc_internal.cuh
// TapOffsets / compile-time tables in ri_simt.cu).  This kernel only builds the B base
// kernels K_b (steered first-quadrant angles, or W / mirror(W)) and the kernel-specific
// operand layouts.  It is elementwise and HBM-bound, <<1% of the layer.
#include <cmath>

#include "rc_internal.cuh"

namespace rc {
namespace {

constexpr int kMaxBases = 64;  // R <= 256
struct SteerCoeffs {
  float s[kMaxBases], c[kMaxBases];
};

// One thread per (b, ci, co) row of K*K taps.  Writes the FilterBank-layout base
// (section 0) and, for K == 3, the SIMT operand layout [B][Cin][Cout][12] (section 1).
__global__ void bank_kernel(const float* __restrict__ w0, const float* __restrict__ w1,
                            float* __restrict__ bases, float* __restrict__ simt, int nb,
                            int cout, int cin, int k, int group, SteerCoeffs co_) {
  const long long total = (long long)nb * cin * cout;
  const int kk = k * k;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int co = (int)(idx % cout);
    const int ci = (int)((idx / cout) % cin);
    const int b = (int)(idx / ((long long)cout * cin));
    const size_t src = ((size_t)co * cin + ci) * kk;
    float v[kMaxK * kMaxK];
    for (int t = 0; t < kk; ++t) {
      float val;
      if (group == RC_GROUP_STEER) {
        // SPEC:439-447 sin(theta)*f_x + cos(theta)*f_y, each op rounded separately
        // (no FMA) so the bank is bit-identical to the oracle's rco_steer.
        val = __fadd_rn(__fmul_rn(co_.s[b], w0[src + t]), __fmul_rn(co_.c[b], w1[src + t]));
      } else if (group == RC_GROUP_P4M && b == 1) {
        const int i = t / k, j = t % k;  // tensor.hpp:363-370 mirror_plane
        val = w0[src + i * k + (k - 1 - j)];
      } else {
        val = w0[src + t];
      }
      v[t] = val;
    }
    float* dst = bases + ((size_t)b * cout + co) * cin * kk + (size_t)ci * kk;
    for (int t = 0; t < kk; ++t) dst[t] = v[t];
    if (simt != nullptr) {  // K == 3
      float4* s4 = reinterpret_cast<float4*>(simt + (((size_t)b * cin + ci) * cout + co) * 12);
      s4[0] = make_float4(v[0], v[1], v[2], v[3]);
      s4[1] = make_float4(v[4], v[5], v[6], v[7]);
      s4[2] = make_float4(v[8], 0.f, 0.f, 0.f);
    }
  }
}

// K == 3: one CTA per (base b, 32 output channels, 32 input channels), staged through shared
// memory so both HBM sides are coalesced: the [co][ci][9] rows of the weights and of the
// FilterBank-layout bases are contiguous 32 x 9-float runs per channel, and the SIMT operand
// [B][Cin][Cout][12] is written as contiguous 32 x 12-float runs per input channel (the
// per-thread kernel above reads and writes 36-byte pieces strided by Cin x 9 floats).
constexpr int BT = 32;
__global__ void __launch_bounds__(256) bank_k3_tiled_kernel(const float* __restrict__ w0, const float* __restrict__ w1,
                                                            float* __restrict__ bases, float* __restrict__ simt,
                                                            int cout, int cin, int group, SteerCoeffs co_) {
  __shared__ float tile[BT][BT * 9 + 1];  // [co_l][ci_l * 9 + t]
  const int b = blockIdx.z, co0 = blockIdx.y * BT, ci0 = blockIdx.x * BT;
  const int nco = min(BT, cout - co0), nci = min(BT, cin - ci0);
  for (int e = threadIdx.x; e < BT * BT * 9; e += blockDim.x) {
    const int col = e / (BT * 9), rem = e % (BT * 9), cil = rem / 9, t = rem % 9;
    if (col >= nco || cil >= nci) continue;
    const size_t src = ((size_t)(co0 + col) * cin + ci0 + cil) * 9;
    float val;
    if (group == RC_GROUP_STEER)  // SPEC:439-447, each op rounded (bit-identical to rco_steer)
      val = __fadd_rn(__fmul_rn(co_.s[b], w0[src + t]), __fmul_rn(co_.c[b], w1[src + t]));
    else if (group == RC_GROUP_P4M && b == 1)
      val = w0[src + (t / 3) * 3 + (2 - t % 3)];  // tensor.hpp:363-370 mirror_plane
    else
      val = w0[src + t];
    tile[col][rem] = val;
    bases[((size_t)b * cout + co0 + col) * cin * 9 + (size_t)(ci0 + cil) * 9 + t] = val;
  }
  if (simt == nullptr) return;
  __syncthreads();
  for (int e = threadIdx.x; e < BT * BT * 12; e += blockDim.x) {
    const int cil = e / (BT * 12), rem = e % (BT * 12), col = rem / 12, j = rem % 12;
    if (col >= nco || cil >= nci) continue;
    simt[(((size_t)b * cin + ci0 + cil) * cout + co0 + col) * 12 + j] = j < 9 ? tile[col][cil * 9 + j] : 0.f;
  }
}

struct RotMaps {
  int8_t src[4][kMaxK * kMaxK];
};

// build_orientation_bank: kernels[o = b*rpb + r] = rot90^r(K_b) (raw rotation, no reverse)
__global__ void orient_bank_kernel(const float* __restrict__ bases, float* __restrict__ out,
                                   int nb, int rpb, int cout, int cin, int k, RotMaps maps) {
  const int kk = k * k;
  const long long per = (long long)cout * cin * kk;
  const long long total = per * nb * rpb;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int pos = (int)(idx % kk);
    const long long plane = (idx / kk) % ((long long)cout * cin);
    const int o = (int)(idx / per);
    const int b = o / rpb, r = o % rpb;
    out[idx] = bases[(long long)b * per + plane * kk + maps.src[r][pos]];
  }
}

// steer at an arbitrary angle: same rounding as bank_kernel
__global__ void steer_kernel(const float* __restrict__ fx, const float* __restrict__ fy, float* __restrict__ out,
                             long long count, float sn, float cs) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = __fadd_rn(__fmul_rn(sn, fx[i]), __fmul_rn(cs, fy[i]));
}

int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  if (g > 148LL * 16) g = 148LL * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

int launch_bank(const rc_desc& d, const float* w0, const float* w1, void* bank, cudaStream_t s) {
  const BankLayout L = bank_layout(d);
  const int nb = num_bases(d);
  SteerCoeffs c{};
  for (int b = 0; b < nb && b < kMaxBases; ++b) {
    const double theta = 2.0 * M_PI * (double)b / (double)d.orientations;
    c.s[b] = (float)std::sin(theta);  // coefficients in double, rounded once (rco_steer)
    c.c[b] = (float)std::cos(theta);
  }
  char* base = static_cast<char*>(bank);
  float* simt = L.simt_bytes ? reinterpret_cast<float*>(base + L.simt_off) : nullptr;
  const long long work = (long long)nb * d.c_in * d.c_out;
  if (work == 0) return RC_OK;
  if (d.k == 3) {
    const dim3 grid((d.c_in + BT - 1) / BT, (d.c_out + BT - 1) / BT, nb);
    bank_k3_tiled_kernel<<<grid, 256, 0, s>>>(w0, d.group == RC_GROUP_STEER ? w1 : w0,
                                               reinterpret_cast<float*>(base + L.bases_off), simt, d.c_out, d.c_in,
                                               d.group, c);
  } else {
    bank_kernel<<<grid_for(work, 256), 256, 0, s>>>(
        w0, d.group == RC_GROUP_STEER ? w1 : w0, reinterpret_cast<float*>(base + L.bases_off), simt,
        nb, d.c_out, d.c_in, d.k, d.group, c);
  }
  RC_CUDA(cudaGetLastError());
  if (L.tc_bytes)  // tcgen05 operand tiles (bf16 hi/lo, SW128) from the fp32 bases
    return launch_tc_wpack(d, reinterpret_cast<const float*>(base + L.bases_off),
                           reinterpret_cast<uint8_t*>(base + L.tc_off), s);
  return RC_OK;
}

int launch_steer(const float* fx, const float* fy, size_t count, double theta, float* out, cudaStream_t s) {
  if (count == 0) return RC_OK;
  steer_kernel<<<grid_for((long long)count, 256), 256, 0, s>>>(fx, fy, out, (long long)count,
                                                               (float)std::sin(theta), (float)std::cos(theta));
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

int launch_orientation_bank(const rc_desc& d, const void* bank, float* out, cudaStream_t s) {
  const BankLayout L = bank_layout(d);
  RotMaps m{};
  TapOffsets unused;
  (void)unused;
  const int k = d.k, kk = k * k;
  for (int r = 0; r < 4; ++r) {
    // rot90^r of the id plane: one CCW turn reads in[j][k-1-i] (tensor.hpp:348-360)
    int cur[kMaxK * kMaxK], nxt[kMaxK * kMaxK];
    for (int t = 0; t < kk; ++t) cur[t] = t;
    for (int q = 0; q < r; ++q) {
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) nxt[i * k + j] = cur[j * k + (k - 1 - i)];
      for (int t = 0; t < kk; ++t) cur[t] = nxt[t];
    }
    for (int t = 0; t < kk; ++t) m.src[r][t] = (int8_t)cur[t];
  }
  const long long total = (long long)d.c_out * d.c_in * kk * num_bases(d) * rot_per_base(d);
  if (total == 0) return RC_OK;
  orient_bank_kernel<<<grid_for(total, 256), 256, 0, s>>>(
      reinterpret_cast<const float*>(static_cast<const char*>(bank) + L.bases_off), out,
      num_bases(d), rot_per_base(d), d.c_out, d.c_in, k, m);
  RC_CUDA(cudaGetLastError());
  return RC_OK;
}

}  // namespace rc
