// rc_internal.cuh -- shared definitions for the sm_100a kernels behind rotconv_c.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "rotconv_c.h"

namespace rc {

// ---- error plumbing (thread-local message, rotconv_c.h "Conventions") ----------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
#define RC_CUDA(call)                                            \
  do {                                                           \
    cudaError_t e_ = (call);                                     \
    if (e_ != cudaSuccess) return ::rc::cuda_fail(e_, #call);    \
  } while (0)

// ---- descriptor helpers ----------------------------------------------------------
inline int num_bases(const rc_desc& d) {
  return d.group == RC_GROUP_P4M ? 2 : (d.group == RC_GROUP_STEER ? d.orientations / 4 : 1);
}
inline int rot_per_base(const rc_desc& d) { return d.group == RC_GROUP_SINGLE ? 1 : 4; }
inline int out_orientations(const rc_desc& d) {
  const int R = num_bases(d) * rot_per_base(d);
  if (d.pool == RC_POOL_NONE) return R;
  if (d.pool == RC_POOL_SUBGROUP) return R / d.pool_group;
  return 1;
}
// group size of the pooling fold: every `g` consecutive orientations reduce to one
inline int pool_fold(const rc_desc& d) {
  const int R = num_bases(d) * rot_per_base(d);
  if (d.pool == RC_POOL_NONE) return 1;
  if (d.pool == RC_POOL_SUBGROUP) return d.pool_group;
  return R;
}
int validate(const rc_desc& d);  // RC_OK or RC_ERR_INVALID + message

// ---- main-kernel timing (rc_profile_enable / rc_profile_collect) -------------------------
// When enabled on the calling thread, every conv launch brackets its MAIN kernel (not the
// operand packing) with a CUDA event pair on the launch stream.
void prof_begin(cudaStream_t s);
void prof_end(cudaStream_t s);

// ---- bank layout (rc_bank_bytes) ---------------------------------------------------
struct BankLayout {
  size_t bases_off, bases_bytes;  // fp32 [B][Cout][Cin][K][K]
  size_t simt_off, simt_bytes;    // K==3 SIMT operand: fp32 [B][Cin][Cout][12] (9 taps + 3 pad)
  size_t tc_off, tc_bytes;        // tcgen05 packed operands (0 if none)
  size_t total;
};
BankLayout bank_layout(const rc_desc& d);

// ---- slice index maps (convention P1) ---------------------------------------------
// For rotation r of a base kernel K_b, the slice kernel read at gather position
// (i, j) is base tap map[i*k+j] (rc_oracle.c rco_slice_tap_map restates the same).
constexpr int kMaxK = 11;
struct TapOffsets {  // per rotation r < 4 and base tap t: gather offset (di, dj)
  int8_t di[4][kMaxK * kMaxK];
  int8_t dj[4][kMaxK * kMaxK];
};
void slice_tap_offsets(int k, int convention, TapOffsets* out);

// ---- kernel launchers ----------------------------------------------------------------
int launch_bank(const rc_desc& d, const float* w0, const float* w1, void* bank,
                cudaStream_t s);
int launch_orientation_bank(const rc_desc& d, const void* bank, float* out, cudaStream_t s);
int launch_steer(const float* fx, const float* fy, size_t count, double theta, float* out, cudaStream_t s);
// returns RC_ERR_UNSUPPORTED if the SIMT K=3 fast kernel cannot handle d
int launch_simt_k3(const rc_desc& d, const float* x, const void* bank, const float* bias,
                   float* y, uint8_t* argmax, cudaStream_t s, bool dry_run, const char** name);
// single-orientation K = 3, Cin <= 32, W in {4, 8, 16, 32} (ri_direct.cu); else RC_ERR_UNSUPPORTED
bool direct_supported(const rc_desc& d);
int launch_direct_k3(const rc_desc& d, const float* x, const void* bank, const float* bias, float* y,
                     uint8_t* am, cudaStream_t s, bool dry_run, const char** name);
int launch_generic(const rc_desc& d, const float* x, const void* bank, const float* bias,
                   float* y, uint8_t* argmax, cudaStream_t s, const char** name);
int launch_pool(int n, int c_out, int r, int h, int w, int pool, int g, const float* f,
                const float* bias, float* y, uint8_t* argmax, cudaStream_t s);
// the forward dispatcher (capi.cu), reused by the backward-input pass
int dispatch_forward(const rc_desc& d, const float* x, const void* bank, const float* bias, float* y,
                     uint8_t* am, void* ws, size_t ws_bytes, cudaStream_t s);
// backward (backward.cu)
size_t bwd_input_ws(const rc_desc& d);
size_t bwd_weight_ws(const rc_desc& d);
int launch_pool_backward(const rc_desc& d, const float* gy, const uint8_t* am, float* df, cudaStream_t s);
int launch_bwd_input(const rc_desc& d, const float* df, const void* bank, float* dx, void* ws, cudaStream_t s);
int launch_bwd_weight(const rc_desc& d, const float* x, const float* df, float* dw0, float* dw1, void* ws,
                      cudaStream_t s);
int launch_relu_backward(const float* y, float* gy, long long n, cudaStream_t s);
int launch_bias_backward(const float* gy, float* db, int n, int cout, long long per, cudaStream_t s);
// stack glue (stack.cu)
int launch_maxpool2x2(int n, int c, int h, int w, const float* x, float* y, cudaStream_t s);
int launch_gap_linear(int n, int c, int h, int w, const float* x, const float* wc, const float* bc, int classes,
                      float* out, cudaStream_t s);

}  // namespace rc

namespace rc {
// tensor-core path (ri_tc.cu)
bool tc_supported(const rc_desc& d);
size_t tc_bank_bytes(const rc_desc& d);
size_t tc_workspace_bytes(const rc_desc& d);
int launch_tc_wpack(const rc_desc& d, const float* bases, uint8_t* tc_section, cudaStream_t s);
int launch_tc(const rc_desc& d, const float* x, const void* bank, const float* bias, float* y, uint8_t* am,
              void* ws, size_t ws_bytes, cudaStream_t s, bool dry_run, const char** name);
// single-orientation implicit GEMM (ri_igemm.cu), reached through launch_tc
bool igemm_supported(const rc_desc& d);
size_t igemm_workspace_bytes(const rc_desc& d);
int launch_igemm(const rc_desc& d, const float* x, const uint8_t* wpk, const uint8_t* whi, const float* bias,
                 float* y, uint8_t* am, void* ws, cudaStream_t s);
// zero-padded pixel-row planes of X (ri_igemm.cu): plane c = [rows][64 ci] bf16 SW128 rows,
// row G + q for padded pixel q = n*Pimg + (h+1)*Wp + (w+1); hi and (xl != null) lo parts
struct PadGeom {
  int Wp, G, Pimg, NC;
  long long rows;
};
PadGeom pad_geom(const rc_desc& d);
size_t pad_planes_bytes(const rc_desc& d, int parts);
int launch_pad_pack(const rc_desc& d, const float* x, uint8_t* xh, uint8_t* xl, cudaStream_t s);
// weight gradient on the tensor cores (ri_wgrad.cu): dF[m][ci*9 + pos] for K = 3
bool wgrad_supported(const rc_desc& d);
size_t wgrad_ws_bytes(const rc_desc& d);
int launch_wgrad(const rc_desc& d, const float* x, const float* df, float* dF, void* ws, cudaStream_t s);
}  // namespace rc
