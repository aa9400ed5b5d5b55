/*
 * rotconv_c.h -- C-ABI of the B200 rotation-invariant scatter convolution
 * (librotconv_b200.so).  Plain pointers, sizes and ints; no torch or C++ types.
 *
 * This is the boundary the reference-side bindings would link against: the
 * reference path is the header-only C++ API in /root/reference/proj/include
 * (namespace rotconv) plus the SPEC-defined group/steerable ops that have no
 * shipped code.  Each entry point below names the reference interface it
 * replaces; include/rotconv/*.hpp re-exposes the reference's C++ signatures on
 * top of this ABI (the drop-in), INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Layouts are the reference containers' (tensor.hpp): a batch of N Tensor3
 *    (C,H,W) is NCHW; FilterBank is (Cout,Cin,K,K); OrientedFeature is (Cout,R,H,W)
 *    per image.  Pooled outputs are (N, Cout, R', H, W) with R' = 1 (avg/max),
 *    R/g (subgroup) or R (none).  Argmax maps are uint8 in the same order.
 *  - Orientation order is orbit-major o = b*4 + r (convention P2);
 *    slice o is scatter_conv_multi(X, rot90^r(K_b)) (P1).
 *  - Every function returns RC_OK (0) or a negative status; rc_last_error()
 *    returns the thread-local message.  Precondition failures use the
 *    reference's own message strings (e.g. "tiled_scatter_conv: invalid halo",
 *    scatter_conv.hpp:345).  No exception crosses the ABI.
 *  - Device entry points (rc_*) take device pointers and a cudaStream_t (as
 *    void*); they never synchronise.  *_host entry points take host pointers,
 *    own their device staging, and return after the result is on the host.
 *  - Thread-safe: no global mutable state except the thread-local error string
 *    and a per-device cache of staging buffers guarded by a mutex.
 */
#ifndef ROTCONV_C_H
#define ROTCONV_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RC_ABI_VERSION 3

enum rc_status {
  RC_OK = 0,
  RC_ERR_INVALID = -1,     /* precondition failure (reference message) */
  RC_ERR_CUDA = -2,        /* CUDA runtime / launch failure */
  RC_ERR_UNSUPPORTED = -3, /* valid request this build has no kernel for */
  RC_ERR_WORKSPACE = -4    /* workspace too small */
};

/* SPEC:250-253 GroupSpec, SPEC:433-436 OrientationSet */
enum rc_group { RC_GROUP_SINGLE = 0, RC_GROUP_P4 = 1, RC_GROUP_P4M = 2, RC_GROUP_STEER = 3 };
/* SPEC:283-309 */
enum rc_pool { RC_POOL_NONE = 0, RC_POOL_AVG = 1, RC_POOL_MAX = 2, RC_POOL_SUBGROUP = 3 };
/* scatter = scatter_conv_multi semantics (scatter_conv.hpp:189-193);
 * raw = scatter_conv_raw_multi semantics (scatter_conv.hpp:151-187) */
enum rc_convention { RC_CONV_SCATTER = 0, RC_CONV_RAW = 1 };
/* arithmetic of the channel contraction:
 *   FP32     -- CUDA-core FP32 FFMA (the parity path)
 *   BF16X3   -- tcgen05 tensor cores, operands split hi+lo bf16, 3 products, FP32 accumulate
 *   BF16     -- tcgen05 tensor cores, one bf16 product, FP32 accumulate
 *   AUTO     -- fastest kernel that meets the FP32 tolerance for the shape */
enum rc_precision { RC_PREC_AUTO = 0, RC_PREC_FP32 = 1, RC_PREC_BF16X3 = 2, RC_PREC_BF16 = 3 };
/* activation fused after the bias (the last op of the epilogue; not in the reference --
 * used by the multi-layer stack) */
enum rc_activation { RC_ACT_NONE = 0, RC_ACT_RELU = 1 };

typedef struct rc_desc {
  int n;            /* images in the batch (>= 0) */
  int c_in, h, w;   /* Tensor3 shape per image */
  int c_out, k;     /* FilterBank Cout, square kernel size K */
  int group;        /* rc_group */
  int orientations; /* R: 1 single, 4 p4, 8 p4m, N (N%4==0) steer */
  int pool;         /* rc_pool */
  int pool_group;   /* subgroup_pool_max group_size */
  int convention;   /* rc_convention */
  int precision;    /* rc_precision */
  int activation;   /* rc_activation (ABI 2) */
} rc_desc;

/* ---- introspection ------------------------------------------------------ */
int rc_abi_version(void);
/* Main-kernel timing for benchmarks/profilers: while enabled on the calling thread, every
 * conv launch brackets its main kernel (not operand packing) with a CUDA event pair on its
 * stream; rc_profile_collect synchronises and returns the durations (ms) in launch order.
 * Enabling again clears the list. */
int rc_profile_enable(int on);
int rc_profile_collect(float* ms, int max_n);
const char* rc_last_error(void);
/* RC_OK or RC_ERR_INVALID (message via rc_last_error) */
int rc_validate(const rc_desc* d);
int rc_num_bases(const rc_desc* d);          /* B */
int rc_out_orientations(const rc_desc* d);   /* R' */
/* MultCounter semantics (scatter_conv.hpp:28-41, 361-366):
 * mults = N*H*W*K*K*Cin*Cout per base kernel (R-independent), adds =
 * clipped_writes*Cout per base. */
int rc_analytic_counts(const rc_desc* d, unsigned long long* mults, unsigned long long* adds);
/* scatter_conv.hpp:94-110 */
unsigned long long rc_clipped_writes(int h, int w, int kh, int kw);
/* contiguous batch shard of rank r out of world */
int rc_shard_range(int n, int world, int rank, int* begin, int* end);

/* ---- rotated-filter-bank precompute (tensor.hpp:348-370) ---
 * Replaces steer / build_orientation_bank / transform_kernel (SPEC-only) and
 * reverse_bank (scatter_conv.hpp:81-90).  The bank is an opaque device buffer of
 * rc_bank_bytes(d) bytes; its first B*Cout*Cin*K*K floats are the base kernels
 * K_b in FilterBank layout, the rest are the kernel-specific packed operands.
 * Rotations are never materialised (index maps inside the conv kernels).
 * w0 = W (single/p4/p4m) or f_x (steer); w1 = f_y (steer) or ignored. */
size_t rc_bank_bytes(const rc_desc* d);
int rc_bank_precompute(const rc_desc* d, const float* d_w0, const float* d_w1, void* d_bank,
                       void* stream);
/* build_orientation_bank: materialise all R kernels, orbit-major,
 * [R][Cout][Cin][K][K] floats, from a precomputed bank. */
int rc_orientation_bank(const rc_desc* d, const void* d_bank, float* d_kernels, void* stream);

/* steer at an arbitrary angle: out = sin(theta)*f_x + cos(theta)*f_y
 * elementwise over `count` floats, coefficients rounded once from double, no FMA. */
int rc_steer(const float* d_fx, const float* d_fy, size_t count, double theta, float* d_out,
             void* stream);

/* ---- the fused layer forward --------------------------------------------
 * Replaces tiled_scatter_conv (scatter_conv.hpp:330-368; R = 1) and the
 * SPEC-defined group_conv_scatter_reuse + orientation_pool_{avg,max} /
 * subgroup_pool_max + bias epilogue, fused into one kernel.
 * d_bias may be NULL (the reference has no bias); d_argmax may be NULL and is
 * only written for max / subgroup pooling. */
size_t rc_workspace_size(const rc_desc* d);
int rc_ri_conv_forward(const rc_desc* d, const float* d_x, const void* d_bank,
                       const float* d_bias, float* d_y, uint8_t* d_argmax, void* d_ws,
                       size_t ws_bytes, void* stream);
/* which kernel rc_ri_conv_forward runs for d (e.g. "simt_k3<8,2,4>",
 * "tc_bf16x3", "generic"); NULL if none */
const char* rc_kernel_name(const rc_desc* d);

/* ---- backward (SPEC backward module) -----------------------------
 * Gradients of the fused layer for an upstream gradient d_gy (N, Cout, R', H, W):
 *   ReLU backward (needs the forward output d_y; d_gy is MASKED IN PLACE), bias gradient
 *   (d_dbias, Cout), pool backward through the forward's argmax map (Eq. 11/12) into
 *   d_scratch (rc_backward_scratch_bytes: the unpooled (N, Cout, R, H, W) gradient),
 *   input gradient d_dx (N, Cin, H, W) as one single-orientation transposed conv on this
 *   library's kernels (Eq. 13/15), and parameter gradients (Eq. 14 via im2col + FP32
 *   cuBLAS SGEMM, Eq. 16 inverse-rotation sum, then the group's chain rule): d_dw0 = dW
 *   (single/p4/p4m) or d f_x (steer), d_dw1 = d f_y (steer).  Any output may be NULL. */
size_t rc_backward_scratch_bytes(const rc_desc* d);
size_t rc_backward_workspace_size(const rc_desc* d);
int rc_ri_conv_backward(const rc_desc* d, const float* d_x, const void* d_bank, const float* d_y,
                        float* d_gy, const uint8_t* d_argmax, float* d_dx, float* d_dw0, float* d_dw1,
                        float* d_dbias, float* d_scratch, void* d_ws, size_t ws_bytes, void* stream);

/* Orientation pooling of an already materialised OrientedFeature batch
 * (N, Cout, R, H, W) -- SPEC:283-309 as standalone ops. */
int rc_orientation_pool(int n, int c_out, int r, int h, int w, int pool, int pool_group,
                        const float* d_f, const float* d_bias, float* d_y, uint8_t* d_argmax,
                        void* stream);

/* ---- multi-layer stack glue (config C5; not in the reference) -----
 * 2x2 max pooling of an NCHW batch (H even, W a multiple of 4) and the classifier head:
 * global average pooling over H*W followed by logits = feat @ Wc^T + bc
 * (Wc: classes x C row-major, bc nullable). */
int rc_maxpool2x2(int n, int c, int h, int w, const float* d_x, float* d_y, void* stream);
int rc_gap_linear(int n, int c, int h, int w, const float* d_x, const float* d_wc, const float* d_bc,
                  int classes, float* d_out, void* stream);

/* ---- host-buffer drop-in entry points ------------------------------------
 * The whole layer with host (ideally pinned) buffers on device `device`:
 * H2D of x and the weights, bank precompute, fused forward, D2H of y/argmax. */
int rc_ri_conv_forward_host(const rc_desc* d, const float* h_x, const float* h_w0,
                            const float* h_w1, const float* h_bias, float* h_y,
                            uint8_t* h_argmax, int device);
/* steer with host buffers. */
int rc_steer_host(const float* h_fx, const float* h_fy, size_t count, double theta, float* h_out,
                  int device);
/* build_orientation_bank / transform_kernel with host buffers:
 * h_kernels receives R*Cout*Cin*K*K floats, orbit-major (o = b*4 + r). */
int rc_orientation_bank_host(const rc_desc* d, const float* h_w0, const float* h_w1,
                             float* h_kernels, int device);
/* orientation_pool_avg / orientation_pool_max / subgroup_pool_max on a
 * host OrientedFeature batch (N, Cout, R, H, W). */
int rc_orientation_pool_host(int n, int c_out, int r, int h, int w, int pool, int pool_group,
                             const float* h_f, const float* h_bias, float* h_y,
                             uint8_t* h_argmax, int device);
/* Batch-sharded multi-GPU layer forward (no reference counterpart: the reference loops
 * over images on one host).  Images are split into contiguous shards
 * (rc_shard_range) over `n_devices` GPUs (`devices` = NULL means 0..n_devices-1), one
 * host thread per GPU; each GPU builds the same bank and writes its shard straight into
 * its slice of h_y / h_argmax.  No collective is involved. */
int rc_mgpu_forward_host(const rc_desc* d, const float* h_x, const float* h_w0,
                         const float* h_w1, const float* h_bias, float* h_y, uint8_t* h_argmax,
                         int n_devices, const int* devices);
/* tiled_scatter_conv drop-in (scatter_conv.hpp:330-368) for float: validates
 * exactly like the reference (channel mismatch, square kernel, tile dims,
 * halo == K/2, workers >= 1) and returns the identical-semantics output for one
 * image.  tile/workers/strategy do not change the result (the reference is
 * bit-identical across them, scatter_conv.hpp:21-23).  mults/adds/aux_bytes
 * (nullable) receive the MultCounter / AuxMemCounter increments with the reference's
 * semantics: aux_bytes = tile_h*tile_w*sizeof(float)*workers for tile_private, 0 for
 * phase_parallel (scatter_conv.hpp:351-360).  `precision` (rc_precision, ABI 3) selects
 * the arithmetic; RC_PREC_AUTO (0) is the default of every drop-in. */
int rc_tiled_scatter_conv_host(const float* h_x, int c_in, int h, int w, const float* h_wt,
                               int c_out, int in_channels_w, int kh, int kw, int tile_h,
                               int tile_w, int halo, int workers, int strategy, float* h_y,
                               unsigned long long* mults, unsigned long long* adds,
                               unsigned long long* aux_bytes, int precision, int device);

#ifdef __cplusplus
}
#endif
#endif /* ROTCONV_C_H */
