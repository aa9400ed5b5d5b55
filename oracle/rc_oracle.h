/*
 * rc_oracle.h -- CPU restatement of the reference's rotation-invariant scatter
 * convolution path (arXiv 2512.08888, /root/reference).
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the *checker*: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  The product path (paper_2512_08888_b200 + librotconv_b200.so) never
 * links or calls it.
 *
 * Every function cites the reference file:line it restates.  Abbreviations:
 *   tensor.hpp         = proj/include/rotconv/tensor.hpp
 *   scatter_conv.hpp   = proj/include/rotconv/scatter_conv.hpp
 *   reference_conv.hpp = proj/include/rotconv/reference_conv.hpp
 *   SPEC               = SPEC.md (group_conv / steerable modules have no shipped code)
 *
 * Parity is pinned two ways:
 *   1. bit-exact against the unmodified reference headers compiled into
 *      oracle/_ref/librc_ref.so (oracle/Makefile, oracle/ref_shim.cpp);
 *   2. the SPEC known-answer examples (tests/test_oracle_kat.py).
 *
 * All tensors are dense row-major, exactly as the reference containers store them:
 *   Tensor3         (C, H, W)            tensor.hpp:30-101
 *   FilterBank      (Cout, Cin, K, K)     tensor.hpp:104-188
 *   OrientedFeature (Cout, R, H, W)       tensor.hpp:191-276
 * A batch is N contiguous per-image tensors (the reference loops over images,
 * SPEC:239).  Compile with -ffp-contract=off so products and sums round exactly
 * like the reference's `dot += x * w` loops.
 */
#ifndef RC_ORACLE_H
#define RC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* group kinds / pool kinds / slice conventions (mirror include/rotconv_c.h) */
enum { RCO_GROUP_SINGLE = 0, RCO_GROUP_P4 = 1, RCO_GROUP_P4M = 2, RCO_GROUP_STEER = 3 };
enum { RCO_POOL_NONE = 0, RCO_POOL_AVG = 1, RCO_POOL_MAX = 2, RCO_POOL_SUBGROUP = 3 };
enum { RCO_CONV_SCATTER = 0, RCO_CONV_RAW = 1 };

typedef struct rco_desc {
  int n, c_in, h, w, c_out, k;
  int group;       /* RCO_GROUP_* */
  int orientations;/* R: 1 single, 4 p4, 8 p4m, N%4==0 steer */
  int pool;        /* RCO_POOL_* */
  int pool_group;  /* group_size for subgroup pooling */
  int convention;  /* RCO_CONV_* */
} rco_desc;

/* number of base kernels B and orientations per base */
int rco_num_bases(const rco_desc* d);
int rco_rot_per_base(const rco_desc* d);
/* pooled orientation count R' (1 for avg/max, R/g subgroup, R none) */
int rco_out_orientations(const rco_desc* d);
/* 0 ok, otherwise negative; fills msg with the reference-style message */
int rco_validate(const rco_desc* d, char* msg, size_t msg_len);

/* scatter_conv.hpp:94-110 */
unsigned long long rco_clipped_writes(int h, int w, int kh, int kw);

/* gather-position index map of slice (b, r): for every gather tap position
 * (i, j) of the slice kernel G_{b,r}, the base-kernel tap it reads.
 * scatter convention: G = reverse(rot90^r(K_b)) (scatter_conv.hpp:189-193 applied
 * to transform_kernel SPEC:256-264); raw convention: G = rot90^r(K_b).
 * map[i*k + j] = m*k + n. */
void rco_slice_tap_map(int k, int r, int convention, int* map);

#define RCO_DECL(T, S)                                                                 \
  void rco_rot90_plane_##S(const T* in, int rows, int cols, int q, T* out,            \
                           int* out_rows, int* out_cols);                             \
  void rco_mirror_plane_##S(const T* in, int rows, int cols, T* out);                 \
  void rco_reverse_plane_##S(const T* in, int rows, int cols, T* out);                \
  void rco_transform_kernel_##S(const T* w, int cout, int cin, int k, int r,          \
                                int mirror, T* out);                                  \
  void rco_steer_##S(const T* fx, const T* fy, size_t count, double theta, T* out);   \
  void rco_build_bases_##S(const rco_desc* d, const T* w0, const T* w1, T* bases);    \
  void rco_build_orientation_bank_##S(const rco_desc* d, const T* w0, const T* w1,    \
                                      T* bank);                                       \
  void rco_scatter_conv_raw_single_##S(const T* x, int h, int w, const T* k, int kh,  \
                                       int kw, T* y, unsigned long long* mults,       \
                                       unsigned long long* adds);                     \
  void rco_scatter_conv_single_##S(const T* x, int h, int w, const T* k, int kh,      \
                                   int kw, T* y, unsigned long long* mults,           \
                                   unsigned long long* adds);                         \
  void rco_scatter_conv_raw_multi_##S(const T* x, int cin, int h, int w, const T* wt, \
                                      int cout, int kh, int kw, T* y);                \
  void rco_scatter_conv_multi_##S(const T* x, int cin, int h, int w, const T* wt,     \
                                  int cout, int kh, int kw, T* y);                    \
  void rco_conv_gather_same_##S(const T* x, int cin, int h, int w, const T* wt,       \
                                int cout, int kh, int kw, T* y);                      \
  void rco_group_conv_scatter_reuse_##S(const rco_desc* d, const T* x, const T* bases, \
                                        T* f);                                        \
  void rco_orientation_pool_avg_##S(const T* f, int cout, int r, int h, int w, T* y); \
  void rco_orientation_pool_max_##S(const T* f, int cout, int r, int h, int w, T* y,  \
                                    uint8_t* argmax);                                 \
  void rco_subgroup_pool_max_##S(const T* f, int cout, int r, int h, int w, int g,    \
                                 T* y, uint8_t* argmax);                              \
  int rco_ri_forward_##S(const rco_desc* d, const T* x, const T* w0, const T* w1,     \
                         const T* bias, T* y, uint8_t* argmax, int nthreads,          \
                         int image_begin, int image_end);

RCO_DECL(float, f)
RCO_DECL(double, d)
#undef RCO_DECL

#ifdef __cplusplus
}
#endif
#endif /* RC_ORACLE_H */
