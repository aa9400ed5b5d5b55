/*
 * rc_oracle.c -- CPU restatement of the reference's RI scatter-conv path.
 * TEST INFRASTRUCTURE ONLY (see rc_oracle.h).  Build: oracle/Makefile.
 */
#define _GNU_SOURCE
#include "rc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* SPEC:250-253 GroupSpec sizes; SPEC:433-436 steerable N/4 first-quadrant bases */
int rco_num_bases(const rco_desc* d) {
  switch (d->group) {
    case RCO_GROUP_P4M: return 2;
    case RCO_GROUP_STEER: return d->orientations / 4;
    default: return 1;
  }
}

int rco_rot_per_base(const rco_desc* d) { return d->group == RCO_GROUP_SINGLE ? 1 : 4; }

int rco_out_orientations(const rco_desc* d) {
  const int R = rco_num_bases(d) * rco_rot_per_base(d);
  switch (d->pool) {
    case RCO_POOL_NONE: return R;
    case RCO_POOL_SUBGROUP: return d->pool_group > 0 ? R / d->pool_group : 0;
    default: return 1;
  }
}

static int fail(char* msg, size_t n, const char* s) {
  if (msg && n) snprintf(msg, n, "%s", s);
  return -1;
}

int rco_validate(const rco_desc* d, char* msg, size_t n) {
  if (d->n < 0) return fail(msg, n, "ri_conv: batch must be >= 0");
  if (d->c_in < 1 || d->h < 1 || d->w < 1) return fail(msg, n, "Tensor3: dimensions must be positive");
  if (d->c_out < 1) return fail(msg, n, "FilterBank: channel counts must be positive");
  if (d->k < 1) return fail(msg, n, "FilterBank: kernel dims must be >= 1");
  switch (d->group) {
    case RCO_GROUP_SINGLE:
      if (d->orientations != 1) return fail(msg, n, "ri_conv: single group needs 1 orientation");
      break;
    case RCO_GROUP_P4:
      if (d->orientations != 4) return fail(msg, n, "GroupSpec: size must be 4 for p4");
      break;
    case RCO_GROUP_P4M:
      if (d->orientations != 8) return fail(msg, n, "GroupSpec: size must be 8 for p4m");
      break;
    case RCO_GROUP_STEER:
      if (d->orientations < 4 || d->orientations % 4 != 0)
        return fail(msg, n, "build_orientation_bank: N must be a multiple of 4");
      break;
    default: return fail(msg, n, "ri_conv: unknown group");
  }
  if (d->group != RCO_GROUP_SINGLE && d->k % 2 == 0)
    return fail(msg, n, "transform_kernel: rotation groups need odd square kernels");
  if (d->orientations > 256) return fail(msg, n, "ri_conv: at most 256 orientations");
  switch (d->pool) {
    case RCO_POOL_NONE: case RCO_POOL_AVG: case RCO_POOL_MAX: break;
    case RCO_POOL_SUBGROUP:
      if (d->pool_group < 1 || d->orientations % d->pool_group != 0)
        return fail(msg, n, "subgroup_pool_max: R not divisible by group_size");
      break;
    default: return fail(msg, n, "ri_conv: unknown pool");
  }
  if (d->convention != RCO_CONV_SCATTER && d->convention != RCO_CONV_RAW)
    return fail(msg, n, "ri_conv: unknown convention");
  return 0;
}

/* scatter_conv.hpp:94-110 */
unsigned long long rco_clipped_writes(int h, int w, int kh, int kw) {
  const int ch = kh / 2, cw = kw / 2;
  unsigned long long total = 0;
  for (int m = 0; m < kh; ++m) {
    const int dm = m - ch;
    const int rows = dm < 0 ? h + dm : h - dm;
    if (rows <= 0) continue;
    for (int nn = 0; nn < kw; ++nn) {
      const int dn = nn - cw;
      const int cols = dn < 0 ? w + dn : w - dn;
      if (cols > 0) total += (unsigned long long)rows * cols;
    }
  }
  return total;
}

/* The slice kernel G_{b,r} as a plane of base-tap ids: rot90^r (tensor.hpp:348-360)
 * of the id plane, then (scatter convention) reverse_plane (scatter_conv.hpp:72-79),
 * because scatter_conv_multi(X, V) == conv_gather_same(X, reverse(V))
 * (scatter_conv.hpp:17-19, 189-193). */
void rco_slice_tap_map(int k, int r, int convention, int* map) {
  const int kk = k * k;
  int* cur = (int*)malloc(sizeof(int) * kk);
  int* nxt = (int*)malloc(sizeof(int) * kk);
  for (int t = 0; t < kk; ++t) cur[t] = t;
  const int q = ((r % 4) + 4) % 4;
  for (int s = 0; s < q; ++s) {
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) nxt[i * k + j] = cur[j * k + (k - 1 - i)];
    int* tmp = cur; cur = nxt; nxt = tmp;
  }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j)
      map[i * k + j] = convention == RCO_CONV_SCATTER ? cur[(k - 1 - i) * k + (k - 1 - j)]
                                                       : cur[i * k + j];
  free(cur);
  free(nxt);
}

#define T float
#define S f
#include "rc_oracle_impl.h"
#undef T
#undef S

#define T double
#define S d
#include "rc_oracle_impl.h"
#undef T
#undef S
