/*
 * rc_oracle_impl.h -- type-generic body of the CPU oracle (TEST INFRASTRUCTURE).
 * Included twice by rc_oracle.c with T = float (S = f) and T = double (S = d),
 * mirroring the reference's templating on the scalar (tensor.hpp:16-17).
 */
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name##_, S)

/* tensor.hpp:348-360 rot90_plane: counterclockwise quarter turns, q mod 4;
 * one turn maps rows x cols to cols x rows with out[i][j] = in[j][cols-1-i]. */
void FN(rco_rot90_plane)(const T* in, int rows, int cols, int q, T* out, int* out_rows,
                         int* out_cols) {
  q = ((q % 4) + 4) % 4;
  int cr = rows, cc = cols;
  T* cur = (T*)malloc(sizeof(T) * (size_t)rows * cols);
  T* nxt = (T*)malloc(sizeof(T) * (size_t)rows * cols);
  memcpy(cur, in, sizeof(T) * (size_t)rows * cols);
  for (int t = 0; t < q; ++t) {
    const int nr = cc, nc = cr;
    for (int i = 0; i < nr; ++i)
      for (int j = 0; j < nc; ++j) nxt[(size_t)i * nc + j] = cur[(size_t)j * cc + (cc - 1 - i)];
    T* tmp = cur; cur = nxt; nxt = tmp;
    cr = nr; cc = nc;
  }
  memcpy(out, cur, sizeof(T) * (size_t)rows * cols);
  if (out_rows) *out_rows = cr;
  if (out_cols) *out_cols = cc;
  free(cur); free(nxt);
}

/* tensor.hpp:363-370 mirror_plane: out[i][j] = in[i][cols-1-j] */
void FN(rco_mirror_plane)(const T* in, int rows, int cols, T* out) {
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out[(size_t)i * cols + j] = in[(size_t)i * cols + (cols - 1 - j)];
}

/* scatter_conv.hpp:72-79 reverse_plane: both axes reversed */
void FN(rco_reverse_plane)(const T* in, int rows, int cols, T* out) {
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j)
      out[(size_t)i * cols + j] = in[(size_t)(rows - 1 - i) * cols + (cols - 1 - j)];
}

/* SPEC:256-264 transform_kernel: per (co, ci) plane, optional mirror (p4m element
 * (r, mirror) = mirror first), then r counterclockwise quarter turns. */
void FN(rco_transform_kernel)(const T* w, int cout, int cin, int k, int r, int mirror,
                              T* out) {
  T* tmp = (T*)malloc(sizeof(T) * (size_t)k * k);
  for (size_t p = 0; p < (size_t)cout * cin; ++p) {
    const T* src = w + p * k * k;
    if (mirror) {
      FN(rco_mirror_plane)(src, k, k, tmp);
      src = tmp;
    }
    FN(rco_rot90_plane)(src, k, k, r, out + p * k * k, NULL, NULL);
  }
  free(tmp);
}

/* SPEC:439-447 steer: sin(theta) * f_x + cos(theta) * f_y, elementwise.  The
 * coefficients are evaluated in double and rounded once to T; the product and the
 * sum are each rounded to T (no fused multiply-add). */
void FN(rco_steer)(const T* fx, const T* fy, size_t count, double theta, T* out) {
  const T s = (T)sin(theta), c = (T)cos(theta);
  for (size_t i = 0; i < count; ++i) {
    const T a = s * fx[i];
    const T b = c * fy[i];
    out[i] = a + b;
  }
}

/* Base kernels K_b (pinned convention P2):
 *   single/p4 : K_0 = W
 *   p4m       : K_0 = W, K_1 = mirror(W)
 *   steer N   : K_b = steer(f_x, f_y, 2*pi*b/N), b<N/4
 * bases layout: [B][Cout][Cin][K][K]. */
void FN(rco_build_bases)(const rco_desc* d, const T* w0, const T* w1, T* bases) {
  const size_t per = (size_t)d->c_out * d->c_in * d->k * d->k;
  const int nb = rco_num_bases(d);
  if (d->group == RCO_GROUP_STEER) {
    for (int b = 0; b < nb; ++b) {
      const double theta = 2.0 * M_PI * (double)b / (double)d->orientations;
      FN(rco_steer)(w0, w1, per, theta, bases + (size_t)b * per);
    }
  } else if (d->group == RCO_GROUP_P4M) {
    memcpy(bases, w0, sizeof(T) * per);
    FN(rco_transform_kernel)(w0, d->c_out, d->c_in, d->k, 0, 1, bases + per);
  } else {
    memcpy(bases, w0, sizeof(T) * per);
  }
}

/* SPEC:448-456 build_orientation_bank: the full list of R kernels in orbit-major
 * order o = b*4 + r: kernel(b, r) = rot90^r(K_b), never re-steered.  For R = 1 the
 * bank is W itself.  bank layout [R][Cout][Cin][K][K]. */
void FN(rco_build_orientation_bank)(const rco_desc* d, const T* w0, const T* w1, T* bank) {
  const size_t per = (size_t)d->c_out * d->c_in * d->k * d->k;
  const int nb = rco_num_bases(d), rpb = rco_rot_per_base(d);
  T* bases = (T*)malloc(sizeof(T) * per * nb);
  FN(rco_build_bases)(d, w0, w1, bases);
  for (int b = 0; b < nb; ++b)
    for (int r = 0; r < rpb; ++r)
      FN(rco_transform_kernel)(bases + (size_t)b * per, d->c_out, d->c_in, d->k, r, 0,
                               bank + (size_t)(b * rpb + r) * per);
  free(bases);
}

/* scatter_conv.hpp:114-141 scatter_conv_raw_single */
void FN(rco_scatter_conv_raw_single)(const T* x, int h, int ww, const T* k, int kh, int kw,
                                     T* y, unsigned long long* mults,
                                     unsigned long long* adds) {
  const int ch = kh / 2, cw = kw / 2;
  memset(y, 0, sizeof(T) * (size_t)h * ww);
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < ww; ++j) {
      const T xv = x[(size_t)i * ww + j];
      for (int m = 0; m < kh; ++m) {
        const int tx = i - m + ch;
        if (tx < 0 || tx >= h) continue;
        for (int n = 0; n < kw; ++n) {
          const int ty = j - n + cw;
          if (ty < 0 || ty >= ww) continue;
          const T p = xv * k[(size_t)m * kw + n];
          y[(size_t)tx * ww + ty] += p;
        }
      }
    }
  if (mults) *mults += (unsigned long long)h * ww * kh * kw;
  if (adds) *adds += rco_clipped_writes(h, ww, kh, kw);
}

/* scatter_conv.hpp:143-149 scatter_conv_single: pre-reversed kernel */
void FN(rco_scatter_conv_single)(const T* x, int h, int w, const T* k, int kh, int kw, T* y,
                                 unsigned long long* mults, unsigned long long* adds) {
  T* rev = (T*)malloc(sizeof(T) * (size_t)kh * kw);
  FN(rco_reverse_plane)(k, kh, kw, rev);
  FN(rco_scatter_conv_raw_single)(x, h, w, rev, kh, kw, y, mults, adds);
  free(rev);
}

/* scatter_conv.hpp:151-187 scatter_conv_raw_multi: per input pixel (i, j) the
 * channel dot sum_ci X[ci,i,j]*W[co,ci,m,n] is formed once per (co, m, n) (ascending
 * ci) and added to Y[co, i-m+ch, j-n+cw] when in range.  Input pixels are visited in
 * ascending order, so every output accumulates in ascending input order. */
void FN(rco_scatter_conv_raw_multi)(const T* x, int cin, int h, int ww, const T* wt, int cout,
                                    int kh, int kw, T* y) {
  const int ch = kh / 2, cw = kw / 2, plane = h * ww, kk = kh * kw;
  T* xcol = (T*)malloc(sizeof(T) * (size_t)cin);
  /* weights transposed to [co][m][n][ci] so the dot reads contiguously; the
   * summation order over ci (ascending) is the reference's, bits are identical. */
  T* wtr = (T*)malloc(sizeof(T) * (size_t)cout * kk * cin);
  for (int co = 0; co < cout; ++co)
    for (int ci = 0; ci < cin; ++ci)
      for (int t = 0; t < kk; ++t)
        wtr[((size_t)co * kk + t) * cin + ci] = wt[((size_t)co * cin + ci) * kk + t];
  memset(y, 0, sizeof(T) * (size_t)cout * plane);
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < ww; ++j) {
      for (int ci = 0; ci < cin; ++ci) xcol[ci] = x[(size_t)ci * plane + i * ww + j];
      for (int co = 0; co < cout; ++co) {
        T* yp = y + (size_t)co * plane;
        for (int m = 0; m < kh; ++m) {
          const int tx = i - m + ch;
          for (int n = 0; n < kw; ++n) {
            const int ty = j - n + cw;
            if (tx < 0 || tx >= h || ty < 0 || ty >= ww) continue; /* dot would be dropped */
            const T* wr = wtr + ((size_t)co * kk + m * kw + n) * cin;
            T dot = 0;
            for (int ci = 0; ci < cin; ++ci) dot += xcol[ci] * wr[ci];
            yp[tx * ww + ty] += dot;
          }
        }
      }
    }
  free(xcol);
  free(wtr);
}

/* scatter_conv.hpp:189-193 scatter_conv_multi = raw_multi(x, reverse_bank(w)) */
void FN(rco_scatter_conv_multi)(const T* x, int cin, int h, int w, const T* wt, int cout, int kh,
                                int kw, T* y) {
  const size_t kk = (size_t)kh * kw;
  T* rev = (T*)malloc(sizeof(T) * (size_t)cout * cin * kk);
  for (size_t p = 0; p < (size_t)cout * cin; ++p)
    FN(rco_reverse_plane)(wt + p * kk, kh, kw, rev + p * kk);
  FN(rco_scatter_conv_raw_multi)(x, cin, h, w, rev, cout, kh, kw, y);
  free(rev);
}

/* reference_conv.hpp:38-67 conv_gather_same (zero pad, centre floor(K/2)) */
void FN(rco_conv_gather_same)(const T* x, int cin, int hh, int ww, const T* wt, int cout,
                              int kh, int kw, T* y) {
  const int ch = kh / 2, cw = kw / 2;
  for (int co = 0; co < cout; ++co)
    for (int p = 0; p < hh; ++p)
      for (int q = 0; q < ww; ++q) {
        T acc = 0;
        for (int ci = 0; ci < cin; ++ci) {
          const T* plane = wt + ((size_t)co * cin + ci) * kh * kw;
          for (int i = 0; i < kh; ++i) {
            const int sh = p + i - ch;
            if (sh < 0 || sh >= hh) continue;
            for (int j = 0; j < kw; ++j) {
              const int sw = q + j - cw;
              if (sw < 0 || sw >= ww) continue;
              acc += plane[i * kw + j] * x[((size_t)ci * hh + sh) * ww + sw];
            }
          }
        }
        y[((size_t)co * hh + p) * ww + q] = acc;
      }
}

/* SPEC:274-282 group_conv_scatter_reuse: for each input pixel, the dot of every
 * base tap (b, t) is computed ONCE and scattered to the rot_per_base destinations
 * of its orbit via the precomputed index maps.  Slice o = b*rpb + r
 * equals scatter_conv_multi(X, rot90^r(K_b)) bit-for-bit (scatter convention): each
 * output still receives its contributions in ascending input order.
 * f layout: (Cout, R, H, W) = OrientedFeature (tensor.hpp:191-276). */
void FN(rco_group_conv_scatter_reuse)(const rco_desc* d, const T* x, const T* bases, T* f) {
  const int cin = d->c_in, h = d->h, ww = d->w, k = d->k, kk = k * k, cout = d->c_out;
  const int nb = rco_num_bases(d), rpb = rco_rot_per_base(d), R = nb * rpb;
  const int c = k / 2, plane = h * ww;
  /* offsets: slice (r) reads base tap t at gather offset (di, dj): the input
   * pixel q feeds output q - (di, dj). */
  int* dI = (int*)malloc(sizeof(int) * rpb * kk);
  int* dJ = (int*)malloc(sizeof(int) * rpb * kk);
  int* map = (int*)malloc(sizeof(int) * kk);
  for (int r = 0; r < rpb; ++r) {
    rco_slice_tap_map(k, r, d->convention, map);
    for (int pos = 0; pos < kk; ++pos) {
      const int t = map[pos];
      dI[r * kk + t] = pos / k - c;
      dJ[r * kk + t] = pos % k - c;
    }
  }
  T* wtr = (T*)malloc(sizeof(T) * (size_t)nb * cout * kk * cin);
  for (int b = 0; b < nb; ++b)
    for (int co = 0; co < cout; ++co)
      for (int ci = 0; ci < cin; ++ci)
        for (int t = 0; t < kk; ++t)
          wtr[(((size_t)b * cout + co) * kk + t) * cin + ci] =
              bases[(((size_t)b * cout + co) * cin + ci) * kk + t];
  T* xcol = (T*)malloc(sizeof(T) * (size_t)cin);
  memset(f, 0, sizeof(T) * (size_t)cout * R * plane);
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < ww; ++j) {
      for (int ci = 0; ci < cin; ++ci) xcol[ci] = x[(size_t)ci * plane + i * ww + j];
      for (int co = 0; co < cout; ++co)
        for (int b = 0; b < nb; ++b)
          for (int t = 0; t < kk; ++t) {
            const T* wr = wtr + (((size_t)b * cout + co) * kk + t) * cin;
            T dot = 0;
            for (int ci = 0; ci < cin; ++ci) dot += xcol[ci] * wr[ci];
            for (int r = 0; r < rpb; ++r) {
              const int ti = i - dI[r * kk + t], tj = j - dJ[r * kk + t];
              if (ti < 0 || ti >= h || tj < 0 || tj >= ww) continue;
              f[(((size_t)co * R + b * rpb + r) * h + ti) * ww + tj] += dot;
            }
          }
    }
  free(dI); free(dJ); free(map); free(wtr); free(xcol);
}

/* SPEC:283-291, Eq. (9): mean over orientations, summed in ascending r then
 * divided by R. */
void FN(rco_orientation_pool_avg)(const T* f, int cout, int r, int h, int w, T* y) {
  const size_t plane = (size_t)h * w;
  for (int co = 0; co < cout; ++co)
    for (size_t p = 0; p < plane; ++p) {
      T acc = 0;
      for (int o = 0; o < r; ++o) acc += f[((size_t)co * r + o) * plane + p];
      y[(size_t)co * plane + p] = acc / (T)r;
    }
}

/* SPEC:292-300, Eq. (10): max over orientations + argmax, ties -> smallest r. */
void FN(rco_orientation_pool_max)(const T* f, int cout, int r, int h, int w, T* y,
                                  uint8_t* argmax) {
  FN(rco_subgroup_pool_max)(f, cout, r, h, w, r, y, argmax);
}

/* SPEC:301-309 subgroup_pool_max: max over each contiguous block of g slices,
 * block-local argmax in [0, g), ties -> smallest index.  Output (Cout, R/g, H, W). */
void FN(rco_subgroup_pool_max)(const T* f, int cout, int r, int h, int w, int g, T* y,
                               uint8_t* argmax) {
  const size_t plane = (size_t)h * w;
  const int ro = r / g;
  for (int co = 0; co < cout; ++co)
    for (int blk = 0; blk < ro; ++blk)
      for (size_t p = 0; p < plane; ++p) {
        T best = f[((size_t)co * r + blk * g) * plane + p];
        int arg = 0;
        for (int o = 1; o < g; ++o) {
          const T v = f[((size_t)co * r + blk * g + o) * plane + p];
          if (v > best) { best = v; arg = o; }
        }
        y[((size_t)co * ro + blk) * plane + p] = best;
        if (argmax) argmax[((size_t)co * ro + blk) * plane + p] = (uint8_t)arg;
      }
}

typedef struct {
  const rco_desc* d;
  const T *x, *bases, *bias;
  T* y;
  uint8_t* argmax;
  int first, step, end;
} FN(rco_job);

static void* FN(rco_worker)(void* arg) {
  FN(rco_job)* job = (FN(rco_job)*)arg;
  const rco_desc* d = job->d;
  const int nb = rco_num_bases(d), rpb = rco_rot_per_base(d), R = nb * rpb;
  const int ro = rco_out_orientations(d);
  const size_t plane = (size_t)d->h * d->w;
  const size_t xin = (size_t)d->c_in * plane;
  const size_t yout = (size_t)d->c_out * ro * plane;
  T* f = (T*)malloc(sizeof(T) * (size_t)d->c_out * R * plane);
  for (int img = job->first; img < job->end; img += job->step) {
    FN(rco_group_conv_scatter_reuse)(d, job->x + (size_t)img * xin, job->bases, f);
    T* yi = job->y + (size_t)img * yout;
    uint8_t* ai = job->argmax ? job->argmax + (size_t)img * yout : NULL;
    switch (d->pool) {
      case RCO_POOL_NONE: memcpy(yi, f, sizeof(T) * yout); break;
      case RCO_POOL_AVG: FN(rco_orientation_pool_avg)(f, d->c_out, R, d->h, d->w, yi); break;
      case RCO_POOL_MAX: FN(rco_orientation_pool_max)(f, d->c_out, R, d->h, d->w, yi, ai); break;
      default: FN(rco_subgroup_pool_max)(f, d->c_out, R, d->h, d->w, d->pool_group, yi, ai); break;
    }
    /* bias epilogue after the reduction (pinned convention P5, not in reference) */
    if (job->bias)
      for (int co = 0; co < d->c_out; ++co)
        for (size_t p = 0; p < (size_t)ro * plane; ++p) yi[(size_t)co * ro * plane + p] += job->bias[co];
  }
  free(f);
  return NULL;
}

/* Full RI layer forward over images [image_begin, image_end) of the batch:
 * base bank -> reuse scatter -> pooling
 * -> bias.  x, y, argmax address the whole batch.  Images are
 * distributed round-robin over nthreads std-thread-like workers (the reference
 * runs one image per call; scatter_conv.hpp:247-255 for the threading). */
int FN(rco_ri_forward)(const rco_desc* d, const T* x, const T* w0, const T* w1, const T* bias,
                       T* y, uint8_t* argmax, int nthreads, int image_begin, int image_end) {
  char msg[256];
  if (rco_validate(d, msg, sizeof msg) != 0) return -1;
  if (image_begin < 0) image_begin = 0;
  if (image_end < 0 || image_end > d->n) image_end = d->n;
  if (nthreads < 1) nthreads = 1;
  const size_t per = (size_t)d->c_out * d->c_in * d->k * d->k;
  T* bases = (T*)malloc(sizeof(T) * per * rco_num_bases(d));
  FN(rco_build_bases)(d, w0, w1, bases);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  FN(rco_job)* jobs = (FN(rco_job)*)malloc(sizeof(FN(rco_job)) * nthreads);
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].d = d; jobs[t].x = x; jobs[t].bases = bases; jobs[t].bias = bias;
    jobs[t].y = y; jobs[t].argmax = argmax;
    jobs[t].first = image_begin + t; jobs[t].step = nthreads; jobs[t].end = image_end;
    if (nthreads == 1) FN(rco_worker)(&jobs[t]);
    else pthread_create(&th[t], NULL, FN(rco_worker), &jobs[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th); free(jobs); free(bases);
  return 0;
}

#undef FN
#undef CAT
#undef CAT2
