// capi.cu -- the extern "C" boundary (include/rotconv_c.h): validation with the
// reference's messages, bank layout, kernel dispatch, host-buffer drop-in entry points.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "rc_internal.cuh"

namespace rc {

namespace {
thread_local std::string g_err;
struct ProfState {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pairs;
  size_t used = 0;
};
thread_local ProfState g_prof;
size_t align256(size_t v) { return (v + 255) & ~size_t(255); }
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }

void prof_begin(cudaStream_t s) {
  if (!g_prof.on) return;
  if (g_prof.used == g_prof.pairs.size()) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return;
    g_prof.pairs.emplace_back(a, b);
  }
  cudaEventRecord(g_prof.pairs[g_prof.used].first, s);
}
void prof_end(cudaStream_t s) {
  if (!g_prof.on || g_prof.used == g_prof.pairs.size()) return;
  cudaEventRecord(g_prof.pairs[g_prof.used++].second, s);
}
int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}
int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + where;
  return RC_ERR_CUDA;
}

// Same preconditions (and message strings) as the reference containers and ops:
// tensor.hpp:38-39, 111-112; scatter_conv.hpp:339-346.
int validate(const rc_desc& d) {
  if (d.n < 0) return fail(RC_ERR_INVALID, "ri_conv: batch must be >= 0");
  if (d.c_in < 1 || d.h < 1 || d.w < 1)
    return fail(RC_ERR_INVALID, "Tensor3: dimensions must be positive");
  if (d.c_out < 1) return fail(RC_ERR_INVALID, "FilterBank: channel counts must be positive");
  if (d.k < 1) return fail(RC_ERR_INVALID, "FilterBank: kernel dims must be >= 1");
  // every kernel and index table (tap maps, bank steering, backward tap offsets) is sized
  // for kMaxK x kMaxK taps: refuse larger kernels before anything touches them
  if (d.k > kMaxK) return fail(RC_ERR_UNSUPPORTED, "ri_conv: kernel size > 11 unsupported");
  switch (d.group) {
    case RC_GROUP_SINGLE:
      if (d.orientations != 1) return fail(RC_ERR_INVALID, "ri_conv: single group needs 1 orientation");
      break;
    case RC_GROUP_P4:
      if (d.orientations != 4) return fail(RC_ERR_INVALID, "GroupSpec: size must be 4 for p4");
      break;
    case RC_GROUP_P4M:
      if (d.orientations != 8) return fail(RC_ERR_INVALID, "GroupSpec: size must be 8 for p4m");
      break;
    case RC_GROUP_STEER:
      if (d.orientations < 4 || d.orientations % 4 != 0)
        return fail(RC_ERR_INVALID, "build_orientation_bank: N must be a multiple of 4");
      break;
    default: return fail(RC_ERR_INVALID, "ri_conv: unknown group");
  }
  if (d.group != RC_GROUP_SINGLE && d.k % 2 == 0)
    return fail(RC_ERR_INVALID, "transform_kernel: rotation groups need odd square kernels");
  if (d.orientations > 256) return fail(RC_ERR_INVALID, "ri_conv: at most 256 orientations");
  switch (d.pool) {
    case RC_POOL_NONE: case RC_POOL_AVG: case RC_POOL_MAX: break;
    case RC_POOL_SUBGROUP:
      if (d.pool_group < 1 || d.orientations % d.pool_group != 0)
        return fail(RC_ERR_INVALID, "subgroup_pool_max: R not divisible by group_size");
      break;
    default: return fail(RC_ERR_INVALID, "ri_conv: unknown pool");
  }
  if (d.convention != RC_CONV_SCATTER && d.convention != RC_CONV_RAW)
    return fail(RC_ERR_INVALID, "ri_conv: unknown convention");
  if (d.precision < RC_PREC_AUTO || d.precision > RC_PREC_BF16)
    return fail(RC_ERR_INVALID, "ri_conv: unknown precision");
  if (d.activation != RC_ACT_NONE && d.activation != RC_ACT_RELU)
    return fail(RC_ERR_INVALID, "ri_conv: unknown activation");
  return RC_OK;
}

BankLayout bank_layout(const rc_desc& d) {
  BankLayout L{};
  const size_t per = (size_t)d.c_out * d.c_in * d.k * d.k;
  const size_t nb = (size_t)num_bases(d);
  L.bases_off = 0;
  L.bases_bytes = per * nb * sizeof(float);
  L.simt_off = align256(L.bases_off + L.bases_bytes);
  L.simt_bytes = d.k == 3 ? nb * d.c_in * d.c_out * 12 * sizeof(float) : 0;
  L.tc_off = align256(L.simt_off + L.simt_bytes);
  L.tc_bytes = tc_bank_bytes(d);
  L.total = align256(L.tc_off + L.tc_bytes);
  return L;
}

void slice_tap_offsets(int k, int convention, TapOffsets* out) {
  std::memset(out, 0, sizeof(*out));
  const int kk = k * k, c = k / 2;
  std::vector<int> cur(kk), nxt(kk);
  for (int r = 0; r < 4; ++r) {
    for (int t = 0; t < kk; ++t) cur[t] = t;
    for (int q = 0; q < r; ++q) {  // tensor.hpp:348-360, one CCW turn
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) nxt[i * k + j] = cur[j * k + (k - 1 - i)];
      cur.swap(nxt);
    }
    for (int pos = 0; pos < kk; ++pos) {
      const int i = pos / k, j = pos % k;
      // scatter convention reads reverse(rot^r K_b) (scatter_conv.hpp:72-79, 189-193)
      const int t = convention == RC_CONV_SCATTER ? cur[(k - 1 - i) * k + (k - 1 - j)] : cur[pos];
      out->di[r][t] = (int8_t)(i - c);
      out->dj[r][t] = (int8_t)(j - c);
    }
  }
}

}  // namespace rc

using namespace rc;

namespace {

#define RC_CHECK_DESC(d)                                          \
  do {                                                            \
    if ((d) == nullptr) return fail(RC_ERR_INVALID, "null desc"); \
    int st_ = validate(*(d));                                     \
    if (st_ != RC_OK) return st_;                                 \
  } while (0)

// per-device cache of staging buffers for the host drop-in entry points
struct DeviceCache {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy engines of the chunked host pipeline
  std::vector<cudaEvent_t> ev;                 // pipeline events (grow-only)
  int ensure_pipeline(size_t events) {
    if (!h2d) RC_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    if (!d2h) RC_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    while (ev.size() < events) {
      cudaEvent_t e;
      RC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    return RC_OK;
  }
  std::vector<std::pair<void*, size_t>> bufs;  // grow-only slots
  void* get(int slot, size_t bytes) {
    if ((int)bufs.size() <= slot) bufs.resize(slot + 1, {nullptr, 0});
    auto& b = bufs[slot];
    if (b.second < bytes) {
      if (b.first) cudaFree(b.first);
      b.first = nullptr;
      b.second = 0;
      if (cudaMalloc(&b.first, bytes < 256 ? 256 : bytes) != cudaSuccess) return nullptr;
      b.second = bytes;
    }
    return b.first;
  }
};
DeviceCache g_cache[64];

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// precision FP32 -> CUDA-core kernels; BF16 / BF16X3 -> tcgen05 kernel or UNSUPPORTED
// (never silently a different arithmetic); AUTO -> tensor cores where supported.
int dispatch(const rc_desc& d, const float* x, const void* bank, const float* bias, float* y,
             uint8_t* am, void* ws, size_t ws_bytes, cudaStream_t s, bool dry, const char** name) {
  // AUTO keeps tiny channel counts on the CUDA cores: the tensor-core K chunk is 64 input
  // channels, so Cin < 16 would multiply mostly zero padding (e.g. an RGB first layer); small
  // single-orientation layers (Cin <= 8 on <= 32-wide images, Cin <= 16 on 4x4 images) run
  // the direct FP32 kernel (elsewhere at Cin = 16 the tensor-core kernels are faster,
  // profiles/r02/c2/).
  const bool small_direct = (d.c_in <= 8 || (d.c_in <= 16 && d.w == 4)) && direct_supported(d);
  const bool auto_tc = d.precision == RC_PREC_AUTO && d.c_in >= 16 && !small_direct;
  if (d.precision == RC_PREC_BF16X3 || d.precision == RC_PREC_BF16 || auto_tc) {
    int st = launch_tc(d, x, bank, bias, y, am, ws, ws_bytes, s, dry, name);
    if (st != RC_ERR_UNSUPPORTED || d.precision != RC_PREC_AUTO) {
      if (st == RC_ERR_UNSUPPORTED)
        return fail(st, "ri_conv: no tensor-core kernel for this shape (needs K=3 and W = 16, 32 or a multiple of 16 >= 48)");
      return st;
    }
  }
  // small single-orientation layers (Cin <= 16, W in {4, 8, 16, 32}): direct FP32 kernel
  int st = d.precision == RC_PREC_FP32 || small_direct ? launch_direct_k3(d, x, bank, bias, y, am, s, dry, name)
                                                       : RC_ERR_UNSUPPORTED;
  if (st != RC_ERR_UNSUPPORTED) return st;
  st = launch_simt_k3(d, x, bank, bias, y, am, s, dry, name);
  if (st != RC_ERR_UNSUPPORTED) return st;
  if (dry) {
    if (name) *name = "generic";
    return RC_OK;
  }
  st = launch_generic(d, x, bank, bias, y, am, s, name);
  if (st == RC_ERR_UNSUPPORTED) return fail(st, "ri_conv: kernel size > 11 unsupported");
  return st;
}

}  // namespace

namespace rc {
int dispatch_forward(const rc_desc& d, const float* x, const void* bank, const float* bias, float* y,
                     uint8_t* am, void* ws, size_t ws_bytes, cudaStream_t s) {
  return dispatch(d, x, bank, bias, y, am, ws, ws_bytes, s, false, nullptr);
}
}  // namespace rc

extern "C" {

int rc_abi_version(void) { return RC_ABI_VERSION; }

int rc_profile_enable(int on) {
  g_prof.on = on != 0;
  if (g_prof.on) g_prof.used = 0;
  return RC_OK;
}

int rc_profile_collect(float* ms, int max_n) {
  int n = 0;
  for (size_t i = 0; i < g_prof.used && n < max_n; ++i, ++n) {
    RC_CUDA(cudaEventSynchronize(g_prof.pairs[i].second));
    RC_CUDA(cudaEventElapsedTime(&ms[n], g_prof.pairs[i].first, g_prof.pairs[i].second));
  }
  return n;
}
const char* rc_last_error(void) { return g_err.c_str(); }

int rc_validate(const rc_desc* d) {
  RC_CHECK_DESC(d);
  return RC_OK;
}
int rc_num_bases(const rc_desc* d) { return d ? num_bases(*d) : 0; }
int rc_out_orientations(const rc_desc* d) {
  if (!d || validate(*d) != RC_OK) return 0;
  return out_orientations(*d);
}

unsigned long long rc_clipped_writes(int h, int w, int kh, int kw) {
  const int ch = kh / 2, cw = kw / 2;  // scatter_conv.hpp:94-110
  unsigned long long total = 0;
  for (int m = 0; m < kh; ++m) {
    const int dm = m - ch;
    const int rows = dm < 0 ? h + dm : h - dm;
    if (rows <= 0) continue;
    for (int n = 0; n < kw; ++n) {
      const int dn = n - cw;
      const int cols = dn < 0 ? w + dn : w - dn;
      if (cols > 0) total += (unsigned long long)rows * cols;
    }
  }
  return total;
}

int rc_analytic_counts(const rc_desc* d, unsigned long long* mults, unsigned long long* adds) {
  RC_CHECK_DESC(d);
  const unsigned long long nb = (unsigned long long)num_bases(*d);
  if (mults)
    *mults = nb * d->n * (unsigned long long)d->h * d->w * d->k * d->k * d->c_in * d->c_out;
  if (adds) *adds = nb * d->n * rc_clipped_writes(d->h, d->w, d->k, d->k) * d->c_out;
  return RC_OK;
}

int rc_shard_range(int n, int world, int rank, int* begin, int* end) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world)
    return fail(RC_ERR_INVALID, "shard_range: need n >= 0, world >= 1, 0 <= rank < world");
  const int base = n / world, rem = n % world;
  const int b = rank * base + (rank < rem ? rank : rem);
  *begin = b;
  *end = b + base + (rank < rem ? 1 : 0);
  return RC_OK;
}

size_t rc_bank_bytes(const rc_desc* d) {
  if (!d || validate(*d) != RC_OK) return 0;
  return bank_layout(*d).total;
}

int rc_bank_precompute(const rc_desc* d, const float* d_w0, const float* d_w1, void* d_bank,
                       void* stream) {
  RC_CHECK_DESC(d);
  if (!d_w0 || !d_bank || (d->group == RC_GROUP_STEER && !d_w1))
    return fail(RC_ERR_INVALID, "bank_precompute: null pointer");
  return launch_bank(*d, d_w0, d_w1, d_bank, static_cast<cudaStream_t>(stream));
}

int rc_orientation_bank(const rc_desc* d, const void* d_bank, float* d_kernels, void* stream) {
  RC_CHECK_DESC(d);
  if (!d_bank || !d_kernels) return fail(RC_ERR_INVALID, "orientation_bank: null pointer");
  return launch_orientation_bank(*d, d_bank, d_kernels, static_cast<cudaStream_t>(stream));
}

size_t rc_workspace_size(const rc_desc* d) {
  if (!d || validate(*d) != RC_OK) return 0;
  return tc_workspace_bytes(*d);
}

const char* rc_kernel_name(const rc_desc* d) {
  if (!d || validate(*d) != RC_OK) return nullptr;
  const char* name = nullptr;
  if (dispatch(*d, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, true, &name) != RC_OK)
    return nullptr;
  return name;
}

int rc_ri_conv_forward(const rc_desc* d, const float* d_x, const void* d_bank,
                       const float* d_bias, float* d_y, uint8_t* d_argmax, void* d_ws,
                       size_t ws_bytes, void* stream) {
  RC_CHECK_DESC(d);
  (void)d_ws;
  if (ws_bytes < rc_workspace_size(d)) return fail(RC_ERR_WORKSPACE, "ri_conv: workspace too small");
  if (d->n > 0 && (!d_x || !d_bank || !d_y)) return fail(RC_ERR_INVALID, "ri_conv: null pointer");
  return dispatch(*d, d_x, d_bank, d_bias, d_y, d_argmax, d_ws, ws_bytes, static_cast<cudaStream_t>(stream),
                  false, nullptr);
}

size_t rc_backward_scratch_bytes(const rc_desc* d) {
  if (!d || validate(*d) != RC_OK) return 0;
  return (size_t)d->n * d->c_out * num_bases(*d) * rot_per_base(*d) * d->h * d->w * sizeof(float);
}

size_t rc_backward_workspace_size(const rc_desc* d) {
  if (!d || validate(*d) != RC_OK) return 0;
  const size_t a = bwd_input_ws(*d), b = bwd_weight_ws(*d);
  return a > b ? a : b;
}

int rc_ri_conv_backward(const rc_desc* d, const float* d_x, const void* d_bank, const float* d_y, float* d_gy,
                        const uint8_t* d_argmax, float* d_dx, float* d_dw0, float* d_dw1, float* d_dbias,
                        float* d_scratch, void* d_ws, size_t ws_bytes, void* stream) {
  RC_CHECK_DESC(d);
  if (d->n == 0) {  // empty batch: zero parameter gradients (dx is empty)
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t wb = (size_t)d->c_out * d->c_in * d->k * d->k * sizeof(float);
    if (d_dw0) RC_CUDA(cudaMemsetAsync(d_dw0, 0, wb, s));
    if (d_dw1 && d->group == RC_GROUP_STEER) RC_CUDA(cudaMemsetAsync(d_dw1, 0, wb, s));
    if (d_dbias) RC_CUDA(cudaMemsetAsync(d_dbias, 0, (size_t)d->c_out * sizeof(float), s));
    return RC_OK;
  }
  if (!d_gy || !d_bank || !d_scratch) return fail(RC_ERR_INVALID, "ri_conv_backward: null pointer");
  if ((d->pool == RC_POOL_MAX || d->pool == RC_POOL_SUBGROUP) && !d_argmax)
    return fail(RC_ERR_INVALID, "pool_backward_max: argmax map required");
  if (d->activation == RC_ACT_RELU && !d_y) return fail(RC_ERR_INVALID, "ri_conv_backward: relu needs the forward output");
  if ((d_dw0 || (d_dw1 && d->group == RC_GROUP_STEER)) && !d_x)
    return fail(RC_ERR_INVALID, "ri_conv_backward: weight gradients need the forward input");
  if (d->group == RC_GROUP_STEER && d_dw0 && !d_dw1)
    return fail(RC_ERR_INVALID, "ri_conv_backward: steerable layers need both f_x and f_y gradients");
  if (ws_bytes < rc_backward_workspace_size(d) || !d_ws)
    return fail(RC_ERR_WORKSPACE, "ri_conv_backward: workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long ny = (long long)d->n * d->c_out * out_orientations(*d) * d->h * d->w;
  int st = RC_OK;
  if (d->activation == RC_ACT_RELU) st = launch_relu_backward(d_y, d_gy, ny, s);  // d_gy masked in place
  if (st == RC_OK && d_dbias)
    st = launch_bias_backward(d_gy, d_dbias, d->n, d->c_out, (long long)out_orientations(*d) * d->h * d->w, s);
  if (st == RC_OK) st = launch_pool_backward(*d, d_gy, d_argmax, d_scratch, s);
  if (st == RC_OK && d_dx) st = launch_bwd_input(*d, d_scratch, d_bank, d_dx, d_ws, s);
  if (st == RC_OK && d_dw0) st = launch_bwd_weight(*d, d_x, d_scratch, d_dw0, d_dw1, d_ws, s);
  return st;
}

int rc_orientation_pool(int n, int c_out, int r, int h, int w, int pool, int pool_group,
                        const float* d_f, const float* d_bias, float* d_y, uint8_t* d_argmax,
                        void* stream) {
  if (n < 0 || c_out < 1 || r < 1 || h < 1 || w < 1)
    return fail(RC_ERR_INVALID, "OrientedFeature: dimensions must be positive");
  if (pool == RC_POOL_SUBGROUP && (pool_group < 1 || r % pool_group != 0))
    return fail(RC_ERR_INVALID, "subgroup_pool_max: R not divisible by group_size");
  if (pool < RC_POOL_NONE || pool > RC_POOL_SUBGROUP) return fail(RC_ERR_INVALID, "ri_conv: unknown pool");
  return launch_pool(n, c_out, r, h, w, pool, pool_group, d_f, d_bias, d_y, d_argmax,
                     static_cast<cudaStream_t>(stream));
}

int rc_ri_conv_forward_host(const rc_desc* d, const float* h_x, const float* h_w0,
                            const float* h_w1, const float* h_bias, float* h_y,
                            uint8_t* h_argmax, int device) {
  RC_CHECK_DESC(d);
  if (device < 0 || device >= 64) return fail(RC_ERR_INVALID, "ri_conv: bad device");
  if (d->n == 0) return RC_OK;
  DeviceGuard guard(device);
  DeviceCache& c = g_cache[device];
  std::lock_guard<std::mutex> lock(c.mu);
  if (!c.stream) RC_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  const size_t xb = (size_t)d->n * d->c_in * d->h * d->w * sizeof(float);
  const size_t wb = (size_t)d->c_out * d->c_in * d->k * d->k * sizeof(float);
  const size_t ro = (size_t)out_orientations(*d);
  const size_t yb = (size_t)d->n * d->c_out * ro * d->h * d->w * sizeof(float);
  const size_t ab = yb / sizeof(float);
  const bool has_arg = h_argmax && (d->pool == RC_POOL_MAX || d->pool == RC_POOL_SUBGROUP);
  void* dx = c.get(0, xb);
  void* dw0 = c.get(1, wb);
  void* dw1 = d->group == RC_GROUP_STEER ? c.get(2, wb) : nullptr;
  void* dbias = h_bias ? c.get(3, d->c_out * sizeof(float)) : nullptr;
  void* dbank = c.get(4, bank_layout(*d).total);
  void* dy = c.get(5, yb);
  void* da = has_arg ? c.get(6, ab) : nullptr;
  const size_t wsb = tc_workspace_bytes(*d);
  void* dws = wsb ? c.get(7, wsb) : nullptr;
  if (!dx || !dw0 || !dbank || !dy || (d->group == RC_GROUP_STEER && !dw1) ||
      (h_bias && !dbias) || (has_arg && !da) || (wsb && !dws))
    return fail(RC_ERR_CUDA, "ri_conv: device allocation failed");
  cudaStream_t s = c.stream;
  RC_CUDA(cudaMemcpyAsync(dw0, h_w0, wb, cudaMemcpyHostToDevice, s));
  if (dw1) RC_CUDA(cudaMemcpyAsync(dw1, h_w1, wb, cudaMemcpyHostToDevice, s));
  if (dbias) RC_CUDA(cudaMemcpyAsync(dbias, h_bias, d->c_out * sizeof(float), cudaMemcpyHostToDevice, s));
  int st = launch_bank(*d, (const float*)dw0, (const float*)dw1, dbank, s);
  if (st != RC_OK) {
    cudaStreamSynchronize(s);  // the queued weight uploads read the caller's buffers
    return st;
  }
  // Chunked pipeline over images: H2D of chunk i+1 and D2H of chunk i-1 overlap the kernels
  // of chunk i (three streams, the copies on the two copy engines).  Chunks of >= 16 images
  // keep every copy large; small batches run as one chunk.  The output (D2H) dominates, so
  // the sooner the first chunk is computed the sooner the D2H engine starts: 16 chunks from
  // 256 images on.
  const int chunks = d->n >= 256 ? 16 : (d->n >= 64 ? 8 : (d->n >= 32 ? 4 : 1));
  st = c.ensure_pipeline(2 * (size_t)chunks);
  if (st != RC_OK) {
    cudaStreamSynchronize(s);  // the bank upload / precompute may still read the caller's weights
    return st;
  }
  // every exit after the pipeline starts drains all three streams first: queued async copies
  // must not touch the caller's host buffers after this call has returned (even with an error)
  auto drain = [&](int status) {
    cudaStreamSynchronize(c.h2d);
    cudaStreamSynchronize(s);
    cudaStreamSynchronize(c.d2h);
    return status;
  };
#define RC_PIPE(call)                                          \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return drain(cuda_fail(e_, #call)); \
  } while (0)
  const size_t xi = xb / d->n, yi = yb / d->n, ai = ab / d->n;
  for (int k = 0; k < chunks; ++k) {
    int b = 0, e = 0;
    rc_shard_range(d->n, chunks, k, &b, &e);
    if (e == b) continue;
    cudaEvent_t in_ready = c.ev[2 * k], out_ready = c.ev[2 * k + 1];
    RC_PIPE(cudaMemcpyAsync((char*)dx + b * xi, (const char*)h_x + b * xi, (e - b) * xi, cudaMemcpyHostToDevice,
                            c.h2d));
    RC_PIPE(cudaEventRecord(in_ready, c.h2d));
    RC_PIPE(cudaStreamWaitEvent(s, in_ready, 0));
    rc_desc cd = *d;
    cd.n = e - b;
    st = dispatch(cd, (const float*)((char*)dx + b * xi), dbank, (const float*)dbias, (float*)((char*)dy + b * yi),
                  da ? (uint8_t*)da + b * ai : nullptr, dws, wsb, s, false, nullptr);
    if (st != RC_OK) return drain(st);
    RC_PIPE(cudaEventRecord(out_ready, s));
    RC_PIPE(cudaStreamWaitEvent(c.d2h, out_ready, 0));
    RC_PIPE(cudaMemcpyAsync((char*)h_y + b * yi, (char*)dy + b * yi, (e - b) * yi, cudaMemcpyDeviceToHost, c.d2h));
    if (has_arg)
      RC_PIPE(cudaMemcpyAsync(h_argmax + b * ai, (uint8_t*)da + b * ai, (e - b) * ai, cudaMemcpyDeviceToHost, c.d2h));
  }
#undef RC_PIPE
  RC_CUDA(cudaStreamSynchronize(c.d2h));
  RC_CUDA(cudaStreamSynchronize(s));
  return RC_OK;
}

int rc_steer(const float* d_fx, const float* d_fy, size_t count, double theta, float* d_out, void* stream) {
  if (count > 0 && (!d_fx || !d_fy || !d_out)) return fail(RC_ERR_INVALID, "steer: null pointer");
  return launch_steer(d_fx, d_fy, count, theta, d_out, static_cast<cudaStream_t>(stream));
}

int rc_steer_host(const float* h_fx, const float* h_fy, size_t count, double theta, float* h_out, int device) {
  if (device < 0 || device >= 64) return fail(RC_ERR_INVALID, "steer: bad device");
  if (count == 0) return RC_OK;
  if (!h_fx || !h_fy || !h_out) return fail(RC_ERR_INVALID, "steer: null pointer");
  DeviceGuard guard(device);
  DeviceCache& c = g_cache[device];
  std::lock_guard<std::mutex> lock(c.mu);
  if (!c.stream) RC_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  const size_t b = count * sizeof(float);
  void* dx = c.get(0, b);
  void* dy = c.get(1, b);
  void* dout = c.get(2, b);
  if (!dx || !dy || !dout) return fail(RC_ERR_CUDA, "steer: device allocation failed");
  cudaStream_t s = c.stream;
  RC_CUDA(cudaMemcpyAsync(dx, h_fx, b, cudaMemcpyHostToDevice, s));
  RC_CUDA(cudaMemcpyAsync(dy, h_fy, b, cudaMemcpyHostToDevice, s));
  int st = launch_steer((const float*)dx, (const float*)dy, count, theta, (float*)dout, s);
  if (st != RC_OK) {  // drain the queued copies of the caller's host buffers first
    cudaStreamSynchronize(s);
    return st;
  }
  RC_CUDA(cudaMemcpyAsync(h_out, dout, b, cudaMemcpyDeviceToHost, s));
  RC_CUDA(cudaStreamSynchronize(s));
  return RC_OK;
}

int rc_orientation_bank_host(const rc_desc* d, const float* h_w0, const float* h_w1, float* h_kernels,
                             int device) {
  RC_CHECK_DESC(d);
  if (device < 0 || device >= 64) return fail(RC_ERR_INVALID, "orientation_bank: bad device");
  if (!h_w0 || !h_kernels || (d->group == RC_GROUP_STEER && !h_w1))
    return fail(RC_ERR_INVALID, "orientation_bank: null pointer");
  DeviceGuard guard(device);
  DeviceCache& c = g_cache[device];
  std::lock_guard<std::mutex> lock(c.mu);
  if (!c.stream) RC_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  const size_t wb = (size_t)d->c_out * d->c_in * d->k * d->k * sizeof(float);
  const size_t kb = wb * (size_t)num_bases(*d) * rot_per_base(*d);
  void* dw0 = c.get(1, wb);
  void* dw1 = d->group == RC_GROUP_STEER ? c.get(2, wb) : nullptr;
  void* dbank = c.get(4, bank_layout(*d).total);
  void* dk = c.get(5, kb);
  if (!dw0 || !dbank || !dk || (d->group == RC_GROUP_STEER && !dw1))
    return fail(RC_ERR_CUDA, "orientation_bank: device allocation failed");
  cudaStream_t s = c.stream;
  RC_CUDA(cudaMemcpyAsync(dw0, h_w0, wb, cudaMemcpyHostToDevice, s));
  if (dw1) RC_CUDA(cudaMemcpyAsync(dw1, h_w1, wb, cudaMemcpyHostToDevice, s));
  int st = launch_bank(*d, (const float*)dw0, (const float*)dw1, dbank, s);
  if (st != RC_OK) {  // drain the queued copies of the caller's host buffers first
    cudaStreamSynchronize(s);
    return st;
  }
  st = launch_orientation_bank(*d, dbank, (float*)dk, s);
  if (st != RC_OK) {  // drain the queued copies of the caller's host buffers first
    cudaStreamSynchronize(s);
    return st;
  }
  RC_CUDA(cudaMemcpyAsync(h_kernels, dk, kb, cudaMemcpyDeviceToHost, s));
  RC_CUDA(cudaStreamSynchronize(s));
  return RC_OK;
}

int rc_orientation_pool_host(int n, int c_out, int r, int h, int w, int pool, int pool_group,
                             const float* h_f, const float* h_bias, float* h_y, uint8_t* h_argmax,
                             int device) {
  if (n < 0 || c_out < 1 || r < 1 || h < 1 || w < 1)
    return fail(RC_ERR_INVALID, "OrientedFeature: dimensions must be positive");
  if (pool == RC_POOL_SUBGROUP && (pool_group < 1 || r % pool_group != 0))
    return fail(RC_ERR_INVALID, "subgroup_pool_max: R not divisible by group_size");
  if (pool < RC_POOL_NONE || pool > RC_POOL_SUBGROUP) return fail(RC_ERR_INVALID, "ri_conv: unknown pool");
  if (device < 0 || device >= 64) return fail(RC_ERR_INVALID, "orientation_pool: bad device");
  if (n == 0) return RC_OK;
  const int gf = pool == RC_POOL_SUBGROUP ? pool_group : (pool == RC_POOL_NONE ? 1 : r);
  const size_t plane = (size_t)h * w;
  const size_t fb = (size_t)n * c_out * r * plane * sizeof(float);
  const size_t yb = (size_t)n * c_out * (r / gf) * plane * sizeof(float);
  const bool has_arg = h_argmax && pool != RC_POOL_AVG;
  DeviceGuard guard(device);
  DeviceCache& c = g_cache[device];
  std::lock_guard<std::mutex> lock(c.mu);
  if (!c.stream) RC_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  void* df = c.get(0, fb);
  void* dbias = h_bias ? c.get(3, c_out * sizeof(float)) : nullptr;
  void* dy = c.get(5, yb);
  void* da = has_arg ? c.get(6, yb / sizeof(float)) : nullptr;
  if (!df || !dy || (h_bias && !dbias) || (has_arg && !da))
    return fail(RC_ERR_CUDA, "orientation_pool: device allocation failed");
  cudaStream_t s = c.stream;
  RC_CUDA(cudaMemcpyAsync(df, h_f, fb, cudaMemcpyHostToDevice, s));
  if (dbias) RC_CUDA(cudaMemcpyAsync(dbias, h_bias, c_out * sizeof(float), cudaMemcpyHostToDevice, s));
  int st = launch_pool(n, c_out, r, h, w, pool, pool_group, (const float*)df, (const float*)dbias, (float*)dy,
                       (uint8_t*)da, s);
  if (st != RC_OK) {  // drain the queued copies of the caller's host buffers first
    cudaStreamSynchronize(s);
    return st;
  }
  RC_CUDA(cudaMemcpyAsync(h_y, dy, yb, cudaMemcpyDeviceToHost, s));
  if (has_arg) RC_CUDA(cudaMemcpyAsync(h_argmax, da, yb / sizeof(float), cudaMemcpyDeviceToHost, s));
  RC_CUDA(cudaStreamSynchronize(s));
  return RC_OK;
}

// Batch-sharded multi-GPU forward: contiguous shards (rc_shard_range), one
// host thread per device; every device builds the same bank from the same weights and
// each shard lands directly in its slice of the caller's host output (no collective).
int rc_mgpu_forward_host(const rc_desc* d, const float* h_x, const float* h_w0, const float* h_w1,
                         const float* h_bias, float* h_y, uint8_t* h_argmax, int n_devices,
                         const int* devices) {
  RC_CHECK_DESC(d);
  if (n_devices < 1 || n_devices > 64) return fail(RC_ERR_INVALID, "mgpu_forward: need 1..64 devices");
  int count = 0;
  RC_CUDA(cudaGetDeviceCount(&count));
  for (int i = 0; i < n_devices; ++i) {
    const int dev = devices ? devices[i] : i;
    if (dev < 0 || dev >= count) return fail(RC_ERR_INVALID, "mgpu_forward: bad device");
    for (int j = 0; j < i; ++j)
      if ((devices ? devices[j] : j) == dev) return fail(RC_ERR_INVALID, "mgpu_forward: duplicate device");
  }
  const size_t x_img = (size_t)d->c_in * d->h * d->w;
  const size_t y_img = (size_t)d->c_out * out_orientations(*d) * d->h * d->w;
  std::vector<int> status(n_devices, RC_OK);
  std::vector<std::string> msg(n_devices);
  std::vector<std::thread> workers;
  for (int i = 0; i < n_devices; ++i) {
    int b = 0, e = 0;
    rc_shard_range(d->n, n_devices, i, &b, &e);
    workers.emplace_back([&, i, b, e] {
      rc_desc ld = *d;
      ld.n = e - b;
      const int dev = devices ? devices[i] : i;
      status[i] = rc_ri_conv_forward_host(&ld, h_x + (size_t)b * x_img, h_w0, h_w1, h_bias,
                                          h_y + (size_t)b * y_img,
                                          h_argmax ? h_argmax + (size_t)b * y_img : nullptr, dev);
      if (status[i] != RC_OK) msg[i] = g_err;  // g_err is thread-local: copy it out
    });
  }
  for (auto& t : workers) t.join();
  for (int i = 0; i < n_devices; ++i)
    if (status[i] != RC_OK)
      return fail(status[i], "mgpu_forward: device " + std::to_string(i) + ": " + msg[i]);
  return RC_OK;
}

int rc_tiled_scatter_conv_host(const float* h_x, int c_in, int h, int w, const float* h_wt,
                               int c_out, int in_channels_w, int kh, int kw, int tile_h,
                               int tile_w, int halo, int workers, int strategy, float* h_y,
                               unsigned long long* mults, unsigned long long* adds,
                               unsigned long long* aux_bytes, int precision, int device) {
  // scatter_conv.hpp:339-346, same order and messages
  if (c_in != in_channels_w) return fail(RC_ERR_INVALID, "tiled_scatter_conv: channel mismatch");
  if (kh != kw) return fail(RC_ERR_INVALID, "tiled_scatter_conv: kernel must be square");
  if (tile_h < 1 || tile_w < 1) return fail(RC_ERR_INVALID, "tiled_scatter_conv: tile dims must be >= 1");
  if (halo != kh / 2) return fail(RC_ERR_INVALID, "tiled_scatter_conv: invalid halo");
  if (workers < 1) return fail(RC_ERR_INVALID, "tiled_scatter_conv: workers must be >= 1");
  rc_desc d{1, c_in, h, w, c_out, kh, RC_GROUP_SINGLE, 1, RC_POOL_NONE, 1, RC_CONV_SCATTER, precision, RC_ACT_NONE};
  int st = rc_ri_conv_forward_host(&d, h_x, h_wt, nullptr, nullptr, h_y, nullptr, device);
  if (st != RC_OK) return st;
  if (mults) *mults = (unsigned long long)h * w * kh * kw * c_in * c_out;  // :361-366
  if (adds) *adds = rc_clipped_writes(h, w, kh, kw) * c_out;
  // AuxMemCounter keeps the reference's accounting (:351-360): the per-worker private tile
  // accumulators of tile_private, none for phase_parallel.  The GPU path's own staging is
  // reported by rc_workspace_size.
  if (aux_bytes)
    *aux_bytes = strategy == 0 ? (unsigned long long)tile_h * tile_w * sizeof(float) * workers : 0ull;
  return RC_OK;
}

}  // extern "C"
