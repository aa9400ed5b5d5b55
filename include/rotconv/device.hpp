// rotconv/device.hpp -- the glue between the drop-in C++ API and the C-ABI
// (include/rotconv_c.h, librotconv_b200.so).
//
// * Which GPU a call runs on: a per-thread current device (default 0), set with
//   rotconv::b200::set_device(d) or scoped with rotconv::b200::DeviceScope.  The
//   reference runs on host threads only (scatter_conv.hpp:247-255); its ops are pure and
//   reentrant, and so are these: each call stages through the library's per-device
//   buffers under a per-device mutex.
// * Errors: the C-ABI returns status codes.  RC_ERR_INVALID becomes std::invalid_argument
//   with the reference's message (e.g. "tiled_scatter_conv: invalid halo",
//   scatter_conv.hpp:345); every other failure becomes std::runtime_error.
// * Arithmetic: the ops take float32 in and out (the reference's benchmark mode,
//   tensor.hpp:16-17).  The channel contraction runs in the per-thread default precision
//   (rotconv::b200::precision(), default Precision::automatic = the FP32-tolerance
//   tcgen05 kernels where a shape has one, FP32 CUDA cores otherwise); set it with
//   set_precision() or scope it with PrecisionScope (e.g. Precision::fp32 for the
//   CUDA-core FFMA path).  Instantiating a GPU op with T = double is a compile-time
//   error -- there is no CPU fallback in the product.
#pragma once

#include <stdexcept>
#include <string>
#include <type_traits>

#include "rotconv_c.h"

namespace rotconv {
namespace b200 {

inline int& current_device_slot() {
  thread_local int dev = 0;
  return dev;
}
inline int device() { return current_device_slot(); }
inline void set_device(int d) { current_device_slot() = d; }

class DeviceScope {
 public:
  explicit DeviceScope(int d) : prev_(device()) { set_device(d); }
  ~DeviceScope() { set_device(prev_); }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;

 private:
  int prev_;
};

// precision of the channel contraction for the fused layer (rc_precision)
enum class Precision { automatic = RC_PREC_AUTO, fp32 = RC_PREC_FP32, bf16x3 = RC_PREC_BF16X3, bf16 = RC_PREC_BF16 };

// per-thread default precision of the reference-signature drop-ins (scatter_conv.hpp,
// group_conv.hpp), which have no precision argument
inline Precision& current_precision_slot() {
  thread_local Precision p = Precision::automatic;
  return p;
}
inline Precision precision() { return current_precision_slot(); }
inline void set_precision(Precision p) { current_precision_slot() = p; }

class PrecisionScope {
 public:
  explicit PrecisionScope(Precision p) : prev_(precision()) { set_precision(p); }
  ~PrecisionScope() { set_precision(prev_); }
  PrecisionScope(const PrecisionScope&) = delete;
  PrecisionScope& operator=(const PrecisionScope&) = delete;

 private:
  Precision prev_;
};

inline void throw_on(int status) {
  if (status == RC_OK) return;
  const char* m = rc_last_error();
  const std::string msg = m ? m : "rotconv: unknown error";
  if (status == RC_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg + " [status " + std::to_string(status) + "]");
}

template <typename T>
struct gpu_scalar {
  static constexpr bool ok = std::is_same_v<T, float>;
};

}  // namespace b200

#define ROTCONV_REQUIRE_FLOAT(T)                                                           \
  static_assert(::rotconv::b200::gpu_scalar<T>::ok,                                        \
                "rotconv B200 ops compute in float32 on the GPU; double is the reference " \
                "oracle's correctness mode and has no device path")

}  // namespace rotconv
