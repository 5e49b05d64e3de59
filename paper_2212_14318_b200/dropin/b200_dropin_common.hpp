// b200_dropin_common.hpp — shared glue of the C++ drop-in sources: device
// selection and mapping of C-ABI status codes to the reference's exceptions.
#pragma once

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "qtensor_b200.h"

namespace qtensor::b200 {

// Device the drop-in runs on: $QTENSOR_B200_DEVICE, default 0.
inline int device() {
  const char* env = std::getenv("QTENSOR_B200_DEVICE");
  return env && *env ? std::atoi(env) : 0;
}

// $QTB_DROPIN_FILL_WS=1: tprod_fast(a, b, ws) leaves Â, B̂, Ĉ in ws as the
// reference does (tproduct.cpp:80-87); off by default (nothing reads them back)
inline bool fill_workspace() {
  const char* env = std::getenv("QTB_DROPIN_FILL_WS");
  return env && *env == '1';
}

// $QTB_DROPIN_NAIVE=gpu: tprod_naive (the definitional oracle) on the B200;
// default: the reference's own CPU definition (an independent checker)
inline bool naive_on_gpu() {
  const char* env = std::getenv("QTB_DROPIN_NAIVE");
  return env && std::string(env) == "gpu";
}

// QT_EINVAL -> std::invalid_argument (what the reference throws), anything else
// -> std::runtime_error.  There is no CPU fallback: a missing GPU is an error.
inline void check(int rc, const char* who) {
  if (rc == QT_OK) return;
  std::string msg = std::string(who) + ": " + qt_last_error();
  if (rc == QT_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

template <class V>
inline const double* dp(const V& v) {
  return reinterpret_cast<const double*>(v.data());
}
template <class V>
inline double* dp(V& v) {
  return reinterpret_cast<double*>(v.data());
}

}  // namespace qtensor::b200
