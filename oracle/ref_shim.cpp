// ref_shim.cpp — C-ABI over the reference compiled from its own sources.
// TEST INFRASTRUCTURE ONLY (oracle/_ref): lets the Python tests, the golden
// fixture generator and bench.py's reference arm call the UNMODIFIED
// reference (namespace renamed qtensor -> qtref at compile time, -Dqtensor=qtref)
// through plain pointers.  The reference's own code does all the work; this
// file only copies arrays in and out of its CdTensor3 containers.
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>

#include "qtensor/rng.hpp"
#include "qtensor/tensor_io.hpp"
#include "qtensor/tproduct.hpp"
#include "qtensor/transform.hpp"

using qtref::CdTensor3;
using qtref::Cx;

namespace {
CdTensor3 in_tensor(const double* t1, const double* t2, uint64_t m, uint64_t n, uint64_t p) {
  CdTensor3 t(m, n, p);
  if (t.size()) {
    std::memcpy(t.t1.data(), t1, t.size() * sizeof(Cx));
    std::memcpy(t.t2.data(), t2, t.size() * sizeof(Cx));
  }
  return t;
}
void out_tensor(const CdTensor3& t, double* t1, double* t2) {
  if (t.size()) {
    std::memcpy(t1, t.t1.data(), t.size() * sizeof(Cx));
    std::memcpy(t2, t.t2.data(), t.size() * sizeof(Cx));
  }
}
}  // namespace

extern "C" {

// 0 ok, 1 std::invalid_argument, 2 other exception
int ref_tprod_fast(const double* a1, const double* a2, const double* b1, const double* b2, double* c1, double* c2,
                   uint64_t m, uint64_t n, uint64_t bm, uint64_t s, uint64_t p, uint64_t bp) {
  try {
    CdTensor3 a = in_tensor(a1, a2, m, n, p), b = in_tensor(b1, b2, bm, s, bp);
    out_tensor(qtref::tprod_fast(a, b), c1, c2);
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 2;
  }
}

int ref_tprod_naive(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                    double* c2, uint64_t m, uint64_t n, uint64_t bm, uint64_t s, uint64_t p, uint64_t bp) {
  try {
    CdTensor3 a = in_tensor(a1, a2, m, n, p), b = in_tensor(b1, b2, bm, s, bp);
    out_tensor(qtref::tprod_naive(a, b), c1, c2);
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 2;
  }
}

int ref_qfft3_conj(const double* x1, const double* x2, double* y1, double* y2, uint64_t m, uint64_t n, uint64_t p) {
  try {
    out_tensor(qtref::qfft3_conj(in_tensor(x1, x2, m, n, p)), y1, y2);
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

int ref_qifft3_conj(const double* x1, const double* x2, double* y1, double* y2, uint64_t m, uint64_t n,
                    uint64_t p) {
  try {
    out_tensor(qtref::qifft3_conj(in_tensor(x1, x2, m, n, p)), y1, y2);
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

int ref_fft_vec(const double* x, uint64_t n, double* y) {
  try {
    std::span<const Cx> in(reinterpret_cast<const Cx*>(x), n);
    auto out = qtref::fft_vec(in);
    std::memcpy(y, out.data(), n * sizeof(Cx));
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

int ref_gen_random_tensor(uint64_t m, uint64_t n, uint64_t p, uint64_t seed, double* t1, double* t2) {
  try {
    out_tensor(qtref::gen_random_tensor(m, n, p, seed), t1, t2);
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

// write_tensor / read_tensor (tensor_io.cpp:85-103): 0 ok, 6/7/8 TensorIoError kind, 9 other
int ref_write_tensor(const char* path, const double* t1, const double* t2, uint64_t m, uint64_t n, uint64_t p) {
  try {
    qtref::write_tensor(path, in_tensor(t1, t2, m, n, p));
    return 0;
  } catch (...) {
    return 9;
  }
}

int ref_read_tensor(const char* path, double* t1, double* t2, uint64_t* dims) {
  try {
    CdTensor3 t = qtref::read_tensor(path);
    dims[0] = t.m;
    dims[1] = t.n;
    dims[2] = t.p;
    if (t1) out_tensor(t, t1, t2);
    return 0;
  } catch (const qtref::TensorIoError& e) {
    return 6 + static_cast<int>(e.kind());
  } catch (...) {
    return 9;
  }
}

uint64_t ref_derive_seed(uint64_t base, uint64_t stream) { return qtref::derive_seed(base, stream); }

uint64_t ref_flops(uint64_t m, uint64_t n, uint64_t s, uint64_t p, uint64_t* out) {
  try {
    auto f = qtref::flops_estimate(m, n, s, p);
    out[0] = f.fast_mults;
    out[1] = f.fast_transform_flops;
    out[2] = f.naive_mults;
    out[3] = f.naive_adds;
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

}  // extern "C"
