// transform_b200.cpp — B200 drop-in for the reference's transform module.
//
// Implements every function declared by the reference's UNCHANGED header
// /root/reference/proj/include/qtensor/transform.hpp:13-64.  The tube
// transforms qfft3_conj / qifft3_conj and the vector FFTs fft_vec / ifft_vec
// run on the GPU through the C-ABI (a vector is one 1x1 tube); dft_vec_naive
// stays the direct O(p^2) summation it is documented to be (the oracle the
// fast transform is tested against, transform.hpp:13-15).
#include <algorithm>
#include <cmath>
#include <numbers>
#include <stdexcept>

#include "b200_dropin_common.hpp"
#include "qtensor/transform.hpp"

namespace qtensor {

std::vector<Cx> dft_vec_naive(std::span<const Cx> x) {
  if (x.empty()) throw std::invalid_argument("dft_vec_naive: empty vector");
  const std::size_t p = x.size();
  std::vector<Cx> y(p);
  for (std::size_t s = 0; s < p; ++s) {
    Cx acc{};
    for (std::size_t r = 0; r < p; ++r) {
      const double ang = -2.0 * std::numbers::pi * static_cast<double>((s * r) % p) / static_cast<double>(p);
      acc += Cx{std::cos(ang), std::sin(ang)} * x[r];
    }
    y[s] = acc;
  }
  return y;
}

// y = F(x): the t1 channel of qfft3_conj computes F(conj(t1)), so feed conj(x).
std::vector<Cx> fft_vec(std::span<const Cx> x) {
  if (x.empty()) throw std::invalid_argument("fft_vec: empty vector");
  const std::size_t p = x.size();
  std::vector<Cx> in1(p), in2(p), y(p), y2(p);
  for (std::size_t k = 0; k < p; ++k) in1[k] = std::conj(x[k]);
  b200::check(qt_qfft3_conj_f64_host(b200::dp(in1), b200::dp(in2), b200::dp(y), b200::dp(y2), 1, 1, p,
                                     b200::device()),
              "fft_vec");
  return y;
}

// ifft(y) = conj(t1 channel of qifft3_conj(y)).
std::vector<Cx> ifft_vec(std::span<const Cx> y) {
  if (y.empty()) throw std::invalid_argument("ifft_vec: empty vector");
  const std::size_t p = y.size();
  std::vector<Cx> in1(y.begin(), y.end()), in2(p), out(p), out2(p);
  b200::check(qt_qifft3_conj_f64_host(b200::dp(in1), b200::dp(in2), b200::dp(out), b200::dp(out2), 1, 1, p,
                                      b200::device()),
              "ifft_vec");
  for (Cx& z : out) z = std::conj(z);
  return out;
}

CdMatrix CdTensor3::slice(std::size_t r) const {
  CdMatrix out(m, n);
  const auto off = static_cast<std::ptrdiff_t>(r * m * n), len = static_cast<std::ptrdiff_t>(m * n);
  out.a1.data.assign(t1.begin() + off, t1.begin() + off + len);
  out.a2.data.assign(t2.begin() + off, t2.begin() + off + len);
  return out;
}

void CdTensor3::set_slice(std::size_t r, const CdMatrix& s) {
  if (s.rows() != m || s.cols() != n) throw std::invalid_argument("set_slice: slice shape mismatch");
  const auto off = static_cast<std::ptrdiff_t>(r * m * n);
  std::copy(s.a1.data.begin(), s.a1.data.end(), t1.begin() + off);
  std::copy(s.a2.data.begin(), s.a2.data.end(), t2.begin() + off);
}

double CdTensor3::frob_norm() const {
  double acc = 0.0;
  for (const Cx& z : t1) acc += std::norm(z);
  for (const Cx& z : t2) acc += std::norm(z);
  return std::sqrt(acc);
}

CdTensor3 qfft3_conj(const CdTensor3& q) {
  CdTensor3 out(q.m, q.n, q.p);
  b200::check(qt_qfft3_conj_f64_host(b200::dp(q.t1), b200::dp(q.t2), b200::dp(out.t1), b200::dp(out.t2), q.m, q.n,
                                     q.p, b200::device()),
              "qfft3_conj");
  return out;
}

CdTensor3 qifft3_conj(const CdTensor3& qhat) {
  CdTensor3 out(qhat.m, qhat.n, qhat.p);
  b200::check(qt_qifft3_conj_f64_host(b200::dp(qhat.t1), b200::dp(qhat.t2), b200::dp(out.t1), b200::dp(out.t2),
                                      qhat.m, qhat.n, qhat.p, b200::device()),
              "qifft3_conj");
  return out;
}

}  // namespace qtensor
