// tproduct_b200.cpp — B200 drop-in for the reference's tproduct module.
//
// Implements every function declared by the reference's UNCHANGED header
// /root/reference/proj/include/qtensor/tproduct.hpp:12-56, so a maintainer
// swaps proj/src/tproduct.cpp for this file and links libqtensor_b200.so
// (INTEGRATION.md).  tprod_fast — the hot path — runs the sm_100a pipeline
// through the C-ABI (qt_tprod_f64_host, include/qtensor_b200.h); the
// remaining functions are the small layout helpers and the definitional
// product the reference ships alongside it.
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "b200_dropin_common.hpp"
#include "qtensor/tproduct.hpp"

namespace qtensor {

// (m p) x n matrix whose row block r is slice r (tproduct.hpp:11-12).
CdMatrix unfold(const CdTensor3& a) {
  CdMatrix out(a.m * a.p, a.n);
  out.a1.data.assign(a.t1.begin(), a.t1.end());
  out.a2.data.assign(a.t2.begin(), a.t2.end());
  return out;
}

// Inverse of unfold (tproduct.hpp:14-15): row count must be a multiple of p.
CdTensor3 fold(const CdMatrix& mat, std::size_t p) {
  if (p == 0 || mat.rows() % p != 0) throw std::invalid_argument("fold: row count not divisible by p");
  CdTensor3 out(mat.rows() / p, mat.cols(), p);
  out.t1.assign(mat.a1.data.begin(), mat.a1.data.end());
  out.t2.assign(mat.a2.data.begin(), mat.a2.data.end());
  return out;
}

// mp x np block circulant, block (row r, col c) = slice (r - c) mod p
// (tproduct.hpp:17-18).
CdMatrix bcirc_of_tensor(const CdTensor3& a) {
  const std::size_t m = a.m, n = a.n, p = a.p;
  CdMatrix out(m * p, n * p);
  for (std::size_t r = 0; r < p; ++r)
    for (std::size_t c = 0; c < p; ++c) {
      const std::size_t slice = (r + p - c) % p;
      for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < n; ++j) {
          const std::size_t from = (slice * m + i) * n + j;
          const std::size_t to = (r * m + i) * (n * p) + c * n + j;
          out.a1.data[to] = a.t1[from];
          out.a2.data[to] = a.t2[from];
        }
    }
  return out;
}

// Identity of the T-product: I_n in slice 0, zeros elsewhere (tproduct.hpp:20-21).
CdTensor3 identity_tensor(std::size_t n, std::size_t p) {
  if (n == 0 || p == 0) throw std::invalid_argument("identity_tensor: zero dims");
  CdTensor3 out(n, n, p);
  for (std::size_t i = 0; i < n; ++i) out.t1[i * n + i] = Cx{1.0, 0.0};
  return out;
}

// Definitional product fold(bcirc(a) . unfold(b)) (tproduct.hpp:23-25) — the
// oracle the fast path is checked against.  By default it stays what the
// reference computes (its own CPU qmatmul of the materialised block circulant,
// linalg.cpp:170-176), so the reference's fast-vs-naive tests and the
// acceptance gate compare the GPU product against an independent CPU oracle
// and criterion 2 measures the speed-up shape it was written for.  With
// $QTB_DROPIN_NAIVE=gpu it runs on the B200 instead: C_k = sum_r
// A_{(k-r) mod p} (.) B_r without materialising bcirc (qt_tprod_naive_f64_host,
// csrc/qt_naive.cu).
CdTensor3 tprod_naive(const CdTensor3& a, const CdTensor3& b) {
  if (a.n != b.m || a.p != b.p) throw std::invalid_argument("tprod_naive: dimension mismatch");
  if (!b200::naive_on_gpu()) return fold(qmatmul(bcirc_of_tensor(a), unfold(b)), a.p);
  CdTensor3 c(a.m, b.n, a.p);
  b200::check(qt_tprod_naive_f64_host(b200::dp(a.t1), b200::dp(a.t2), b200::dp(b.t1), b200::dp(b.t2),
                                      b200::dp(c.t1), b200::dp(c.t2), a.m, a.n, b.n, a.p, b200::device()),
              "tprod_naive");
  return c;
}

// FFT-domain T-product on the B200 (tproduct.hpp:35-46).  By default the
// transformed operands live in stream-ordered device scratch and `ws` is left
// untouched (no caller in the reference reads it back; the copies would cost
// three extra PCIe transfers); with $QTB_DROPIN_FILL_WS=1 the call leaves Â,
// B̂ and Ĉ in ws.ahat / ws.bhat / ws.chat exactly as the reference does
// (tproduct.cpp:80-87), from the product's own kernels
// (qt_tprod_f64_host_spectra).  Repeated calls (with or without a workspace)
// are bitwise identical, the property test_tproduct.cpp:118-128 pins.
CdTensor3 tprod_fast(const CdTensor3& a, const CdTensor3& b, TProdWorkspace& ws) {
  if (a.n != b.m || a.p != b.p) throw std::invalid_argument("tprod_fast: dimension mismatch");
  CdTensor3 c(a.m, b.n, a.p);
  if (b200::fill_workspace()) {
    ws.ahat = CdTensor3(a.m, a.n, a.p);
    ws.bhat = CdTensor3(b.m, b.n, b.p);
    ws.chat = CdTensor3(a.m, b.n, a.p);
    b200::check(qt_tprod_f64_host_spectra(b200::dp(a.t1), b200::dp(a.t2), b200::dp(b.t1), b200::dp(b.t2),
                                          b200::dp(c.t1), b200::dp(c.t2), a.m, a.n, b.n, a.p, b200::device(),
                                          b200::dp(ws.ahat.t1), b200::dp(ws.ahat.t2), b200::dp(ws.bhat.t1),
                                          b200::dp(ws.bhat.t2), b200::dp(ws.chat.t1), b200::dp(ws.chat.t2)),
                "tprod_fast");
    return c;
  }
  b200::check(qt_tprod_f64_host(b200::dp(a.t1), b200::dp(a.t2), b200::dp(b.t1), b200::dp(b.t2), b200::dp(c.t1),
                                b200::dp(c.t2), a.m, a.n, b.n, a.p, b200::device()),
              "tprod_fast");
  return c;
}

CdTensor3 tprod_fast(const CdTensor3& a, const CdTensor3& b) {
  TProdWorkspace ws;
  return tprod_fast(a, b, ws);
}

// Operation counts of both routes (tproduct.hpp:48-56).
TprodFlops flops_estimate(std::size_t m, std::size_t n, std::size_t s, std::size_t p) {
  if (m == 0 || n == 0 || s == 0 || p == 0) throw std::invalid_argument("flops_estimate: zero dims");
  const std::uint64_t M = m, N = n, S = s, P = p;
  TprodFlops f;
  f.fast_mults = 16 * M * N * S * P;
  const double lg = p > 1 ? std::log2(static_cast<double>(p)) : 0.0;
  f.fast_transform_flops =
      static_cast<std::uint64_t>(std::llround(2.0 * static_cast<double>(M * N + N * S + M * S) * P * lg));
  f.naive_mults = f.fast_mults * P;
  f.naive_adds = 4 * M * P * S * (N * P - 1) + 12 * M * N * S * P * P;
  return f;
}

}  // namespace qtensor
