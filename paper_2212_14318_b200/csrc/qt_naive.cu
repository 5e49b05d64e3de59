// qt_naive.cu — the definitional T-product on the GPU.
//
// tprod_naive(a, b) = fold(bcirc(a) . unfold(b))  (/root/reference/proj/src/tproduct.cpp:49-53)
// never materialises bcirc(a) here: block (k, r) of bcirc(a) is slice
// (k - r) mod p (tproduct.cpp:25-39), so slice k of C is
//     C_k = sum_r  A_{(k-r) mod p} (.) B_r
// with (.) the Cayley-Dickson quaternion matrix product of qmatmul
// (linalg.hpp:90, linalg.cpp:170-176):
//     (a1 + a2 j)(b1 + b2 j) = (a1 b1 - a2 conj(b2)) + (a1 b2 + a2 conj(b1)) j.
// One CTA owns a tile of slice k and runs K = p*n steps (r ascending, then the
// inner index, as the reference's cmatmul walks bcirc's columns) through the
// same DMMA tile machinery as the spectral GEMM.  16 m n s p^2 real
// multiplications: an independent O(p^2) cross-check of the fast path, and the
// GPU implementation behind the drop-in's tprod_naive.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "qt_dmma_tile.cuh"
#include "qt_internal.cuh"

namespace qtb {

namespace {

// C1 += A1 B1 - A2 conj(B2);  C2 += A1 B2 + A2 conj(B1)   (components 0..3 =
// C1 re, C1 im, C2 re, C2 im; planes 0, 1 of the staged tile = part 1, 2)
template <class C>
__device__ __forceinline__ void mma_stage_naive(const double2* sa, const double2* sb, double (&acc)[4][C::RB][2],
                                                int wm, int wn, int g, int q) {
#pragma unroll
  for (int ks = 0; ks < C::BK / 4; ++ks) {
    const int kb = ks * 4 + q;
    const int jb = (wn * 8 + g) ^ (q << 1);
    const double2 b1 = sb[0 * C::B_PLANE + kb * C::BN + jb];
    const double2 b2 = sb[1 * C::B_PLANE + kb * C::BN + jb];
    const double nb1i = dneg(b1.y), nb2r = dneg(b2.x), nb2i = dneg(b2.y);
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb) {
      const int i = wm * (C::RB * 8) + rb * 8 + g;
      const int ca = (ks * 4 + q) ^ ((i & 1) << 2);
      const double2 a1 = sa[0 * C::A_PLANE + i * C::BK + ca];
      const double2 a2 = sa[1 * C::A_PLANE + i * C::BK + ca];
      dmma(acc[0][rb], a1.x, b1.x);  // C1 re: a1r b1r - a1i b1i - a2r b2r - a2i b2i
      dmma(acc[0][rb], a1.y, nb1i);
      dmma(acc[0][rb], a2.x, nb2r);
      dmma(acc[0][rb], a2.y, nb2i);
      dmma(acc[1][rb], a1.x, b1.y);  // C1 im: a1r b1i + a1i b1r + a2r b2i - a2i b2r
      dmma(acc[1][rb], a1.y, b1.x);
      dmma(acc[1][rb], a2.x, b2.y);
      dmma(acc[1][rb], a2.y, nb2r);
      dmma(acc[2][rb], a1.x, b2.x);  // C2 re: a1r b2r - a1i b2i + a2r b1r + a2i b1i
      dmma(acc[2][rb], a1.y, nb2i);
      dmma(acc[2][rb], a2.x, b1.x);
      dmma(acc[2][rb], a2.y, b1.y);
      dmma(acc[3][rb], a1.x, b2.y);  // C2 im: a1r b2i + a1i b2r - a2r b1i + a2i b1r
      dmma(acc[3][rb], a1.y, b2.x);
      dmma(acc[3][rb], a2.x, nb1i);
      dmma(acc[3][rb], a2.y, b1.x);
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
    naive_tprod_kernel(const double2* __restrict__ a1, const double2* __restrict__ a2,
                       const double2* __restrict__ b1, const double2* __restrict__ b2, double2* __restrict__ c1,
                       double2* __restrict__ c2, int m, int n, int s, int p, int slice0) {
  extern __shared__ double2 smem[];
  const int k = slice0 + blockIdx.y;
  const int ntm = (m + C::BM - 1) / C::BM;
  const int tm = blockIdx.x % ntm, tn = blockIdx.x / ntm;
  const int row0 = tm * C::BM, col0 = tn * C::BN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp % C::WM, wn = warp / C::WM;
  const size_t amn = (size_t)m * n, bns = (size_t)n * s, cms = (size_t)m * s;
  const int ktn = (n + C::BK - 1) / C::BK;
  const int ktiles = p * ktn;  // r outer, inner index tiles inner
  auto stage_args = [&](int kt, int* kk) {
    const int r = kt / ktn;
    *kk = kt - r * ktn;
    const int ar = (k - r + p) % p;
    PairArgs P;
    P.a[0] = a1 + ar * amn;
    P.a[1] = a2 + ar * amn;
    P.a[2] = P.a[0];
    P.a[3] = P.a[1];
    P.b[0] = b1 + r * bns;
    P.b[1] = b2 + r * bns;
    P.b[2] = P.b[0];
    P.b[3] = P.b[1];
    P.c[0] = c1 + k * cms;
    P.c[1] = c2 + k * cms;
    P.c[2] = P.c[0];
    P.c[3] = P.c[1];
    return P;
  };

  double acc[4][C::RB][2];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb) acc[c][rb][0] = acc[c][rb][1] = 0.0;

#pragma unroll
  for (int st = 0; st < C::STAGES - 1; ++st) {
    if (st < ktiles) {
      int kk;
      const PairArgs P = stage_args(st, &kk);
      load_stage<C, true>(smem + st * C::STAGE_ELEMS, P, kk, row0, col0, m, n, s, s);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    const int nk = kt + C::STAGES - 1;
    if (nk < ktiles) {
      int kk;
      const PairArgs P = stage_args(nk, &kk);
      load_stage<C, true>(smem + (nk % C::STAGES) * C::STAGE_ELEMS, P, kk, row0, col0, m, n, s, s);
    }
    cp_async_commit();
    const double2* sa = smem + (kt % C::STAGES) * C::STAGE_ELEMS;
    mma_stage_naive<C>(sa, sa + 4 * C::A_PLANE, acc, wm, wn, g, q);
  }
  cp_async_wait<0>();
  int kk;
  const PairArgs P = stage_args(0, &kk);
  store_tile<C, true>(P, acc, row0, col0, m, s, s, wm, wn, g, q);
}

template <class C>
cudaError_t launch_naive_cfg(const double2* a1, const double2* a2, const double2* b1, const double2* b2, double2* c1,
                             double2* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, cudaStream_t stream) {
  static std::mutex mu;
  static uint64_t done = 0;
  const cudaError_t attr = once_per_device(mu, done, [] {
    return cudaFuncSetAttribute(naive_tprod_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)C::SMEM_BYTES);
  });
  if (attr != cudaSuccess) return attr;
  const uint64_t tiles = ((m + C::BM - 1) / C::BM) * ((s + C::BN - 1) / C::BN);
  if (tiles > 0x7fffffffULL) return cudaErrorInvalidConfiguration;
  for (uint64_t k0 = 0; k0 < p; k0 += 65535) {
    const unsigned chunk = (unsigned)std::min<uint64_t>(65535, p - k0);
    naive_tprod_kernel<C><<<dim3((unsigned)tiles, chunk), C::NTHREADS, C::SMEM_BYTES, stream>>>(
        a1, a2, b1, b2, c1, c2, (int)m, (int)n, (int)s, (int)p, (int)k0);
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_naive_tprod(const double2* a1, const double2* a2, const double2* b1, const double2* b2,
                               double2* c1, double2* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                               cudaStream_t stream) {
  if (m == 0 || s == 0 || p == 0) return cudaSuccess;
  if (m <= 32 && s <= 32) return launch_naive_cfg<SmallCfg>(a1, a2, b1, b2, c1, c2, m, n, s, p, stream);
  return launch_naive_cfg<BigCfg>(a1, a2, b1, b2, c1, c2, m, n, s, p, stream);
}

}  // namespace qtb
