// qt_fft_reg.cuh — complex arithmetic and register DFT butterflies shared by
// the tube-FFT kernels (qt_fft.cu) and the one-launch small-product kernel
// (qt_small.cu).  Both must evaluate a tube with the same operations in the
// same order, so the results of the two paths are bitwise identical.
#pragma once

#include <cuda_runtime.h>

namespace qtb {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }  // a * (-i)

template <int R>
__device__ __forceinline__ void dft_reg(double2 (&v)[R]);

template <>
__device__ __forceinline__ void dft_reg<2>(double2 (&v)[2]) {
  double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft_reg<4>(double2 (&v)[4]) {
  double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
  double2 t2 = cadd(v[1], v[3]), t3 = cmul_mi(csub(v[1], v[3]));
  v[0] = cadd(t0, t2);
  v[2] = csub(t0, t2);
  v[1] = cadd(t1, t3);
  v[3] = csub(t1, t3);
}

template <>
__device__ __forceinline__ void dft_reg<8>(double2 (&v)[8]) {
  const double c = 0.70710678118654752440084436210484903928;  // 1/sqrt(2)
  double2 e[4] = {v[0], v[2], v[4], v[6]};
  double2 o[4] = {v[1], v[3], v[5], v[7]};
  dft_reg<4>(e);
  dft_reg<4>(o);
  // o[k] *= W8^k
  double2 o1 = make_double2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));
  double2 o2 = cmul_mi(o[2]);
  double2 o3 = make_double2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}

}  // namespace qtb
