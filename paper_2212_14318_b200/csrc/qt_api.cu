// qt_api.cu — the C-ABI (include/qtensor_b200.h): argument checking with the
// reference's error semantics, stream-ordered workspace, the three-stage
// pipeline K1 -> K2 -> K3, the host-buffer path and launch accounting.
//
// Pipeline of one T-product (tproduct.cpp:75-106 restated for the device):
//   K1  tube FFT of A and B in ONE launch (4 jobs: A.t1 conj-in, A.t2 negate,
//       B.t1 conj-in, B.t2 negate)                        -> Â, B̂ (workspace)
//   K2  paired-frequency DMMA GEMM                         -> Ĉ (written into C)
//   K3  inverse tube FFT of Ĉ in place in C (2 jobs)        -> C
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/qtensor_b200.h"
#include "qt_internal.cuh"

namespace qtb {

namespace {
thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) return fail(QT_ENOMEM, "%s: %s", where, cudaGetErrorString(e));
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver || e == cudaErrorNoKernelImageForDevice)
    return fail(QT_ENODEV, "%s: %s", where, cudaGetErrorString(e));
  return fail(QT_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

// current device, checked to be an sm_100 part (the kernels are sm_100a only)
int current_device(int* dev) {
  cudaError_t e = cudaGetDevice(dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, *dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, *dev);
  if (major != 10 || minor != 0)
    return fail(QT_ENODEV, "device %d is sm_%d%d; this library is built for sm_100a only", *dev, major, minor);
  return QT_OK;
}

constexpr uint64_t kIntMax = 0x7fffffffULL;

int check_dims(uint64_t m, uint64_t n, uint64_t s, uint64_t p, const char* who) {
  if (p == 0) return fail(QT_EINVAL, "%s: p must be >= 1", who);  // transform.cpp:152
  if (m > kIntMax || n > kIntMax || s > kIntMax || p > kIntMax)
    return fail(QT_EINVAL, "%s: dimension exceeds 2^31-1", who);
  return QT_OK;
}

TubeJob job(const double* in, double* out, uint64_t ntubes, int conj_in, int conj_out, double scale) {
  TubeJob j;
  j.in = reinterpret_cast<const double2*>(in);
  j.out = reinterpret_cast<double2*>(out);
  j.ntubes = ntubes;
  j.conj_in = conj_in;
  j.conj_out = conj_out;
  j.scale = scale;
  return j;
}

// Forward jobs of qfft3_conj (transform.cpp:155-156).
void add_forward(TubeBatch& b, const double* x1, const double* x2, double* y1, double* y2, uint64_t ntubes) {
  b.job[b.njobs++] = job(x1, y1, ntubes, 1, 0, 1.0);   // ConjInForward
  b.job[b.njobs++] = job(x2, y2, ntubes, 0, 0, -1.0);  // NegateForward
}

// Inverse jobs of qifft3_conj (transform.cpp:164-165).
void add_inverse(TubeBatch& b, const double* x1, const double* x2, double* y1, double* y2, uint64_t ntubes,
                 uint64_t p) {
  const double ip = 1.0 / (double)p;
  b.job[b.njobs++] = job(x1, y1, ntubes, 1, 0, ip);   // InverseConjOut: F(conj x)/p
  b.job[b.njobs++] = job(x2, y2, ntubes, 1, 1, -ip);  // NegateInverse: -conj(F(conj x))/p
}

int tprod_device_impl(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                      double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, cudaStream_t st) {
  int rc = check_dims(m, n, s, p, "tprod_fast");
  if (rc) return rc;
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  if (m == 0 || s == 0) return QT_OK;  // empty result
  cudaError_t e;
  const uint64_t cbytes = m * s * p * sizeof(double2);
  if (n == 0) {  // reference: chat stays zero, qifft3_conj(0) = 0
    if ((e = cudaMemsetAsync(c1, 0, cbytes, st)) != cudaSuccess) return cuda_fail(e, "memset");
    if ((e = cudaMemsetAsync(c2, 0, cbytes, st)) != cudaSuccess) return cuda_fail(e, "memset");
    return QT_OK;
  }
  const uint64_t an = m * n * p, bn = n * s * p;  // complex counts per plane
  double2* ws = nullptr;
  if ((e = cudaMallocAsync(&ws, (2 * an + 2 * bn) * sizeof(double2), st)) != cudaSuccess)
    return cuda_fail(e, "cudaMallocAsync(workspace)");
  double2* ah1 = ws;
  double2* ah2 = ah1 + an;
  double2* bh1 = ah2 + an;
  double2* bh2 = bh1 + bn;

  TubeBatch fwd{};
  add_forward(fwd, a1, a2, (double*)ah1, (double*)ah2, m * n);
  add_forward(fwd, b1, b2, (double*)bh1, (double*)bh2, n * s);
  if ((e = launch_tube_fft(fwd, (int)p, st, dev)) != cudaSuccess) {
    cudaFreeAsync(ws, st);
    return cuda_fail(e, "K1 tube FFT");
  }
  if ((e = launch_spectral_gemm(ah1, ah2, bh1, bh2, (double2*)c1, (double2*)c2, m, n, s, p, st)) != cudaSuccess) {
    cudaFreeAsync(ws, st);
    return cuda_fail(e, "K2 paired spectral GEMM");
  }
  TubeBatch inv{};
  add_inverse(inv, c1, c2, c1, c2, m * s, p);
  if ((e = launch_tube_fft(inv, (int)p, st, dev)) != cudaSuccess) {
    cudaFreeAsync(ws, st);
    return cuda_fail(e, "K3 inverse tube FFT");
  }
  if ((e = cudaFreeAsync(ws, st)) != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return QT_OK;
}

int transform_device_impl(bool inverse, const double* x1, const double* x2, double* y1, double* y2, uint64_t m,
                          uint64_t n, uint64_t p, cudaStream_t st) {
  const char* who = inverse ? "qifft3_conj" : "qfft3_conj";
  int rc = check_dims(m, n, 1, p, who);
  if (rc) return rc;
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  if (m * n == 0) return QT_OK;
  TubeBatch b{};
  if (inverse) add_inverse(b, x1, x2, y1, y2, m * n, p);
  else add_forward(b, x1, x2, y1, y2, m * n);
  cudaError_t e = launch_tube_fft(b, (int)p, st, dev);
  if (e != cudaSuccess) return cuda_fail(e, who);
  return QT_OK;
}

// RAII device buffer + stream for the host-buffer entry points.
struct HostCall {
  cudaStream_t st = nullptr;
  int prev = -1;
  ~HostCall() {
    if (st) cudaStreamDestroy(st);
    if (prev >= 0) cudaSetDevice(prev);
  }
  int begin(int device) {
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) { prev = -1; return cuda_fail(e, "cudaGetDevice"); }
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
    return QT_OK;
  }
};

int h2d(void* d, const void* h, size_t bytes, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "H2D copy");
}
int d2h(void* h, const void* d, size_t bytes, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "D2H copy");
}

}  // namespace

void count_launches(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

}  // namespace qtb

using namespace qtb;

extern "C" {

int qt_abi_version(void) { return QT_B200_ABI_VERSION; }

const char* qt_last_error(void) { return t_err.c_str(); }

uint64_t qt_kernel_launches(void) { return g_launches.load(); }

int qt_tprod_f64_device(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                        double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, void* stream) {
  t_err.clear();
  return tprod_device_impl(a1, a2, b1, b2, c1, c2, m, n, s, p, (cudaStream_t)stream);
}

int qt_qfft3_conj_f64_device(const double* x1, const double* x2, double* y1, double* y2, uint64_t m, uint64_t n,
                             uint64_t p, void* stream) {
  t_err.clear();
  return transform_device_impl(false, x1, x2, y1, y2, m, n, p, (cudaStream_t)stream);
}

int qt_qifft3_conj_f64_device(const double* x1, const double* x2, double* y1, double* y2, uint64_t m, uint64_t n,
                              uint64_t p, void* stream) {
  t_err.clear();
  return transform_device_impl(true, x1, x2, y1, y2, m, n, p, (cudaStream_t)stream);
}

int qt_spectral_product_f64_device(const double* ah1, const double* ah2, const double* bh1, const double* bh2,
                                   double* ch1, double* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                   void* stream) {
  t_err.clear();
  int rc = check_dims(m, n, s, p, "spectral_product");
  if (rc) return rc;
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  cudaError_t e = launch_spectral_gemm((const double2*)ah1, (const double2*)ah2, (const double2*)bh1,
                                       (const double2*)bh2, (double2*)ch1, (double2*)ch2, m, n, s, p,
                                       (cudaStream_t)stream);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "K2 paired spectral GEMM");
}

int qt_tprod_f64_host(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                      double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, int device) {
  t_err.clear();
  int rc = check_dims(m, n, s, p, "tprod_fast");
  if (rc) return rc;
  HostCall hc;
  if ((rc = hc.begin(device))) return rc;
  const size_t ab = m * n * p * sizeof(double2), bb = n * s * p * sizeof(double2), cb = m * s * p * sizeof(double2);
  double* d = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&d, 2 * (ab + bb + cb) + 64, hc.st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(host call)");
  char* base = (char*)d;
  double* da1 = (double*)base;
  double* da2 = (double*)(base + ab);
  double* db1 = (double*)(base + 2 * ab);
  double* db2 = (double*)(base + 2 * ab + bb);
  double* dc1 = (double*)(base + 2 * ab + 2 * bb);
  double* dc2 = (double*)(base + 2 * ab + 2 * bb + cb);
  rc = QT_OK;
  if (!rc && ab) rc = h2d(da1, a1, ab, hc.st);
  if (!rc && ab) rc = h2d(da2, a2, ab, hc.st);
  if (!rc && bb) rc = h2d(db1, b1, bb, hc.st);
  if (!rc && bb) rc = h2d(db2, b2, bb, hc.st);
  if (!rc) rc = tprod_device_impl(da1, da2, db1, db2, dc1, dc2, m, n, s, p, hc.st);
  if (!rc && cb) rc = d2h(c1, dc1, cb, hc.st);
  if (!rc && cb) rc = d2h(c2, dc2, cb, hc.st);
  cudaFreeAsync(d, hc.st);
  e = cudaStreamSynchronize(hc.st);
  if (!rc && e != cudaSuccess) rc = cuda_fail(e, "tprod_fast (host) sync");
  return rc;
}

static int transform_host(bool inverse, const double* x1, const double* x2, double* y1, double* y2, uint64_t m,
                          uint64_t n, uint64_t p, int device) {
  t_err.clear();
  int rc = check_dims(m, n, 1, p, inverse ? "qifft3_conj" : "qfft3_conj");
  if (rc) return rc;
  HostCall hc;
  if ((rc = hc.begin(device))) return rc;
  const size_t xb = m * n * p * sizeof(double2);
  if (xb == 0) return QT_OK;
  double* d = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&d, 2 * xb, hc.st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(host call)");
  double* d1 = d;
  double* d2 = (double*)((char*)d + xb);
  rc = h2d(d1, x1, xb, hc.st);
  if (!rc) rc = h2d(d2, x2, xb, hc.st);
  if (!rc) rc = transform_device_impl(inverse, d1, d2, d1, d2, m, n, p, hc.st);
  if (!rc) rc = d2h(y1, d1, xb, hc.st);
  if (!rc) rc = d2h(y2, d2, xb, hc.st);
  cudaFreeAsync(d, hc.st);
  e = cudaStreamSynchronize(hc.st);
  if (!rc && e != cudaSuccess) rc = cuda_fail(e, "transform (host) sync");
  return rc;
}

int qt_qfft3_conj_f64_host(const double* x1, const double* x2, double* y1, double* y2, uint64_t m, uint64_t n,
                           uint64_t p, int device) {
  return transform_host(false, x1, x2, y1, y2, m, n, p, device);
}

int qt_qifft3_conj_f64_host(const double* x1, const double* x2, double* y1, double* y2, uint64_t m, uint64_t n,
                            uint64_t p, int device) {
  return transform_host(true, x1, x2, y1, y2, m, n, p, device);
}

}  // extern "C"
