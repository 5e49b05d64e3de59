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

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
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
  // Keep freed workspace in the device's stream-ordered pool across syncs: the
  // default release threshold (0) would unmap it at every synchronize and make
  // the next call pay for fresh page mappings.
  static std::mutex mu;
  static bool pool_set[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (*dev >= 0 && *dev < 64 && !pool_set[*dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, *dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_set[*dev] = true;
  }
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
    int dev = 0;
    int rc = current_device(&dev);
    if (rc) return rc;
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

// Row-slab pipelined host path.  Row i of C depends only on row i of A, so A
// and C stream through the GPU in slabs of R rows while B is uploaded and
// transformed once: two slab streams alternate so that the H2D copy of slab
// j+1 and the D2H copy of slab j-1 (separate copy engines) overlap the
// K1 -> K2 -> K3 compute of slab j.  Output is bitwise identical to the
// one-shot path (same kernels, same per-row arithmetic).
static int tprod_host_pipelined(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                                double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, uint64_t R,
                                HostCall& hc) {
  const size_t cx = sizeof(double2);
  const size_t bb = n * s * p * cx, slab_a = R * n * p * cx, slab_c = R * s * p * cx;
  cudaError_t e;
  int dev = 0;
  int rc = current_device(&dev);
  if (rc) return rc;
  cudaStream_t ss[2] = {nullptr, nullptr};
  cudaEvent_t evB = nullptr;
  char* d = nullptr;
  const size_t total = 4 * bb + 2 * (4 * slab_a + 2 * slab_c) + 256;
  auto cleanup = [&](int code) {
    for (auto& x : ss)
      if (x) { cudaStreamSynchronize(x); cudaStreamDestroy(x); }
    if (d) cudaFreeAsync(d, hc.st);
    if (evB) cudaEventDestroy(evB);
    cudaError_t se = cudaStreamSynchronize(hc.st);
    if (!code && se != cudaSuccess) return cuda_fail(se, "tprod_fast (host) sync");
    return code;
  };
  for (auto& x : ss)
    if ((e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking)) != cudaSuccess) return cleanup(cuda_fail(e, "stream"));
  if ((e = cudaEventCreateWithFlags(&evB, cudaEventDisableTiming)) != cudaSuccess) return cleanup(cuda_fail(e, "event"));
  if ((e = cudaMallocAsync((void**)&d, total, hc.st)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaMallocAsync(host call)"));
  double* dB1 = (double*)d;
  double* dB2 = (double*)(d + bb);
  double* dBh1 = (double*)(d + 2 * bb);
  double* dBh2 = (double*)(d + 3 * bb);
  char* slabs = d + 4 * bb;
  // B: upload + K1(B) once on the call stream
  if ((rc = h2d(dB1, b1, bb, hc.st)) || (rc = h2d(dB2, b2, bb, hc.st))) return cleanup(rc);
  {
    TubeBatch fb{};
    add_forward(fb, dB1, dB2, dBh1, dBh2, n * s);
    if ((e = launch_tube_fft(fb, (int)p, hc.st, dev)) != cudaSuccess) return cleanup(cuda_fail(e, "K1 tube FFT (B)"));
  }
  if ((e = cudaEventRecord(evB, hc.st)) != cudaSuccess) return cleanup(cuda_fail(e, "event"));
  for (auto& x : ss)
    if ((e = cudaStreamWaitEvent(x, evB, 0)) != cudaSuccess) return cleanup(cuda_fail(e, "wait"));

  for (uint64_t r0 = 0, j = 0; r0 < m; r0 += R, ++j) {
    const uint64_t rows = std::min<uint64_t>(R, m - r0);
    cudaStream_t st = ss[j & 1];
    char* base = slabs + (j & 1) * (4 * slab_a + 2 * slab_c);
    double* dA1 = (double*)base;
    double* dA2 = (double*)(base + slab_a);
    double* dAh1 = (double*)(base + 2 * slab_a);
    double* dAh2 = (double*)(base + 3 * slab_a);
    double* dC1 = (double*)(base + 4 * slab_a);
    double* dC2 = (double*)(base + 4 * slab_a + slab_c);
    // slab of A = p strided chunks of rows x n complex (slice-major)
    const size_t apitch = m * n * cx, awidth = rows * n * cx;
    if ((e = cudaMemcpy2DAsync(dA1, awidth, a1 + 2 * r0 * n, apitch, awidth, p, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpy2DAsync(dA2, awidth, a2 + 2 * r0 * n, apitch, awidth, p, cudaMemcpyHostToDevice, st)))
      return cleanup(cuda_fail(e, "H2D A slab"));
    TubeBatch fa{};
    add_forward(fa, dA1, dA2, dAh1, dAh2, rows * n);
    if ((e = launch_tube_fft(fa, (int)p, st, dev)) != cudaSuccess) return cleanup(cuda_fail(e, "K1 tube FFT (A)"));
    if ((e = launch_spectral_gemm((const double2*)dAh1, (const double2*)dAh2, (const double2*)dBh1,
                                  (const double2*)dBh2, (double2*)dC1, (double2*)dC2, rows, n, s, p, st)) !=
        cudaSuccess)
      return cleanup(cuda_fail(e, "K2 paired spectral GEMM"));
    TubeBatch ic{};
    add_inverse(ic, dC1, dC2, dC1, dC2, rows * s, p);
    if ((e = launch_tube_fft(ic, (int)p, st, dev)) != cudaSuccess) return cleanup(cuda_fail(e, "K3 inverse tube FFT"));
    const size_t cpitch = m * s * cx, cwidth = rows * s * cx;
    if ((e = cudaMemcpy2DAsync(c1 + 2 * r0 * s, cpitch, dC1, cwidth, cwidth, p, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemcpy2DAsync(c2 + 2 * r0 * s, cpitch, dC2, cwidth, cwidth, p, cudaMemcpyDeviceToHost, st)))
      return cleanup(cuda_fail(e, "D2H C slab"));
  }
  // the call stream frees the buffers only after both slab streams are done
  cudaEvent_t done[2] = {nullptr, nullptr};
  for (int k = 0; k < 2; ++k) {
    cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
    cudaEventRecord(done[k], ss[k]);
    cudaStreamWaitEvent(hc.st, done[k], 0);
  }
  rc = cleanup(QT_OK);
  for (auto& ev : done) cudaEventDestroy(ev);
  return rc;
}

int qt_tprod_f64_host(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                      double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, int device) {
  t_err.clear();
  int rc = check_dims(m, n, s, p, "tprod_fast");
  if (rc) return rc;
  HostCall hc;
  if ((rc = hc.begin(device))) return rc;
  const size_t ab = m * n * p * sizeof(double2), bb = n * s * p * sizeof(double2), cb = m * s * p * sizeof(double2);
  // Large problems stream row slabs (>= 4 slabs of >= 64 rows, <= ~256 MB of A each).
  if (n > 0 && s > 0 && m >= 256 && ab + cb >= (64ull << 20)) {
    uint64_t R = std::max<uint64_t>(64, (m + 7) / 8);
    const uint64_t row_bytes = n * p * sizeof(double2) * 2;
    while (R > 64 && R * row_bytes > (256ull << 20)) R = (R + 1) / 2;
    R = (R + 63) / 64 * 64;
    return tprod_host_pipelined(a1, a2, b1, b2, c1, c2, m, n, s, p, R, hc);
  }
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
