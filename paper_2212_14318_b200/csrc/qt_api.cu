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
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

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
  // Per-device one-time checks, cached: (1) sm_100 only; (2) keep freed
  // workspace in the device's stream-ordered pool across syncs — the default
  // release threshold (0) would unmap it at every synchronize and make the next
  // call pay for fresh page mappings.
  static std::mutex mu;
  static int state[64] = {};  // 0 unchecked, 1 ok, 2 wrong arch
  static int arch[64] = {};
  const int d = *dev;
  if (d >= 0 && d < 64) {
    std::lock_guard<std::mutex> lk(mu);
    if (state[d] == 0) {
      int major = 0, minor = 0;
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, d);
      arch[d] = major * 10 + minor;
      state[d] = (major == 10 && minor == 0) ? 1 : 2;
      if (state[d] == 1) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
          uint64_t thr = UINT64_MAX;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
      }
    }
    if (state[d] == 2)
      return fail(QT_ENODEV, "device %d is sm_%d; this library is built for sm_100a only", d, arch[d]);
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
  if (small_fused_eligible(m, n, s, p)) {  // one launch: K1, K2, K3 in one cluster kernel (qt_small.cu)
    if ((e = launch_small_tprod((const double2*)a1, (const double2*)a2, (const double2*)b1, (const double2*)b2,
                                (double2*)c1, (double2*)c2, m, n, s, p, st, dev)) != cudaSuccess)
      return cuda_fail(e, "one-launch small T-product");
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

// Per-thread, per-device non-blocking stream for the host-buffer entry
// points (created once: stream creation costs more than a small T-product).
cudaStream_t thread_stream(int device) {
  thread_local cudaStream_t streams[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  if (!streams[device]) cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking);
  return streams[device];
}

// Device switch + stream for the host-buffer entry points (restores the
// caller's device on exit).
struct HostCall {
  cudaStream_t st = nullptr;
  int prev = -1;
  ~HostCall() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  int begin(int device) {
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) { prev = -1; return cuda_fail(e, "cudaGetDevice"); }
    if (device != prev && (e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    int dev = 0;
    int rc = current_device(&dev);
    if (rc) return rc;
    st = thread_stream(dev);
    if (!st) return fail(QT_ECUDA, "cannot create a stream on device %d", dev);
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

namespace {
// set while a stream capture records a small product's launches into a graph:
// those launches are counted when the graph runs, not when it is recorded
thread_local uint64_t* t_capture_count = nullptr;
}  // namespace

void count_launches(uint64_t k) {
  if (t_capture_count) {
    *t_capture_count += k;
    return;
  }
  g_launches.fetch_add(k, std::memory_order_relaxed);
}

namespace {
std::atomic<bool> g_prof{false};
std::mutex g_prof_mu;
std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> g_prof_ev;
// timeline mode (qt_prof_enable(2)): every scope also kept in launch order
struct TlRec {
  const char* tag;
  cudaStream_t st;
  cudaEvent_t e0, e1;
};
std::atomic<bool> g_tl{false};
std::vector<TlRec> g_tl_rec;
cudaEvent_t g_tl_base = nullptr;
}  // namespace

bool prof_on() { return g_prof.load(std::memory_order_relaxed); }

ProfScope::ProfScope(const char* t, cudaStream_t s) : tag(t), st(s) {
  if (prof_on() && cudaEventCreate(&e0) == cudaSuccess) {
    cudaEventRecord(e0, st);
    if (g_tl.load(std::memory_order_relaxed) && cudaEventCreate(&t0) == cudaSuccess) cudaEventRecord(t0, st);
  }
}

void ProfScope::stop() {
  if (!e0) return;
  cudaEvent_t e1 = nullptr;
  if (cudaEventCreate(&e1) != cudaSuccess) return;
  cudaEventRecord(e1, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_ev[tag].emplace_back(e0, e1);
  if (t0) {
    cudaEvent_t t1 = nullptr;
    if (cudaEventCreate(&t1) == cudaSuccess) {
      cudaEventRecord(t1, st);
      g_tl_rec.push_back(TlRec{tag, st, t0, t1});
    } else {
      cudaEventDestroy(t0);
    }
    t0 = nullptr;
  }
  e0 = nullptr;
}

}  // namespace qtb

using namespace qtb;

extern "C" {

int qt_abi_version(void) { return QT_B200_ABI_VERSION; }

const char* qt_last_error(void) { return t_err.c_str(); }

uint64_t qt_kernel_launches(void) { return g_launches.load(); }

void qt_prof_enable(int on) {
  if (on == 2) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaDeviceSynchronize();
    if (!g_tl_base) cudaEventCreate(&g_tl_base);
    cudaEventRecord(g_tl_base, 0);
    g_tl.store(true);
  } else if (!on) {
    g_tl.store(false);
  }
  g_prof.store(on != 0);
}

int qt_prof_timeline(char* buf, uint64_t cap) {
  t_err.clear();
  std::vector<TlRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    recs.swap(g_tl_rec);
  }
  std::string out;
  int rc = QT_OK;
  for (auto& r : recs) {
    float a = 0.f, b = 0.f;
    cudaError_t e = cudaEventSynchronize(r.e1);
    if (e == cudaSuccess && g_tl_base) e = cudaEventElapsedTime(&a, g_tl_base, r.e0);
    if (e == cudaSuccess && g_tl_base) e = cudaEventElapsedTime(&b, g_tl_base, r.e1);
    if (e != cudaSuccess && rc == QT_OK) rc = cuda_fail(e, "qt_prof_timeline");
    char line[160];
    snprintf(line, sizeof line, "%s %p %.4f %.4f\n", r.tag, (void*)r.st, a, b);
    out += line;
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  if (buf && cap) {
    const size_t k = std::min<size_t>(out.size(), cap - 1);
    memcpy(buf, out.data(), k);
    buf[k] = 0;
  }
  return rc != QT_OK ? -rc : (int)out.size();
}

int qt_prof_read(const char* tag, double* ms, uint64_t* launches) {
  t_err.clear();
  if (!tag || !ms || !launches) return fail(QT_EINVAL, "qt_prof_read: null argument");
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    auto it = g_prof_ev.find(tag);
    if (it != g_prof_ev.end()) evs.swap(it->second);
  }
  double total = 0.0;
  int rc = QT_OK;
  for (auto& [a, b] : evs) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, a, b);
    if (e != cudaSuccess && rc == QT_OK) rc = cuda_fail(e, "qt_prof_read");
    total += t;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  *ms = total;
  *launches = evs.size();
  return rc;
}

// ----------------------------------------------- CUDA graphs for small products
// A small product (<= 256 MB, fp64 DMMA stage 2, one- or two-pass tube FFTs) is three to five
// short launches whose launch gaps rival their run time.  The device entry
// point records such a call once into a CUDA graph (stream capture on a
// private stream, after one ordinary run that also creates the twiddle tables)
// keyed by (device, the six pointers, m, n, s, p) and replays it on the
// caller's stream afterwards: the same kernels with the same arguments, so the
// results are bitwise the same.  QTB_GRAPH=0 disables it; profiling
// (qt_prof_enable) bypasses it.
namespace {
struct GraphKey {
  int dev;
  uintptr_t ptr[6];
  uint64_t m, n, s, p;
  bool operator<(const GraphKey& o) const {
    return std::tie(dev, ptr[0], ptr[1], ptr[2], ptr[3], ptr[4], ptr[5], m, n, s, p) <
           std::tie(o.dev, o.ptr[0], o.ptr[1], o.ptr[2], o.ptr[3], o.ptr[4], o.ptr[5], o.m, o.n, o.s, o.p);
  }
};
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;  // null: capture failed, run directly
  uint64_t kernels = 0;
};
std::mutex g_graph_mu;
std::map<GraphKey, GraphEntry> g_graphs;
constexpr size_t kMaxGraphs = 64;

bool graph_eligible(uint64_t m, uint64_t n, uint64_t s, uint64_t p) {
  static const bool on = [] {
    const char* v = getenv("QTB_GRAPH");
    return !(v && *v == '0');
  }();
  if (!on || prof_on() || m == 0 || n == 0 || s == 0 || p == 0 || p > kIntMax) return false;
  if ((m * n + n * s + m * s) * p * 32 > (256ull << 20)) return false;
  // the int8 stage 2 forks streams of its own; the one-launch-per-stage path
  // for long prime lengths is left out as well
  return choose_gemm_algo(n, s, p) == kAlgoDmma && (fft_single_pass((int)p) || fft_split_length((int)p));
}

cudaStream_t capture_stream(int device) {
  thread_local cudaStream_t streams[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  if (!streams[device]) cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking);
  return streams[device];
}
}  // namespace

int qt_tprod_f64_device(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                        double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, void* stream) {
  t_err.clear();
  cudaStream_t st = (cudaStream_t)stream;
  if (check_dims(m, n, s, p, "tprod_fast") != QT_OK || !graph_eligible(m, n, s, p)) {
    t_err.clear();
    return tprod_device_impl(a1, a2, b1, b2, c1, c2, m, n, s, p, st);
  }
  int dev = 0;
  int rc = current_device(&dev);
  if (rc) return rc;
  const GraphKey key{dev, {(uintptr_t)a1, (uintptr_t)a2, (uintptr_t)b1, (uintptr_t)b2, (uintptr_t)c1, (uintptr_t)c2},
                     m, n, s, p};
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = g_graphs.find(key);
    if (it != g_graphs.end()) {
      if (!it->second.exec) return tprod_device_impl(a1, a2, b1, b2, c1, c2, m, n, s, p, st);
      const cudaError_t e = cudaGraphLaunch(it->second.exec, st);
      if (e != cudaSuccess) return cuda_fail(e, "tprod_fast (graph launch)");
      count_launches(it->second.kernels);
      return QT_OK;
    }
  }
  // first call with this key: run it, then record it for the next ones
  if ((rc = tprod_device_impl(a1, a2, b1, b2, c1, c2, m, n, s, p, st)) != QT_OK) return rc;
  GraphEntry ent;
  cudaStream_t cs = capture_stream(dev);
  if (cs && cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    t_capture_count = &ent.kernels;
    const int crc = tprod_device_impl(a1, a2, b1, b2, c1, c2, m, n, s, p, cs);
    t_capture_count = nullptr;
    cudaGraph_t g = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(cs, &g);
    if (crc == QT_OK && ee == cudaSuccess && g && cudaGraphInstantiate(&ent.exec, g, 0) != cudaSuccess)
      ent.exec = nullptr;
    if (g) cudaGraphDestroy(g);
    if (!ent.exec) ent.kernels = 0;
  }
  (void)cudaGetLastError();  // a failed capture leaves nothing behind: that key runs directly
  t_err.clear();
  std::lock_guard<std::mutex> lk(g_graph_mu);
  if (g_graphs.size() >= kMaxGraphs) {
    for (auto& kv : g_graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    g_graphs.clear();
  }
  auto ins = g_graphs.emplace(key, ent);
  if (!ins.second && ent.exec) cudaGraphExecDestroy(ent.exec);  // another thread recorded it first
  return QT_OK;
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

int qt_fft_routable(uint64_t p) { return p >= 1 && p <= (uint64_t)kIntMax && fft_single_pass((int)p) ? 1 : 0; }

int qt_qfft3_conj_f64_device_routed(const double* x1, const double* x2, double* const* y1_rows,
                                    double* const* y2_rows, uint64_t m, uint64_t n, uint64_t p, void* stream) {
  t_err.clear();
  int rc = check_dims(m, n, 1, p, "qfft3_conj (routed)");
  if (rc) return rc;
  if (!qt_fft_routable(p)) return fail(QT_EINVAL, "qfft3_conj (routed): this length is transformed in two passes");
  if (!y1_rows || !y2_rows) return fail(QT_EINVAL, "qfft3_conj (routed): null row table");
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  if (m * n == 0) return QT_OK;
  TubeBatch b{};
  add_forward(b, x1, x2, nullptr, nullptr, m * n);
  b.job[0].out_rows = reinterpret_cast<double2* const*>(y1_rows);
  b.job[1].out_rows = reinterpret_cast<double2* const*>(y2_rows);
  cudaError_t e = launch_tube_fft(b, (int)p, (cudaStream_t)stream, dev);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "qfft3_conj (routed)");
}

int qt_qfft3_conj_f64_device_routed_n(const double* x1, const double* x2, double* const* y1_rows,
                                      double* const* y2_rows, int ndst, uint64_t m, uint64_t n, uint64_t p,
                                      void* stream) {
  t_err.clear();
  int rc = check_dims(m, n, 1, p, "qfft3_conj (routed, n destinations)");
  if (rc) return rc;
  if (!qt_fft_routable(p)) return fail(QT_EINVAL, "qfft3_conj (routed): this length is transformed in two passes");
  if (!y1_rows || !y2_rows || ndst < 1 || ndst > 64) return fail(QT_EINVAL, "qfft3_conj (routed): bad row tables");
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  if (m * n == 0) return QT_OK;
  TubeBatch b{};
  add_forward(b, x1, x2, nullptr, nullptr, m * n);
  for (int i = 0; i < 2; ++i) {
    b.job[i].out_rows = reinterpret_cast<double2* const*>(i ? y2_rows : y1_rows);
    b.job[i].out_ndst = ndst;
    b.job[i].out_rows_stride = (int)p;
  }
  cudaError_t e = launch_tube_fft(b, (int)p, (cudaStream_t)stream, dev);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "qfft3_conj (routed)");
}

int qt_qifft3_conj_f64_device_routed(const double* const* x1_rows, const double* const* x2_rows, double* y1,
                                     double* y2, uint64_t m, uint64_t n, uint64_t p, void* stream) {
  t_err.clear();
  int rc = check_dims(m, n, 1, p, "qifft3_conj (routed)");
  if (rc) return rc;
  if (!qt_fft_routable(p)) return fail(QT_EINVAL, "qifft3_conj (routed): this length is transformed in two passes");
  if (!x1_rows || !x2_rows) return fail(QT_EINVAL, "qifft3_conj (routed): null row table");
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  if (m * n == 0) return QT_OK;
  TubeBatch b{};
  add_inverse(b, nullptr, nullptr, y1, y2, m * n, p);
  b.job[0].in_rows = reinterpret_cast<const double2* const*>(x1_rows);
  b.job[1].in_rows = reinterpret_cast<const double2* const*>(x2_rows);
  cudaError_t e = launch_tube_fft(b, (int)p, (cudaStream_t)stream, dev);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "qifft3_conj (routed)");
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

// Optional phase tracing of the host pipeline ($QTB_TRACE=1): CUDA events at
// phase boundaries, printed to stderr as milliseconds from the call start.
struct PhaseTrace {
  bool on = false;
  cudaEvent_t t0 = nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  explicit PhaseTrace(cudaStream_t st) {
    const char* env = getenv("QTB_TRACE");
    on = env && *env && *env != '0';
    if (on) {
      cudaEventCreate(&t0);
      cudaEventRecord(t0, st);
    }
  }
  void mark(const std::string& label, cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    marks.emplace_back(label, e);
  }
  void dump() {
    if (!on) return;
    cudaDeviceSynchronize();
    for (auto& [label, e] : marks) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, t0, e);
      fprintf(stderr, "[qtb trace] %8.3f ms  %s\n", ms, label.c_str());
      cudaEventDestroy(e);
    }
    cudaEventDestroy(t0);
  }
};

// ------------------------------------------------- pageable host buffers
// A drop-in caller hands over pageable std::vector storage.  DMA from pageable
// memory goes through the driver's small bounce buffer one strided row at a
// time (config 5: ~1.8 s instead of 0.27 s).  For large calls the inputs are
// therefore first copied into a cached pinned arena by all host cores, the
// pinned tiled pipeline runs, and C is copied back the same way.
bool is_pinned(const void* ptr) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

void parallel_copy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t per = std::max<size_t>(size_t(16) << 20, (bytes + hw - 1) / hw);
  std::vector<std::thread> th;
  for (size_t off = 0; off < bytes; off += per) {
    const size_t len = std::min(per, bytes - off);
    th.emplace_back([=] { std::memcpy((char*)dst + off, (const char*)src + off, len); });
  }
  for (auto& t : th) t.join();
}

struct PinnedArena {
  std::mutex mu;
  void* ptr = nullptr;
  size_t size = 0;
};
PinnedArena& pinned_arena() {
  static PinnedArena a;
  return a;
}

// Tiled streaming host path (large problems).  Row i of C depends only on row
// i of A and column j of C only on column j of B, so C is computed in
// (row slab x column chunk) tiles while A and B stream in over PCIe:
//   copy-in stream : A slab 0, B chunk 0, A slab 1, B chunk 1, ...  (wavefront)
//   compute stream : K1 of each arriving slab/chunk into resident Â / B̂, then
//                    every tile (i, j) whose slab i and chunk j have arrived:
//                    K2 -> K3 into one of three tile buffers
//   copy-out stream: the tile's strided 3-D copy back into host C
// so the GPU starts computing after one slab + one chunk instead of after all
// of B, and the compute stream never waits on a download.  Every tile runs the
// same kernels with the same per-element arithmetic, so the result is bitwise
// identical to the device-resident path.
static int tprod_host_tiled(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                            double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, uint64_t R, uint64_t Q,
                            HostCall& hc) {
  const size_t cx = sizeof(double2);
  const uint64_t NI = (m + R - 1) / R, NJ = (s + Q - 1) / Q;
  const size_t ahat = m * n * p * cx, bhat = n * s * p * cx;       // per plane, resident
  const size_t stA = R * n * p * cx, stB = n * Q * p * cx;        // per plane, staging
  const size_t tile = R * Q * p * cx;                              // per plane, C tile
  cudaError_t e;
  int dev = 0;
  int rc = current_device(&dev);
  if (rc) return rc;
  cudaStream_t sin = nullptr, scomp = nullptr, sout = nullptr;
  std::vector<cudaEvent_t> evs;
  auto mkev = [&]() {
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) evs.push_back(ev);
    return ev;
  };
  char* d = nullptr;
  const size_t total = 2 * ahat + 2 * bhat + 2 * (2 * stA) + 2 * (2 * stB) + 3 * (2 * tile) + 256;
  auto cleanup = [&](int code) {
    for (cudaStream_t x : {sin, scomp, sout})
      if (x) cudaStreamSynchronize(x);
    if (d) cudaFreeAsync(d, hc.st);
    cudaError_t se = cudaStreamSynchronize(hc.st);
    for (cudaStream_t x : {sin, scomp, sout})
      if (x) cudaStreamDestroy(x);
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
    if (!code && se != cudaSuccess) return cuda_fail(se, "tprod_fast (host) sync");
    return code;
  };
  for (cudaStream_t* x : {&sin, &scomp, &sout})
    if ((e = cudaStreamCreateWithFlags(x, cudaStreamNonBlocking)) != cudaSuccess) return cleanup(cuda_fail(e, "stream"));
  if ((e = cudaMallocAsync((void**)&d, total, hc.st)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaMallocAsync(host call)"));
  cudaEvent_t ready = mkev();
  cudaEventRecord(ready, hc.st);  // allocation visible to the worker streams
  for (cudaStream_t x : {sin, scomp, sout}) cudaStreamWaitEvent(x, ready, 0);

  char* cur = d;
  auto take = [&](size_t bytes) { char* r = cur; cur += (bytes + 255) / 256 * 256; return (double*)r; };
  double* Ah1 = take(ahat);
  double* Ah2 = take(ahat);
  double* Bh1 = take(bhat);
  double* Bh2 = take(bhat);
  double* SA[2][2] = {{take(stA), take(stA)}, {take(stA), take(stA)}};
  double* SB[2][2] = {{take(stB), take(stB)}, {take(stB), take(stB)}};
  double* T[3][2] = {{take(tile), take(tile)}, {take(tile), take(tile)}, {take(tile), take(tile)}};
  cudaEvent_t stA_free[2] = {nullptr, nullptr}, stB_free[2] = {nullptr, nullptr};
  cudaEvent_t tile_free[3] = {nullptr, nullptr, nullptr};
  PhaseTrace tr(hc.st);

  auto rows_of = [&](uint64_t i) { return std::min<uint64_t>(R, m - i * R); };
  auto cols_of = [&](uint64_t j) { return std::min<uint64_t>(Q, s - j * Q); };
  // B̂ chunk j is stored as its own contiguous n x cols(j) x p tensor
  auto bh_chunk = [&](double* base, uint64_t j) { return (double*)((char*)base + j * Q * n * p * cx); };
  auto ah_slab = [&](double* base, uint64_t i) { return (double*)((char*)base + i * R * n * p * cx); };

  auto upload_a = [&](uint64_t i) -> int {
    const int b = (int)(i & 1);
    if (stA_free[b]) cudaStreamWaitEvent(sin, stA_free[b], 0);
    const uint64_t rows = rows_of(i);
    const size_t pitch = m * n * cx, width = rows * n * cx;
    if ((e = cudaMemcpy2DAsync(SA[b][0], width, a1 + 2 * i * R * n, pitch, width, p, cudaMemcpyHostToDevice, sin)) ||
        (e = cudaMemcpy2DAsync(SA[b][1], width, a2 + 2 * i * R * n, pitch, width, p, cudaMemcpyHostToDevice, sin)))
      return cuda_fail(e, "H2D A slab");
    cudaEvent_t in = mkev();
    cudaEventRecord(in, sin);
    cudaStreamWaitEvent(scomp, in, 0);
    TubeBatch fb{};
    add_forward(fb, SA[b][0], SA[b][1], ah_slab(Ah1, i), ah_slab(Ah2, i), rows * n);
    if ((e = launch_tube_fft(fb, (int)p, scomp, dev)) != cudaSuccess) return cuda_fail(e, "K1 tube FFT (A)");
    stA_free[b] = mkev();
    cudaEventRecord(stA_free[b], scomp);
    tr.mark("A slab " + std::to_string(i) + " transformed", scomp);
    return QT_OK;
  };
  auto upload_b = [&](uint64_t j) -> int {
    const int b = (int)(j & 1);
    if (stB_free[b]) cudaStreamWaitEvent(sin, stB_free[b], 0);
    const uint64_t cols = cols_of(j);
    // column chunk: p*n rows of `cols` complex at host pitch s (uniform over slices)
    const size_t pitch = s * cx, width = cols * cx;
    if ((e = cudaMemcpy2DAsync(SB[b][0], width, b1 + 2 * j * Q, pitch, width, p * n, cudaMemcpyHostToDevice, sin)) ||
        (e = cudaMemcpy2DAsync(SB[b][1], width, b2 + 2 * j * Q, pitch, width, p * n, cudaMemcpyHostToDevice, sin)))
      return cuda_fail(e, "H2D B chunk");
    cudaEvent_t in = mkev();
    cudaEventRecord(in, sin);
    cudaStreamWaitEvent(scomp, in, 0);
    TubeBatch fb{};
    add_forward(fb, SB[b][0], SB[b][1], bh_chunk(Bh1, j), bh_chunk(Bh2, j), n * cols);
    if ((e = launch_tube_fft(fb, (int)p, scomp, dev)) != cudaSuccess) return cuda_fail(e, "K1 tube FFT (B)");
    stB_free[b] = mkev();
    cudaEventRecord(stB_free[b], scomp);
    tr.mark("B chunk " + std::to_string(j) + " transformed", scomp);
    return QT_OK;
  };
  uint64_t unit = 0;
  const int algo = choose_gemm_algo(n, s, p);  // one algorithm for every tile of the product
  auto compute_tile = [&](uint64_t i, uint64_t j) -> int {
    const int t = (int)(unit % 3);
    ++unit;
    if (tile_free[t]) cudaStreamWaitEvent(scomp, tile_free[t], 0);
    const uint64_t rows = rows_of(i), cols = cols_of(j);
    if ((e = launch_spectral_gemm((const double2*)ah_slab(Ah1, i), (const double2*)ah_slab(Ah2, i),
                                  (const double2*)bh_chunk(Bh1, j), (const double2*)bh_chunk(Bh2, j),
                                  (double2*)T[t][0], (double2*)T[t][1], rows, n, cols, p, scomp, algo)) != cudaSuccess)
      return cuda_fail(e, "K2 paired spectral GEMM");
    TubeBatch ic{};
    add_inverse(ic, T[t][0], T[t][1], T[t][0], T[t][1], rows * cols, p);
    if ((e = launch_tube_fft(ic, (int)p, scomp, dev)) != cudaSuccess) return cuda_fail(e, "K3 inverse tube FFT");
    cudaEvent_t done = mkev();
    cudaEventRecord(done, scomp);
    cudaStreamWaitEvent(sout, done, 0);
    // tile [p][rows][cols] -> host C rows i*R.., cols j*Q.. of every slice
    for (int plane = 0; plane < 2; ++plane) {
      cudaMemcpy3DParms cp{};
      cp.srcPtr = make_cudaPitchedPtr(T[t][plane], cols * cx, cols * cx, rows);
      double* hc_base = plane == 0 ? c1 : c2;
      cp.dstPtr = make_cudaPitchedPtr(hc_base, s * cx, s * cx, m);
      cp.dstPos = make_cudaPos(j * Q * cx, i * R, 0);
      cp.extent = make_cudaExtent(cols * cx, rows, p);
      cp.kind = cudaMemcpyDeviceToHost;
      if ((e = cudaMemcpy3DAsync(&cp, sout)) != cudaSuccess) return cuda_fail(e, "D2H C tile");
    }
    tile_free[t] = mkev();
    cudaEventRecord(tile_free[t], sout);
    return QT_OK;
  };

  // wavefront over shells k: slab k and chunk k arrive, then every new tile
  const uint64_t K = std::max(NI, NJ);
  for (uint64_t k = 0; k < K; ++k) {
    if (k < NI && (rc = upload_a(k))) return cleanup(rc);
    if (k < NJ && (rc = upload_b(k))) return cleanup(rc);
    if (k < NI)
      for (uint64_t j = 0; j < std::min<uint64_t>(k + 1, NJ); ++j)
        if ((rc = compute_tile(k, j))) return cleanup(rc);
    if (k < NJ)
      for (uint64_t i = 0; i < std::min<uint64_t>(k, NI); ++i)
        if ((rc = compute_tile(i, k))) return cleanup(rc);
  }
  tr.mark("all tiles computed", scomp);
  tr.mark("all tiles downloaded", sout);
  // the call stream frees the buffers only after every worker stream is done
  for (cudaStream_t x : {sin, scomp, sout}) {
    cudaEvent_t fin = mkev();
    cudaEventRecord(fin, x);
    cudaStreamWaitEvent(hc.st, fin, 0);
  }
  tr.dump();
  return cleanup(QT_OK);
}

// Host path for products that take the int8 (Ozaki) K2 (qt_ozaki.cu).  Its
// residues of B̂ are the expensive, reusable half, so instead of (row x column)
// tiles it streams ROW SLABS against a resident B':
//   phase 1: B copied in (chunks on the copy-in stream), one K1, B' residues for
//            every frequency (overlapping slab 0's upload);
//   phase 2: per A row slab: copy-in -> K1 -> A' residues + int8 GEMMs + CRT ->
//            K3 -> copy-out of the slab's rows, slabs double-buffered so the
//            copy-in of slab i+1 and the copy-out of slab i-1 run under slab i.
// Every element goes through the same exact integer product as the device
// path, so the result is bitwise identical to it (finite inputs).
static int tprod_host_slabs_ozaki(const double* a1, const double* a2, const double* b1, const double* b2,
                                  double* c1, double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                  uint64_t R, HostCall& hc) {
  const size_t cx = sizeof(double2);
  const uint64_t NI = (m + R - 1) / R;
  const size_t bpl = n * s * p * cx;       // B (and B̂) per plane
  const size_t stA = R * n * p * cx;       // A slab per plane
  const size_t stC = R * s * p * cx;       // C slab per plane
  cudaError_t e;
  int dev = 0;
  int rc = current_device(&dev);
  if (rc) return rc;
  cudaStream_t sin = nullptr, scomp = nullptr, sout = nullptr;
  std::vector<cudaEvent_t> evs;
  auto mkev = [&]() {
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) evs.push_back(ev);
    return ev;
  };
  char* d = nullptr;
  OzakiB B;
  auto a256 = [](size_t x) { return (x + 255) / 256 * 256; };
  // B staging (2 planes) + B̂ (2) + A staging (2 x 2) + Â slab (2 x 2) + C slab (2 x 2) + flag
  const size_t total = 2 * a256(bpl) * 2 + 4 * a256(stA) * 2 + 4 * a256(stC) + a256(int8_flag_ints(p) * sizeof(int));
  auto cleanup = [&](int code) {
    for (cudaStream_t x : {sin, scomp, sout})
      if (x) cudaStreamSynchronize(x);
    if (B.res) ozaki_release(B, hc.st);
    if (d) cudaFreeAsync(d, hc.st);
    cudaError_t se = cudaStreamSynchronize(hc.st);
    for (cudaStream_t x : {sin, scomp, sout})
      if (x) cudaStreamDestroy(x);
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
    if (!code && se != cudaSuccess) return cuda_fail(se, "tprod_fast (host) sync");
    return code;
  };
  for (cudaStream_t* x : {&sin, &scomp, &sout})
    if ((e = cudaStreamCreateWithFlags(x, cudaStreamNonBlocking)) != cudaSuccess) return cleanup(cuda_fail(e, "stream"));
  if ((e = cudaMallocAsync((void**)&d, total, hc.st)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaMallocAsync(host call)"));
  {
    cudaEvent_t ready = mkev();
    cudaEventRecord(ready, hc.st);
    for (cudaStream_t x : {sin, scomp, sout}) cudaStreamWaitEvent(x, ready, 0);
  }
  char* cur = d;
  auto take = [&](size_t bytes) { char* r = cur; cur += a256(bytes); return (double*)r; };
  double* Bs1 = take(bpl);
  double* Bs2 = take(bpl);
  double* Bh1 = take(bpl);
  double* Bh2 = take(bpl);
  double* SA[2][2] = {{take(stA), take(stA)}, {take(stA), take(stA)}};
  double* AH[2][2] = {{take(stA), take(stA)}, {take(stA), take(stA)}};
  double* CS[2][2] = {{take(stC), take(stC)}, {take(stC), take(stC)}};
  int* flag = (int*)take(int8_flag_ints(p) * sizeof(int));
  PhaseTrace tr(hc.st);

  // phase 1: B in ~8 chunks per plane, then K1 and the B' residues
  if ((e = cudaMemsetAsync(flag, 0, int8_flag_ints(p) * sizeof(int), scomp)) != cudaSuccess)
    return cleanup(cuda_fail(e, "memset"));
  const size_t bchunk = std::max<size_t>(size_t(64) << 20, (bpl + 7) / 8);
  for (int plane = 0; plane < 2; ++plane)
    for (size_t off = 0; off < bpl; off += bchunk)
      if ((e = cudaMemcpyAsync((char*)(plane ? Bs2 : Bs1) + off, (const char*)(plane ? b2 : b1) + off,
                               std::min(bchunk, bpl - off), cudaMemcpyHostToDevice, sin)) != cudaSuccess)
        return cleanup(cuda_fail(e, "H2D B"));
  {
    cudaEvent_t in = mkev();
    cudaEventRecord(in, sin);
    cudaStreamWaitEvent(scomp, in, 0);
  }
  tr.mark("B uploaded", sin);
  {
    TubeBatch fb{};
    add_forward(fb, Bs1, Bs2, Bh1, Bh2, n * s);
    if ((e = launch_tube_fft(fb, (int)p, scomp, dev)) != cudaSuccess) return cleanup(cuda_fail(e, "K1 tube FFT (B)"));
  }
  if ((e = ozaki_prepare_b((const double2*)Bh1, (const double2*)Bh2, R, n, s, p, s, n * s, flag, true, &B, scomp)) !=
      cudaSuccess)
    return cleanup(cuda_fail(e, "K2 B residues"));
  tr.mark("B' residues ready", scomp);

  // phase 2: A row slabs.  The last slab is split in two halves (when each
  // keeps >= 128 rows) so the work left after the final upload — its compute
  // and its copy-out — is halved.
  std::vector<std::pair<uint64_t, uint64_t>> slabs;  // (first row, rows)
  for (uint64_t i = 0; i < NI; ++i) {
    const uint64_t r0 = i * R, rows = std::min<uint64_t>(R, m - r0);
    if (i == NI - 1 && NI > 1 && rows >= 256) {
      slabs.emplace_back(r0, rows / 2);
      slabs.emplace_back(r0 + rows / 2, rows - rows / 2);
    } else {
      slabs.emplace_back(r0, rows);
    }
  }
  cudaEvent_t sa_free[2] = {nullptr, nullptr}, cs_free[2] = {nullptr, nullptr};
  for (uint64_t i = 0; i < slabs.size(); ++i) {
    const int b = (int)(i & 1);
    const uint64_t row0 = slabs[i].first, rows = slabs[i].second;
    if (sa_free[b]) cudaStreamWaitEvent(sin, sa_free[b], 0);
    const size_t apitch = m * n * cx, awidth = rows * n * cx;
    if ((e = cudaMemcpy2DAsync(SA[b][0], awidth, a1 + 2 * row0 * n, apitch, awidth, p, cudaMemcpyHostToDevice, sin)) ||
        (e = cudaMemcpy2DAsync(SA[b][1], awidth, a2 + 2 * row0 * n, apitch, awidth, p, cudaMemcpyHostToDevice, sin)))
      return cleanup(cuda_fail(e, "H2D A slab"));
    cudaEvent_t in = mkev();
    cudaEventRecord(in, sin);
    cudaStreamWaitEvent(scomp, in, 0);
    TubeBatch fb{};
    add_forward(fb, SA[b][0], SA[b][1], AH[b][0], AH[b][1], rows * n);
    if ((e = launch_tube_fft(fb, (int)p, scomp, dev)) != cudaSuccess) return cleanup(cuda_fail(e, "K1 tube FFT (A)"));
    sa_free[b] = mkev();
    cudaEventRecord(sa_free[b], scomp);
    if (cs_free[b]) cudaStreamWaitEvent(scomp, cs_free[b], 0);
    const double2 *ah1 = (const double2*)AH[b][0], *ah2 = (const double2*)AH[b][1];
    double2 *cc1 = (double2*)CS[b][0], *cc2 = (double2*)CS[b][1];
    if ((e = ozaki_multiply(B, ah1, ah2, (const double2*)Bh1, (const double2*)Bh2, rows, cc1, cc2, s, rows * s, flag,
                            scomp)) != cudaSuccess)
      return cleanup(cuda_fail(e, "K2 int8 GEMM"));
    // non-finite inputs / pairs the accuracy guard did not certify: the fp64
    // DMMA kernels recompute them (no-op otherwise)
    if ((e = dmma_spectral_gemm(ah1, ah2, (const double2*)Bh1, (const double2*)Bh2, cc1, cc2, rows, n, s, p, s, s,
                                n * s, rows * s, scomp, flag)) != cudaSuccess)
      return cleanup(cuda_fail(e, "K2 fallback"));
    TubeBatch ic{};
    add_inverse(ic, CS[b][0], CS[b][1], CS[b][0], CS[b][1], rows * s, p);
    if ((e = launch_tube_fft(ic, (int)p, scomp, dev)) != cudaSuccess) return cleanup(cuda_fail(e, "K3 inverse tube FFT"));
    cudaEvent_t done = mkev();
    cudaEventRecord(done, scomp);
    cudaStreamWaitEvent(sout, done, 0);
    const size_t cpitch = m * s * cx, cwidth = rows * s * cx;
    if ((e = cudaMemcpy2DAsync(c1 + 2 * row0 * s, cpitch, CS[b][0], cwidth, cwidth, p, cudaMemcpyDeviceToHost, sout)) ||
        (e = cudaMemcpy2DAsync(c2 + 2 * row0 * s, cpitch, CS[b][1], cwidth, cwidth, p, cudaMemcpyDeviceToHost, sout)))
      return cleanup(cuda_fail(e, "D2H C slab"));
    cs_free[b] = mkev();
    cudaEventRecord(cs_free[b], sout);
    tr.mark("slab " + std::to_string(i) + " computed", scomp);
  }
  tr.mark("all slabs downloaded", sout);
  for (cudaStream_t x : {sin, scomp, sout}) {
    cudaEvent_t fin = mkev();
    cudaEventRecord(fin, x);
    cudaStreamWaitEvent(hc.st, fin, 0);
  }
  tr.dump();
  return cleanup(QT_OK);
}

int qt_spectral_product_f64_device_ld_algo(const double* ah1, const double* ah2, const double* bh1,
                                           const double* bh2, double* ch1, double* ch2, uint64_t m, uint64_t n,
                                           uint64_t s, uint64_t p, uint64_t ldb, uint64_t ldc, uint64_t bslice,
                                           uint64_t cslice, int algo, void* stream) {
  t_err.clear();
  int rc = check_dims(m, n, s, p, "spectral_product");
  if (rc) return rc;
  if (ldb < s || ldc < s || bslice < n * ldb || cslice < m * ldc || ldb > kIntMax || ldc > kIntMax)
    return fail(QT_EINVAL, "spectral_product: leading dimensions smaller than the matrices");
  if (algo != QT_GEMM_AUTO && algo != QT_GEMM_DMMA && algo != QT_GEMM_INT8_EXACT)
    return fail(QT_EINVAL, "spectral_product: unknown algorithm");
  if (algo == QT_GEMM_INT8_EXACT && (n % 32 != 0 || n > 8192 || p > 65534))
    return fail(QT_EINVAL, "spectral_product: the int8 path needs n %% 32 == 0, n <= 8192 and p <= 65534");
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  cudaError_t e = launch_spectral_gemm_ld((const double2*)ah1, (const double2*)ah2, (const double2*)bh1,
                                          (const double2*)bh2, (double2*)ch1, (double2*)ch2, m, n, s, p, ldb, ldc,
                                          bslice, cslice, (cudaStream_t)stream, algo);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "K2 paired spectral GEMM");
}

int qt_spectral_product_f64_device_ld(const double* ah1, const double* ah2, const double* bh1, const double* bh2,
                                      double* ch1, double* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                      uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice, void* stream) {
  return qt_spectral_product_f64_device_ld_algo(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice,
                                                QT_GEMM_AUTO, stream);
}

namespace {
struct Int8Slots {
  OzakiB B;
  int* nonfinite = nullptr;
  int* flags = nullptr;  // int8_flag_ints(p): [0] non-finite (sticky), [1 + k] pair k to recompute
  const double2* bh1 = nullptr;
  const double2* bh2 = nullptr;
  int device = 0;
};
}  // namespace

int qt_slot_frequency(uint64_t p, uint64_t slot) {
  if (p == 0 || slot >= p) return -1;
  const uint64_t npairs = (p - 1) / 2;
  if (slot < 2 * npairs) return (int)((slot & 1) ? p - (slot / 2 + 1) : slot / 2 + 1);
  return slot == 2 * npairs ? 0 : (int)(p / 2);
}

int qt_int8_slots_create(const double* bh1, const double* bh2, uint64_t n, uint64_t s, uint64_t p, int slot0,
                         int nslots, int* nonfinite, void* stream, void** handle) {
  t_err.clear();
  if (!handle) return fail(QT_EINVAL, "int8 slots: null handle pointer");
  *handle = nullptr;
  int rc = check_dims(1, n, s, p, "int8 slots");
  if (rc) return rc;
  if (n == 0 || s == 0 || n % 32 != 0 || n > 8192 || p > 65534)
    return fail(QT_EINVAL, "int8 slots: needs s > 0, n %% 32 == 0, 0 < n <= 8192 and p <= 65534");
  const uint64_t pair_end = 2 * ((p - 1) / 2);  // slots [0, pair_end) hold pairs (2j, 2j+1)
  auto splits = [&](uint64_t b) { return (b & 1) && b < pair_end; };
  if (slot0 < 0 || nslots <= 0 || (uint64_t)slot0 + nslots > p || splits((uint64_t)slot0) ||
      splits((uint64_t)slot0 + nslots))
    return fail(QT_EINVAL, "int8 slots: the slot range must lie inside [0, p) and keep pairs whole");
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  Int8Slots* H = new Int8Slots;
  H->nonfinite = nonfinite;
  H->device = dev;
  H->bh1 = (const double2*)bh1;
  H->bh2 = (const double2*)bh2;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t fb = int8_flag_ints(p) * sizeof(int);
  cudaError_t e = cudaMallocAsync(&H->flags, fb, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(H->flags, 0, fb, st);
  if (e == cudaSuccess)
    e = ozaki_prepare_b_slots((const double2*)bh1, (const double2*)bh2, n, s, p, slot0, nslots, H->flags, &H->B, st);
  if (e != cudaSuccess) {
    if (H->flags) cudaFreeAsync(H->flags, st);
    delete H;
    return cuda_fail(e, "int8 slots: residues of B");
  }
  *handle = H;
  return QT_OK;
}

int qt_int8_slots_multiply(void* handle, const double* ah1, const double* ah2, uint64_t m, double* ch1, double* ch2,
                           void* stream) {
  t_err.clear();
  Int8Slots* H = (Int8Slots*)handle;
  if (!H) return fail(QT_EINVAL, "int8 slots: null handle");
  int rc = check_dims(m, H->B.n, H->B.s, H->B.p, "int8 slots multiply");
  if (rc) return rc;
  if (m == 0) return QT_OK;
  const uint64_t n = H->B.n, s = H->B.s, p = H->B.p;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = ozaki_multiply(H->B, (const double2*)ah1, (const double2*)ah2, nullptr, nullptr, m, (double2*)ch1,
                                 (double2*)ch2, s, m * s, H->flags, st);
  // non-finite inputs / uncertified pairs: the fp64 DMMA kernels recompute
  // them on the compact slot tensors (no-op otherwise)
  if (e == cudaSuccess)
    e = dmma_spectral_gemm_slots((const double2*)ah1, (const double2*)ah2, H->bh1, H->bh2, (double2*)ch1,
                                 (double2*)ch2, m, n, s, p, H->B.s0, H->B.ns, st, H->flags);
  // the caller's flag reports non-finite inputs (the result is the DMMA one then)
  if (e == cudaSuccess && H->nonfinite) e = cudaMemcpyAsync(H->nonfinite, H->flags, sizeof(int), cudaMemcpyDeviceToDevice, st);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "int8 slots multiply");
}

int qt_int8_slots_destroy(void* handle, void* stream) {
  t_err.clear();
  Int8Slots* H = (Int8Slots*)handle;
  if (!H) return QT_OK;
  cudaError_t e = ozaki_release(H->B, (cudaStream_t)stream);
  const cudaError_t fe = cudaFreeAsync(H->flags, (cudaStream_t)stream);
  if (e == cudaSuccess) e = fe;
  delete H;
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "int8 slots destroy");
}

uint64_t qt_int8_guard_fallbacks(void) { return int8_guard_fallbacks(); }

int qt_small_fused(uint64_t m, uint64_t n, uint64_t s, uint64_t p) {
  return small_fused_eligible(m, n, s, p) ? 1 : 0;
}

int qt_gemm_algo(uint64_t m, uint64_t n, uint64_t s, uint64_t p) {
  (void)m;
  (void)p;
  return choose_gemm_algo(n, s, p);
}

static int tprod_host_impl(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                           double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, HostCall& hc) {
  int rc = QT_OK;
  const size_t ab = m * n * p * sizeof(double2), bb = n * s * p * sizeof(double2), cb = m * s * p * sizeof(double2);
  // Large problems stream (row slab x column chunk) tiles: ~8 slabs of >= 64
  // rows and ~8 chunks of >= 64 columns (a multiple of the GEMM tile).
  // Products on the int8 K2 stream row slabs against resident B' residues.
  if (n > 0 && s > 0 && m >= 128 && ab + bb + cb >= (128ull << 20) && choose_gemm_algo(n, s, p) == kAlgoOzaki) {
    // ~16 slabs of >= 128 rows (measured on config 5: 4 slabs 196 ms, 8 slabs
    // 182 ms, 16 slabs 175 ms end to end — finer slabs start computing sooner
    // and leave less after the last upload)
    const uint64_t nsl = (uint64_t)std::max(1, atoi(getenv("QTB_E2E_SLABS") ? getenv("QTB_E2E_SLABS") : "16"));
    uint64_t R = std::max<uint64_t>(128, (m + nsl - 1) / nsl);
    R = (R + 127) / 128 * 128;
    return tprod_host_slabs_ozaki(a1, a2, b1, b2, c1, c2, m, n, s, p, R, hc);
  }
  if (n > 0 && s > 0 && m >= 128 && ab + bb + cb >= (128ull << 20)) {
    uint64_t R = std::max<uint64_t>(64, (m + 7) / 8);
    R = (R + 63) / 64 * 64;
    uint64_t Q = s >= 128 ? std::max<uint64_t>(64, (s + 7) / 8) : s;
    if (Q < s) Q = (Q + 15) / 16 * 16;
    return tprod_host_tiled(a1, a2, b1, b2, c1, c2, m, n, s, p, R, Q, hc);
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

int qt_tprod_f64_host(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                      double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, int device) {
  t_err.clear();
  int rc = check_dims(m, n, s, p, "tprod_fast");
  if (rc) return rc;
  HostCall hc;
  if ((rc = hc.begin(device))) return rc;
  const size_t ab = m * n * p * sizeof(double2), bb = n * s * p * sizeof(double2), cb = m * s * p * sizeof(double2);
  // pageable caller buffers (e.g. the drop-in's std::vector): stage through the
  // cached pinned arena with all host cores (see is_pinned / parallel_copy)
  if (ab + bb + cb >= (256ull << 20) && getenv("QTB_NO_PINNED_STAGING") == nullptr &&
      !(is_pinned(a1) && is_pinned(a2) && is_pinned(b1) && is_pinned(b2) && is_pinned(c1) && is_pinned(c2))) {
    PinnedArena& ar = pinned_arena();
    std::unique_lock<std::mutex> lk(ar.mu, std::try_to_lock);
    if (lk.owns_lock()) {
      const size_t need = 2 * (ab + bb + cb);
      if (ar.size < need) {
        if (ar.ptr) cudaFreeHost(ar.ptr);
        ar.ptr = nullptr;
        ar.size = 0;
        if (cudaHostAlloc(&ar.ptr, need, cudaHostAllocDefault) == cudaSuccess) ar.size = need;
        else cudaGetLastError();
      }
      if (ar.ptr) {
        char* base = (char*)ar.ptr;
        double* pa1 = (double*)base;
        double* pa2 = (double*)(base + ab);
        double* pb1 = (double*)(base + 2 * ab);
        double* pb2 = (double*)(base + 2 * ab + bb);
        double* pc1 = (double*)(base + 2 * ab + 2 * bb);
        double* pc2 = (double*)(base + 2 * ab + 2 * bb + cb);
        parallel_copy(pa1, a1, ab);
        parallel_copy(pa2, a2, ab);
        parallel_copy(pb1, b1, bb);
        parallel_copy(pb2, b2, bb);
        rc = tprod_host_impl(pa1, pa2, pb1, pb2, pc1, pc2, m, n, s, p, hc);
        if (rc == QT_OK) {
          parallel_copy(c1, pc1, cb);
          parallel_copy(c2, pc2, cb);
        }
        return rc;
      }
    }
  }
  return tprod_host_impl(a1, a2, b1, b2, c1, c2, m, n, s, p, hc);
}

// tprod_fast with the reference's workspace side effect (tproduct.cpp:80-87:
// after a call ws.ahat / ws.bhat / ws.chat hold Â, B̂, Ĉ): the device
// pipeline with each stage's output also copied back to the caller's host
// buffers.  The stages are the product's own kernels, so C is the same as
// qt_tprod_f64_host's (for sizes whose host path does not stream).
int qt_tprod_f64_host_spectra(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                              double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, int device, double* ah1,
                              double* ah2, double* bh1, double* bh2, double* ch1, double* ch2) {
  t_err.clear();
  int rc = check_dims(m, n, s, p, "tprod_fast");
  if (rc) return rc;
  HostCall hc;
  if ((rc = hc.begin(device))) return rc;
  const size_t ab = m * n * p * sizeof(double2), bb = n * s * p * sizeof(double2), cb = m * s * p * sizeof(double2);
  char* d = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&d, 4 * ab + 4 * bb + 2 * cb + 64, hc.st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(host call)");
  double* da1 = (double*)d;
  double* da2 = (double*)(d + ab);
  double* dh1 = (double*)(d + 2 * ab);
  double* dh2 = (double*)(d + 3 * ab);
  double* db1 = (double*)(d + 4 * ab);
  double* db2 = (double*)(d + 4 * ab + bb);
  double* dk1 = (double*)(d + 4 * ab + 2 * bb);
  double* dk2 = (double*)(d + 4 * ab + 3 * bb);
  double* dc1 = (double*)(d + 4 * ab + 4 * bb);
  double* dc2 = (double*)(d + 4 * ab + 4 * bb + cb);
  if (ab) rc = h2d(da1, a1, ab, hc.st);
  if (!rc && ab) rc = h2d(da2, a2, ab, hc.st);
  if (!rc && bb) rc = h2d(db1, b1, bb, hc.st);
  if (!rc && bb) rc = h2d(db2, b2, bb, hc.st);
  if (!rc && m && n) rc = transform_device_impl(false, da1, da2, dh1, dh2, m, n, p, hc.st);
  if (!rc && n && s) rc = transform_device_impl(false, db1, db2, dk1, dk2, n, s, p, hc.st);
  if (!rc && ab) rc = d2h(ah1, dh1, ab, hc.st);
  if (!rc && ab) rc = d2h(ah2, dh2, ab, hc.st);
  if (!rc && bb) rc = d2h(bh1, dk1, bb, hc.st);
  if (!rc && bb) rc = d2h(bh2, dk2, bb, hc.st);
  if (!rc && cb) {
    if (n == 0) {
      if ((e = cudaMemsetAsync(dc1, 0, 2 * cb, hc.st)) != cudaSuccess) rc = cuda_fail(e, "memset");
    } else if ((e = launch_spectral_gemm((const double2*)dh1, (const double2*)dh2, (const double2*)dk1,
                                         (const double2*)dk2, (double2*)dc1, (double2*)dc2, m, n, s, p, hc.st)) !=
               cudaSuccess) {
      rc = cuda_fail(e, "K2 paired spectral GEMM");
    }
  }
  if (!rc && cb) rc = d2h(ch1, dc1, cb, hc.st);
  if (!rc && cb) rc = d2h(ch2, dc2, cb, hc.st);
  if (!rc && cb && n) rc = transform_device_impl(true, dc1, dc2, dc1, dc2, m, s, p, hc.st);  // (n = 0: C = 0, as tprod_fast)
  if (!rc && cb) rc = d2h(c1, dc1, cb, hc.st);
  if (!rc && cb) rc = d2h(c2, dc2, cb, hc.st);
  cudaFreeAsync(d, hc.st);
  e = cudaStreamSynchronize(hc.st);
  if (!rc && e != cudaSuccess) rc = cuda_fail(e, "tprod_fast (host) sync");
  return rc;
}

int qt_tprod_naive_f64_device(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                              double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, void* stream) {
  t_err.clear();
  int rc = check_dims(m, n, s, p, "tprod_naive");
  if (rc) return rc;
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  cudaError_t e = launch_naive_tprod((const double2*)a1, (const double2*)a2, (const double2*)b1, (const double2*)b2,
                                     (double2*)c1, (double2*)c2, m, n, s, p, (cudaStream_t)stream);
  return e == cudaSuccess ? QT_OK : cuda_fail(e, "definitional T-product");
}

int qt_tprod_naive_f64_host(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                            double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, int device) {
  t_err.clear();
  int rc = check_dims(m, n, s, p, "tprod_naive");
  if (rc) return rc;
  HostCall hc;
  if ((rc = hc.begin(device))) return rc;
  const size_t ab = m * n * p * sizeof(double2), bb = n * s * p * sizeof(double2), cb = m * s * p * sizeof(double2);
  char* d = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&d, 2 * (ab + bb + cb) + 64, hc.st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(host call)");
  double* da1 = (double*)d;
  double* da2 = (double*)(d + ab);
  double* db1 = (double*)(d + 2 * ab);
  double* db2 = (double*)(d + 2 * ab + bb);
  double* dc1 = (double*)(d + 2 * ab + 2 * bb);
  double* dc2 = (double*)(d + 2 * ab + 2 * bb + cb);
  rc = QT_OK;
  if (!rc && ab) rc = h2d(da1, a1, ab, hc.st);
  if (!rc && ab) rc = h2d(da2, a2, ab, hc.st);
  if (!rc && bb) rc = h2d(db1, b1, bb, hc.st);
  if (!rc && bb) rc = h2d(db2, b2, bb, hc.st);
  if (!rc) rc = qt_tprod_naive_f64_device(da1, da2, db1, db2, dc1, dc2, m, n, s, p, hc.st);
  if (!rc && cb) rc = d2h(c1, dc1, cb, hc.st);
  if (!rc && cb) rc = d2h(c2, dc2, cb, hc.st);
  cudaFreeAsync(d, hc.st);
  e = cudaStreamSynchronize(hc.st);
  if (!rc && e != cudaSuccess) rc = cuda_fail(e, "tprod_naive (host) sync");
  return rc;
}

int qt_qt3_probe(const char* path, uint64_t* m, uint64_t* n, uint64_t* p) {
  t_err.clear();
  if (!path || !m || !n || !p) return fail(QT_EINVAL, "qt3_probe: null argument");
  std::string err;
  const int rc = qt3_probe(path, m, n, p, &err);
  return rc ? fail(rc, "read_tensor: %s", err.c_str()) : QT_OK;
}

int qt_qt3_read_f64_device(const char* path, double* t1, double* t2, uint64_t m, uint64_t n, uint64_t p,
                           void* stream) {
  t_err.clear();
  if (!path) return fail(QT_EINVAL, "qt3_read: null path");
  int dev = 0;
  int rc = current_device(&dev);
  if (rc) return rc;
  std::string err;
  rc = qt3_read_device(path, t1, t2, m, n, p, (cudaStream_t)stream, &err);
  return rc ? fail(rc, "read_tensor: %s", err.c_str()) : QT_OK;
}

int qt_qt3_write_f64_device(const char* path, const double* t1, const double* t2, uint64_t m, uint64_t n, uint64_t p,
                            void* stream) {
  t_err.clear();
  if (!path) return fail(QT_EINVAL, "qt3_write: null path");
  int dev = 0;
  int rc = current_device(&dev);
  if (rc) return rc;
  std::string err;
  rc = qt3_write_device(path, t1, t2, m, n, p, (cudaStream_t)stream, &err);
  return rc ? fail(rc, "write_tensor: %s", err.c_str()) : QT_OK;
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
