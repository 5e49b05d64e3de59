// qt_multi.cu — single-process multi-GPU driver for the T-product.
//
// The reference is single-threaded and has no distributed path;
// this is the B200-native scale-out of tprod_fast (tproduct.cpp:75-111):
//   * rows of A and C are split into contiguous slabs of ceil(m/G) rows — row i
//     of C depends only on row i of A and all of B, so slabs are independent;
//   * B is the only exchange: column chunk j is uploaded by device j mod G
//     (each device moves ~1/G of B over its own PCIe link); with peer access
//     the owner transforms it once and K1's routed stores write B̂ into every
//     device's chunk buffer over NVLink (the broadcast fused into the
//     transform), else it is broadcast raw with ncclBroadcast on a
//     communication stream and every device transforms it; each compute
//     stream waits only for the chunk it needs and multiplies it into the
//     matching columns of its C slab (strided K2), so the transfer of chunk
//     j+1 overlaps the compute of chunk j;
//   * one inverse transform (K3) per slab, then the slab goes back to the host.
// Every element is computed with the same kernels and arithmetic as the
// single-GPU path, so the result is bitwise identical for every G (and equal to
// qt_tprod_f64_host).  NCCL is resolved at run time (dlopen) so the library
// does not pin an NCCL build: an NCCL the process already loaded (torch's) is
// reused first, then $QTB_NCCL_LIB, then the loader's libnccl.so.2.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qtensor_b200.h"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // 1) an NCCL the process already loaded (e.g. torch's bundled build) — a
    //    second libnccl.so.2 would shadow it by soname and break its users;
    // 2) $QTB_NCCL_LIB; 3) the loader's libnccl.so.2.
    for (const char* nm : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (api.h) break;
    }
    if (!api.h) {
      const char* env = getenv("QTB_NCCL_LIB");
      if (env && *env) api.h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    }
    for (const char* nm : {"libnccl.so.2", "libnccl.so"}) {
      if (api.h) break;
      api.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
    }
    if (!api.h) return;
    api.CommInitAll = (decltype(api.CommInitAll))dlsym(api.h, "ncclCommInitAll");
    api.Broadcast = (decltype(api.Broadcast))dlsym(api.h, "ncclBroadcast");
    api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
    api.ok = api.CommInitAll && api.Broadcast && api.GroupStart && api.GroupEnd;
  });
  return api;
}

std::mutex g_comm_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_comms;

struct DevState {
  int dev = 0;
  cudaStream_t comp = nullptr, comm = nullptr;
  double* buf = nullptr;  // A slab, Â slab, C slab, B chunks, B̂ chunk (2 planes each)
  std::vector<cudaEvent_t> evs;
  int rc = QT_OK;
};

}  // namespace

extern "C" {

int qt_tprod_f64_multi(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                       double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, const int* devices, int ndev) {
  if (ndev <= 0 || !devices) return QT_EINVAL;
  if (p == 0) return QT_EINVAL;
  if (m == 0 || s == 0 || n == 0 || (uint64_t)ndev > m)
    return qt_tprod_f64_host(a1, a2, b1, b2, c1, c2, m, n, s, p, devices[0]);
  NcclApi& api = nccl();
  if (!api.ok) return QT_ENCCL;

  std::vector<int> key(devices, devices + ndev);
  std::vector<ncclComm_t> comms;
  {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    auto it = g_comms.find(key);
    if (it == g_comms.end()) {
      std::vector<ncclComm_t> c(ndev);
      if (api.CommInitAll(c.data(), ndev, devices) != ncclSuccess) return QT_ENCCL;
      it = g_comms.emplace(key, c).first;
    }
    comms = it->second;
  }

  const size_t cx = 2 * sizeof(double);
  const uint64_t slab = (m + ndev - 1) / ndev;
  // column chunks of B: ~8, a multiple of the 16-column GEMM tile
  uint64_t Q = std::max<uint64_t>(16, (s + 7) / 8);
  Q = std::min<uint64_t>(s, (Q + 15) / 16 * 16);
  const uint64_t NJ = (s + Q - 1) / Q;
  std::vector<DevState> st(ndev);
  std::vector<uint64_t> r0(ndev), rows(ndev);
  for (int g = 0; g < ndev; ++g) {
    r0[g] = std::min<uint64_t>(m, g * slab);
    rows[g] = std::min<uint64_t>(m, r0[g] + slab) - r0[g];
  }
  auto chunk_cols = [&](uint64_t j) { return std::min<uint64_t>(Q, s - j * Q); };
  const size_t bchunk = n * Q * p * cx;  // per plane

  // 1) per device: streams, buffers, A slab upload + K1(A)
  auto setup = [&](int g) {
    DevState& d = st[g];
    d.dev = devices[g];
    if (cudaSetDevice(d.dev) != cudaSuccess) { d.rc = QT_ECUDA; return; }
    if (cudaStreamCreateWithFlags(&d.comp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&d.comm, cudaStreamNonBlocking) != cudaSuccess) {
      d.rc = QT_ECUDA;
      return;
    }
    const size_t ab = rows[g] * n * p * cx, cb = rows[g] * s * p * cx;
    const size_t total = 4 * ab + 2 * cb + NJ * 2 * bchunk + 2 * bchunk + 1024;
    if (cudaMallocAsync((void**)&d.buf, total, d.comp) != cudaSuccess) { d.rc = QT_ENOMEM; return; }
    cudaEvent_t ready;
    cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    cudaEventRecord(ready, d.comp);
    cudaStreamWaitEvent(d.comm, ready, 0);
    d.evs.push_back(ready);
    char* base = (char*)d.buf;
    double* A1 = (double*)base;
    double* A2 = (double*)(base + ab);
    const size_t spitch = m * n * cx, width = rows[g] * n * cx;
    if (cudaMemcpy2DAsync(A1, width, a1 + 2 * r0[g] * n, spitch, width, p, cudaMemcpyHostToDevice, d.comp) ||
        cudaMemcpy2DAsync(A2, width, a2 + 2 * r0[g] * n, spitch, width, p, cudaMemcpyHostToDevice, d.comp)) {
      d.rc = QT_ECUDA;
      return;
    }
    d.rc = qt_qfft3_conj_f64_device(A1, A2, (double*)(base + 2 * ab), (double*)(base + 3 * ab), rows[g], n, p,
                                    d.comp);
  };
  {
    std::vector<std::thread> th;
    for (int g = 0; g < ndev; ++g) th.emplace_back(setup, g);
    for (auto& t : th) t.join();
  }
  int rc = QT_OK;
  for (int g = 0; g < ndev; ++g) rc = rc ? rc : st[g].rc;

  auto chunk_ptr = [&](int g, uint64_t j, int plane) {
    const size_t ab = rows[g] * n * p * cx, cb = rows[g] * s * p * cx;
    return (double*)((char*)st[g].buf + 4 * ab + 2 * cb + (2 * j + plane) * bchunk);
  };
  auto bhat_ptr = [&](int g, int plane) {
    const size_t ab = rows[g] * n * p * cx, cb = rows[g] * s * p * cx;
    return (double*)((char*)st[g].buf + 4 * ab + 2 * cb + 2 * NJ * bchunk + plane * bchunk);
  };

  // 2) B chunks: chunk j is uploaded by device owner(j) = j mod ndev (so each
  //    device moves ~1/ndev of B over its own PCIe link).  Fused form (every
  //    device pair has peer access; QTB_MULTI_FUSED=0 turns it off): the owner
  //    transforms the chunk once and K1's stores put each frequency row of B̂
  //    straight into every device's chunk buffer over NVLink
  //    (qt_qfft3_conj_f64_device_routed_n) — the broadcast and the replicated
  //    K1 of the chunk disappear.  Otherwise the raw chunk is broadcast (one
  //    NCCL group per chunk) and every device transforms it.
  bool fused = qt_fft_routable(p) == 1 && [] {
    const char* v = getenv("QTB_MULTI_FUSED");
    return !(v && *v == '0');
  }();
  for (int a = 0; a < ndev && fused; ++a)
    for (int b = 0; b < ndev && fused; ++b) {
      if (a == b) continue;
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]) != cudaSuccess || !ok) {
        fused = false;
        break;
      }
      cudaSetDevice(devices[a]);
      const cudaError_t pe = cudaDeviceEnablePeerAccess(devices[b], 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) fused = false;
      (void)cudaGetLastError();
    }
  std::vector<void*> tabs;  // per chunk: device row tables (in the owner's memory)
  std::vector<std::vector<cudaEvent_t>> arrived(ndev, std::vector<cudaEvent_t>(NJ, nullptr));
  for (uint64_t j = 0; j < NJ && !rc && fused; ++j) {
    const uint64_t cols = chunk_cols(j);
    const int own = (int)(j % (uint64_t)ndev);
    cudaSetDevice(st[own].dev);
    const size_t pitch = s * cx, width = cols * cx;
    if (cudaMemcpy2DAsync(chunk_ptr(own, j, 0), width, b1 + 2 * j * Q, pitch, width, p * n, cudaMemcpyHostToDevice,
                          st[own].comm) ||
        cudaMemcpy2DAsync(chunk_ptr(own, j, 1), width, b2 + 2 * j * Q, pitch, width, p * n, cudaMemcpyHostToDevice,
                          st[own].comm)) {
      rc = QT_ECUDA;
      break;
    }
    // row tables [plane][device][frequency]: frequency k of device g's chunk j
    std::vector<double*> h(2 * (size_t)ndev * p);
    for (int pl = 0; pl < 2; ++pl)
      for (int g = 0; g < ndev; ++g)
        for (uint64_t k = 0; k < p; ++k) h[((size_t)pl * ndev + g) * p + k] = chunk_ptr(g, j, pl) + 2 * k * n * cols;
    double** dt = nullptr;
    if (cudaMallocAsync((void**)&dt, h.size() * sizeof(double*), st[own].comm) != cudaSuccess ||
        cudaMemcpyAsync(dt, h.data(), h.size() * sizeof(double*), cudaMemcpyHostToDevice, st[own].comm) != cudaSuccess ||
        cudaStreamSynchronize(st[own].comm) != cudaSuccess) {  // (h is a host temporary)
      rc = QT_ECUDA;
      break;
    }
    tabs.push_back(dt);
    // in place on the owner: each tube tile is read whole before it is written
    rc = qt_qfft3_conj_f64_device_routed_n(chunk_ptr(own, j, 0), chunk_ptr(own, j, 1), dt, dt + (size_t)ndev * p,
                                           ndev, n, cols, p, st[own].comm);
    if (rc) break;
    cudaEvent_t done;
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    cudaEventRecord(done, st[own].comm);
    for (int g = 0; g < ndev; ++g) arrived[g][j] = g == own ? done : nullptr;
    for (int g = 0; g < ndev; ++g)
      if (g != own) {  // every device waits on the owner's event (cross-device waits are legal in one process)
        cudaSetDevice(st[g].dev);
        cudaEventCreateWithFlags(&arrived[g][j], cudaEventDisableTiming);
        cudaStreamWaitEvent(st[g].comm, done, 0);
        cudaEventRecord(arrived[g][j], st[g].comm);
      }
  }
  for (uint64_t j = 0; j < NJ && !rc && !fused; ++j) {
    const uint64_t cols = chunk_cols(j);
    const int own = (int)(j % (uint64_t)ndev);
    cudaSetDevice(st[own].dev);
    const size_t pitch = s * cx, width = cols * cx;
    if (cudaMemcpy2DAsync(chunk_ptr(own, j, 0), width, b1 + 2 * j * Q, pitch, width, p * n, cudaMemcpyHostToDevice,
                          st[own].comm) ||
        cudaMemcpy2DAsync(chunk_ptr(own, j, 1), width, b2 + 2 * j * Q, pitch, width, p * n, cudaMemcpyHostToDevice,
                          st[own].comm)) {
      rc = QT_ECUDA;
      break;
    }
    const size_t count = 2 * n * cols * p * 2;  // doubles in both planes (planes are adjacent chunks)
    if (api.GroupStart() != ncclSuccess) { rc = QT_ENCCL; break; }
    for (int g = 0; g < ndev; ++g) {
      cudaSetDevice(st[g].dev);
      // both planes of chunk j are contiguous: [plane0 (n*cols*p)][gap][plane1] — broadcast each plane
      if (api.Broadcast(chunk_ptr(g, j, 0), chunk_ptr(g, j, 0), count / 2, ncclFloat64, own, comms[g], st[g].comm) !=
              ncclSuccess ||
          api.Broadcast(chunk_ptr(g, j, 1), chunk_ptr(g, j, 1), count / 2, ncclFloat64, own, comms[g], st[g].comm) !=
              ncclSuccess)
        rc = QT_ENCCL;
    }
    if (api.GroupEnd() != ncclSuccess) rc = QT_ENCCL;
    for (int g = 0; g < ndev; ++g) {
      cudaSetDevice(st[g].dev);
      cudaEventCreateWithFlags(&arrived[g][j], cudaEventDisableTiming);
      cudaEventRecord(arrived[g][j], st[g].comm);
    }
  }

  // 3) per device: for each chunk K1(B chunk) + strided K2 into the C slab; K3; download
  const int algo = qt_gemm_algo(m, n, s, p);  // every rank and chunk: the full product's choice
  auto compute = [&](int g) {
    DevState& d = st[g];
    cudaSetDevice(d.dev);
    const size_t ab = rows[g] * n * p * cx, cb = rows[g] * s * p * cx;
    char* base = (char*)d.buf;
    const double* Ah1 = (double*)(base + 2 * ab);
    const double* Ah2 = (double*)(base + 3 * ab);
    double* C1 = (double*)(base + 4 * ab);
    double* C2 = (double*)(base + 4 * ab + cb);
    int& r = d.rc;
    void* plan = nullptr;  // exact int8 stage 2: Â slab residues built once, reused by every chunk
    if (r == QT_OK && algo == QT_GEMM_INT8_EXACT && rows[g] > 0)
      r = qt_int8_plan_create(Ah1, Ah2, rows[g], n, p, d.comp, &plan);
    for (uint64_t j = 0; j < NJ && r == QT_OK; ++j) {
      const uint64_t cols = chunk_cols(j);
      cudaStreamWaitEvent(d.comp, arrived[g][j], 0);
      // fused: chunk j already holds B̂ (stored by its owner's K1)
      const double* bh1 = fused ? chunk_ptr(g, j, 0) : bhat_ptr(g, 0);
      const double* bh2 = fused ? chunk_ptr(g, j, 1) : bhat_ptr(g, 1);
      if (!fused)
        r = qt_qfft3_conj_f64_device(chunk_ptr(g, j, 0), chunk_ptr(g, j, 1), bhat_ptr(g, 0), bhat_ptr(g, 1), n,
                                     cols, p, d.comp);
      if (r == QT_OK && plan)
        r = qt_int8_plan_multiply(plan, bh1, bh2, C1 + 2 * j * Q, C2 + 2 * j * Q, cols, cols, s, n * cols,
                                  rows[g] * s, d.comp);
      else if (r == QT_OK)
        r = qt_spectral_product_f64_device_ld_algo(Ah1, Ah2, bh1, bh2, C1 + 2 * j * Q, C2 + 2 * j * Q, rows[g], n,
                                                   cols, p, cols, s, n * cols, rows[g] * s, algo, d.comp);
    }
    if (plan) {
      const int dr = qt_int8_plan_destroy(plan, d.comp);
      if (r == QT_OK) r = dr;
    }
    if (r == QT_OK) r = qt_qifft3_conj_f64_device(C1, C2, C1, C2, rows[g], s, p, d.comp);
    if (r == QT_OK) {
      const size_t dpitch = m * s * cx, width = rows[g] * s * cx;
      if (cudaMemcpy2DAsync(c1 + 2 * r0[g] * s, dpitch, C1, width, width, p, cudaMemcpyDeviceToHost, d.comp) ||
          cudaMemcpy2DAsync(c2 + 2 * r0[g] * s, dpitch, C2, width, width, p, cudaMemcpyDeviceToHost, d.comp))
        r = QT_ECUDA;
    }
    if (cudaStreamSynchronize(d.comp) != cudaSuccess && r == QT_OK) r = QT_ECUDA;
  };
  if (!rc) {
    std::vector<std::thread> th;
    for (int g = 0; g < ndev; ++g) th.emplace_back(compute, g);
    for (auto& t : th) t.join();
    for (int g = 0; g < ndev; ++g) rc = rc ? rc : st[g].rc;
  }

  for (uint64_t j = 0; j < tabs.size(); ++j) {  // row tables: on chunk j's owner, freed after its stream drains
    const int own = (int)(j % (uint64_t)ndev);
    cudaSetDevice(st[own].dev);
    cudaFreeAsync(tabs[j], st[own].comm);
    cudaStreamSynchronize(st[own].comm);
  }
  for (int g = 0; g < ndev; ++g) {
    DevState& d = st[g];
    if (!d.comp) continue;
    cudaSetDevice(d.dev);
    cudaStreamSynchronize(d.comm);
    if (d.buf) cudaFreeAsync(d.buf, d.comp);
    cudaStreamSynchronize(d.comp);
    for (cudaEvent_t e : d.evs) cudaEventDestroy(e);
    for (cudaEvent_t e : arrived[g])
      if (e) cudaEventDestroy(e);
    cudaStreamDestroy(d.comp);
    cudaStreamDestroy(d.comm);
  }
  return rc;
}

}  // extern "C"
