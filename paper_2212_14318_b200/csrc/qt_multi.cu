// qt_multi.cu — single-process multi-GPU driver for the T-product.
//
// The reference is single-threaded and has no distributed path;
// this is the B200-native scale-out of tprod_fast (tproduct.cpp:75-111):
//   * rows of A and C are split into contiguous slabs of ceil(m/G) rows — row i
//     of C depends only on row i of A and all of B, so slabs are independent
//     and the result is bitwise identical for every G;
//   * B is copied host->device once (to devices[0]) and broadcast over NVLink /
//     NVSwitch with one ncclBroadcast per call (both CD planes in one buffer);
//   * each device runs the same K1 -> K2 -> K3 pipeline on its slab.
// NCCL is resolved at run time with dlopen("libnccl.so.2") so the library does
// not pin an NCCL build (torch bundles its own); G == 1 never touches NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
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
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.CommInitAll = (decltype(api.CommInitAll))dlsym(api.h, "ncclCommInitAll");
    api.Broadcast = (decltype(api.Broadcast))dlsym(api.h, "ncclBroadcast");
    api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
    api.ok = api.CommInitAll && api.Broadcast && api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  return api;
}

std::mutex g_comm_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_comms;

thread_local std::string t_multi_err;

}  // namespace

extern "C" {

// declared in qtensor_b200.h
int qt_tprod_f64_multi(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                       double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, const int* devices, int ndev) {
  if (ndev <= 0 || !devices) return QT_EINVAL;
  if (p == 0) return QT_EINVAL;
  if (ndev == 1 || m < (uint64_t)ndev) {
    return qt_tprod_f64_host(a1, a2, b1, b2, c1, c2, m, n, s, p, devices[0]);
  }
  NcclApi& api = nccl();
  if (!api.ok) return QT_ENCCL;

  std::vector<int> key(devices, devices + ndev);
  std::vector<ncclComm_t> comms;
  {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    auto it = g_comms.find(key);
    if (it == g_comms.end()) {
      std::vector<ncclComm_t> c(ndev);
      ncclResult_t r = api.CommInitAll(c.data(), ndev, devices);
      if (r != ncclSuccess) return QT_ENCCL;
      it = g_comms.emplace(key, c).first;
    }
    comms = it->second;
  }

  const uint64_t slab = (m + ndev - 1) / ndev;
  const size_t cx = sizeof(double) * 2;
  const size_t bbytes = n * s * p * cx;
  std::vector<int> rcs(ndev, QT_OK);
  std::vector<cudaStream_t> streams(ndev, nullptr);
  std::vector<double*> dB(ndev, nullptr), dA(ndev, nullptr), dC(ndev, nullptr);
  std::vector<uint64_t> r0(ndev), rows(ndev);
  for (int g = 0; g < ndev; ++g) {
    r0[g] = std::min<uint64_t>(m, g * slab);
    rows[g] = std::min<uint64_t>(m, r0[g] + slab) - r0[g];
  }

  // 1) per-device setup + A slab upload; B to device 0
  auto setup = [&](int g) {
    int& rc = rcs[g];
    if (cudaSetDevice(devices[g]) != cudaSuccess) { rc = QT_ECUDA; return; }
    if (cudaStreamCreateWithFlags(&streams[g], cudaStreamNonBlocking) != cudaSuccess) { rc = QT_ECUDA; return; }
    cudaStream_t st = streams[g];
    const size_t ab = rows[g] * n * p * cx, cb = rows[g] * s * p * cx;
    if (cudaMallocAsync((void**)&dB[g], 2 * bbytes + 16, st) != cudaSuccess) { rc = QT_ENOMEM; return; }
    if (cudaMallocAsync((void**)&dA[g], 2 * ab + 16, st) != cudaSuccess) { rc = QT_ENOMEM; return; }
    if (cudaMallocAsync((void**)&dC[g], 2 * cb + 16, st) != cudaSuccess) { rc = QT_ENOMEM; return; }
    if (rows[g] && n) {
      // slab = p strided chunks of rows x n complex (slice-major layout)
      const size_t spitch = m * n * cx, width = rows[g] * n * cx;
      const double* src1 = a1 + 2 * r0[g] * n;
      const double* src2 = a2 + 2 * r0[g] * n;
      if (cudaMemcpy2DAsync(dA[g], width, src1, spitch, width, p, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaMemcpy2DAsync((char*)dA[g] + ab, width, src2, spitch, width, p, cudaMemcpyHostToDevice, st) !=
              cudaSuccess) {
        rc = QT_ECUDA;
        return;
      }
    }
    if (g == 0 && bbytes) {
      if (cudaMemcpyAsync(dB[0], b1, bbytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaMemcpyAsync((char*)dB[0] + bbytes, b2, bbytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
        rc = QT_ECUDA;
      }
    }
  };
  {
    std::vector<std::thread> th;
    for (int g = 0; g < ndev; ++g) th.emplace_back(setup, g);
    for (auto& t : th) t.join();
  }
  int rc = QT_OK;
  for (int g = 0; g < ndev; ++g) rc = rc ? rc : rcs[g];

  // 2) broadcast both B planes from devices[0] (one NCCL group)
  if (!rc && bbytes) {
    const size_t count = 2 * bbytes / sizeof(double) + 0;
    api.GroupStart();
    for (int g = 0; g < ndev && !rc; ++g) {
      cudaSetDevice(devices[g]);
      if (api.Broadcast(dB[g], dB[g], count, ncclFloat64, 0, comms[g], streams[g]) != ncclSuccess) rc = QT_ENCCL;
    }
    if (api.GroupEnd() != ncclSuccess) rc = QT_ENCCL;
  }

  // 3) per-device pipeline + strided download of the C slab
  auto compute = [&](int g) {
    int& r = rcs[g];
    cudaSetDevice(devices[g]);
    cudaStream_t st = streams[g];
    const size_t ab = rows[g] * n * p * cx, cb = rows[g] * s * p * cx;
    r = qt_tprod_f64_device(dA[g], (double*)((char*)dA[g] + ab), dB[g], (double*)((char*)dB[g] + bbytes), dC[g],
                            (double*)((char*)dC[g] + cb), rows[g], n, s, p, st);
    if (r == QT_OK && rows[g] && s) {
      const size_t dpitch = m * s * cx, width = rows[g] * s * cx;
      double* dst1 = c1 + 2 * r0[g] * s;
      double* dst2 = c2 + 2 * r0[g] * s;
      if (cudaMemcpy2DAsync(dst1, dpitch, dC[g], width, width, p, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaMemcpy2DAsync(dst2, dpitch, (char*)dC[g] + cb, width, width, p, cudaMemcpyDeviceToHost, st) !=
              cudaSuccess)
        r = QT_ECUDA;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && r == QT_OK) r = QT_ECUDA;
  };
  if (!rc) {
    std::vector<std::thread> th;
    for (int g = 0; g < ndev; ++g) th.emplace_back(compute, g);
    for (auto& t : th) t.join();
    for (int g = 0; g < ndev; ++g) rc = rc ? rc : rcs[g];
  }

  for (int g = 0; g < ndev; ++g) {
    if (!streams[g]) continue;
    cudaSetDevice(devices[g]);
    cudaFreeAsync(dA[g], streams[g]);
    cudaFreeAsync(dB[g], streams[g]);
    cudaFreeAsync(dC[g], streams[g]);
    cudaStreamSynchronize(streams[g]);
    cudaStreamDestroy(streams[g]);
  }
  return rc;
}

}  // extern "C"
