// qt_multi.cu — single-process multi-GPU driver for the T-product: the
// north_star split (BASELINE.json) of tprod_fast (tproduct.cpp:75-111).
//
// The reference is single-threaded and has no distributed path.
//   * rows of A and C are split into contiguous slabs of ceil(m/G) rows — row i
//     of C depends only on row i of A and all of B, so slabs are independent;
//   * B is the only exchange: uploaded once to devices[0] and broadcast to the
//     others with one grouped ncclBroadcast per CD plane (NVLink / NVSwitch);
//   * every device then runs the whole single-GPU pipeline on its slab
//     (qt_tprod_f64_device: K1 of its A rows and of B, stage 2, K3) and copies
//     its rows of C back.
// A slab runs the same kernels with the same per-element arithmetic as the
// full product (the int8 stage 2's scalings are per row of A and per column /
// contraction index of B, and B is whole on every device), so C is bitwise
// identical to the single-GPU result for every G (up to the int8 accuracy
// guard, which certifies each slab's frequency pairs on their own; a pair it
// rejects on one slab is recomputed there by the fp64 kernels).
// NCCL is resolved at run time (qt_nccl.h) so the library does not pin an
// NCCL build.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/qtensor_b200.h"
#include "qt_nccl.h"

namespace {

using qtb::NcclApi;

std::mutex g_comm_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_comms;

struct DevState {
  int dev = 0;
  cudaStream_t st = nullptr;
  double* buf = nullptr;  // A slab (2 planes), B (2), C slab (2)
  int rc = QT_OK;
};

}  // namespace

extern "C" {

int qt_tprod_f64_multi(const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                       double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, const int* devices, int ndev) {
  if (ndev <= 0 || !devices) return QT_EINVAL;
  if (p == 0) return QT_EINVAL;
  if (ndev == 1 || m == 0 || s == 0 || n == 0 || (uint64_t)ndev > m)
    return qt_tprod_f64_host(a1, a2, b1, b2, c1, c2, m, n, s, p, devices[0]);
  NcclApi& api = qtb::nccl();
  if (!api.ok) return QT_ENCCL;
  qtb::DeviceGuard guard;

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
  std::vector<DevState> st(ndev);
  std::vector<uint64_t> r0(ndev), rows(ndev);
  for (int g = 0; g < ndev; ++g) {
    r0[g] = std::min<uint64_t>(m, g * slab);
    rows[g] = std::min<uint64_t>(m, r0[g] + slab) - r0[g];
  }
  const size_t bb = n * s * p * cx;
  struct Planes {
    double *A1, *A2, *B1, *B2, *C1, *C2;
  };
  auto planes = [&](int g) {
    const size_t ab = rows[g] * n * p * cx, cb = rows[g] * s * p * cx;
    char* base = (char*)st[g].buf;
    return Planes{(double*)base, (double*)(base + ab), (double*)(base + 2 * ab), (double*)(base + 2 * ab + bb),
                  (double*)(base + 2 * ab + 2 * bb), (double*)(base + 2 * ab + 2 * bb + cb)};
  };
  auto run_all = [&](auto fn) {
    std::vector<std::thread> th;
    for (int g = 0; g < ndev; ++g) th.emplace_back(fn, g);
    for (auto& t : th) t.join();
    int rc = QT_OK;
    for (int g = 0; g < ndev; ++g) rc = rc ? rc : st[g].rc;
    return rc;
  };

  // 1) per device: stream, buffers, its A slab (and on devices[0] all of B) in
  int rc = run_all([&](int g) {
    DevState& d = st[g];
    d.dev = devices[g];
    if (cudaSetDevice(d.dev) != cudaSuccess || cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking) != cudaSuccess) {
      d.rc = QT_ECUDA;
      return;
    }
    const size_t ab = rows[g] * n * p * cx, cb = rows[g] * s * p * cx;
    if (cudaMalloc((void**)&d.buf, 2 * ab + 2 * bb + 2 * cb) != cudaSuccess) {
      d.buf = nullptr;
      d.rc = QT_ENOMEM;
      return;
    }
    const Planes P = planes(g);
    const size_t spitch = m * n * cx, width = rows[g] * n * cx;
    if (cudaMemcpy2DAsync(P.A1, width, a1 + 2 * r0[g] * n, spitch, width, p, cudaMemcpyHostToDevice, d.st) ||
        cudaMemcpy2DAsync(P.A2, width, a2 + 2 * r0[g] * n, spitch, width, p, cudaMemcpyHostToDevice, d.st) ||
        (g == 0 && (cudaMemcpyAsync(P.B1, b1, bb, cudaMemcpyHostToDevice, d.st) ||
                    cudaMemcpyAsync(P.B2, b2, bb, cudaMemcpyHostToDevice, d.st))))
      d.rc = QT_ECUDA;
  });

  // 2) B from devices[0] to every device: one NCCL group, one broadcast per
  //    plane and device (stream-ordered after the uploads above)
  if (!rc) {
    if (api.GroupStart() != ncclSuccess) rc = QT_ENCCL;
    for (int g = 0; g < ndev && !rc; ++g) {
      const Planes P = planes(g);
      cudaSetDevice(st[g].dev);
      if (api.Broadcast(P.B1, P.B1, bb / sizeof(double), ncclFloat64, 0, comms[g], st[g].st) != ncclSuccess ||
          api.Broadcast(P.B2, P.B2, bb / sizeof(double), ncclFloat64, 0, comms[g], st[g].st) != ncclSuccess)
        rc = QT_ENCCL;
    }
    if (api.GroupEnd() != ncclSuccess && !rc) rc = QT_ENCCL;
  }

  // 3) per device: the whole pipeline on its slab, then its rows of C out
  if (!rc)
    rc = run_all([&](int g) {
      DevState& d = st[g];
      cudaSetDevice(d.dev);
      const Planes P = planes(g);
      int& r = d.rc;
      r = qt_tprod_f64_device(P.A1, P.A2, P.B1, P.B2, P.C1, P.C2, rows[g], n, s, p, d.st);
      if (r == QT_OK) {
        const size_t dpitch = m * s * cx, width = rows[g] * s * cx;
        if (cudaMemcpy2DAsync(c1 + 2 * r0[g] * s, dpitch, P.C1, width, width, p, cudaMemcpyDeviceToHost, d.st) ||
            cudaMemcpy2DAsync(c2 + 2 * r0[g] * s, dpitch, P.C2, width, width, p, cudaMemcpyDeviceToHost, d.st))
          r = QT_ECUDA;
      }
      if (cudaStreamSynchronize(d.st) != cudaSuccess && r == QT_OK) r = QT_ECUDA;
    });

  for (int g = 0; g < ndev; ++g) {
    DevState& d = st[g];
    if (!d.st) continue;
    cudaSetDevice(d.dev);
    cudaStreamSynchronize(d.st);
    if (d.buf) cudaFree(d.buf);
    cudaStreamDestroy(d.st);
  }
  return rc;
}

}  // extern "C"
