// qt_rank.cu — per-rank multi-GPU drivers of the T-product (one process per
// GPU, launched by torchrun; the C++ owns the NCCL communicator, the
// schedule and every transfer; Python only starts the processes and hands
// the 128-byte NCCL id around).  The reference is single-process
// (tproduct.cpp:75-111; "distributed benchmarking" is a non-goal),
// so both decompositions are this repo's:
//
// rows (the north_star split, qt_rank_tprod_rows): rank r owns a contiguous
//   slab of rows of A and C (row i of C needs only row i of A and all of B);
//   B is broadcast once from the root with ncclBroadcast (one grouped call per
//   CD plane), then each rank runs the whole single-GPU pipeline on its slab.
//   Bitwise identical to the one-GPU product (same per-element arithmetic).
//   Replicates the B-side work (K1 of B; for the int8 stage 2 its column
//   scalings and residues) on every rank.
//
// freq (frequency-parallel, qt_rank_freq_*): nothing is replicated.  K1 and K3
//   are independent per tube, stage 2 per frequency pair (k, p - k):
//     K1  rank r transforms rows [a0, a1) of A and rows [b0, b1) of B;
//     ->  every (frequency slot t, rows) piece goes to the owner of slot t
//         (the contiguous slot range ranges[j] of rank j);
//     K2  rank j runs stage 2 of its slots for all m x s (int8 on compact
//         slot tensors, qt_int8_slots_*, or fp64 DMMA on them);
//     ->  the Ĉ pieces go back to the row owners;
//     K3  rank r inverse-transforms its rows of C.
//   Every piece is a contiguous block of both the sender's and the receiver's
//   buffer, so each exchange is one NCCL group of send/recv pairs straight
//   from and into the stage buffers (the rank's own pieces are device
//   copies).  Each slot is evaluated exactly as in the single-GPU product (its
//   scalings and balancing depend on its own data only): bitwise identical.
//
// Partition rules (identical to paper_2212_14318_b200/shard.py, tested):
//   row_slab(m, G, r) = [min(m, r ceil(m/G)), min(m, (r+1) ceil(m/G)));
//   slot ranges: boundaries at round-half-even(k p / G), moved off an odd
//   slot below 2 ((p - 1) / 2) (a pair is never split).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/qtensor_b200.h"
#include "qt_internal.cuh"
#include "qt_nccl.h"

namespace {

using qtb::NcclApi;

struct Comm {
  ncclComm_t nc = nullptr;
  int rank = 0, world = 1, device = 0;
};

void row_slab(uint64_t m, int world, int rank, uint64_t* lo, uint64_t* hi) {
  const uint64_t slab = (m + world - 1) / world;
  *lo = std::min<uint64_t>(m, (uint64_t)rank * slab);
  *hi = std::min<uint64_t>(m, *lo + slab);
}

std::vector<std::pair<int, int>> slot_ranges(uint64_t p, int world) {
  const int64_t pair_end = 2 * (((int64_t)p - 1) / 2);
  std::vector<int64_t> b{0};
  for (int k = 1; k < world; ++k) {
    const double ideal = (double)k * (double)p / (double)world;
    int64_t x = (int64_t)std::nearbyint(ideal);  // round half to even, as Python's round()
    if ((x & 1) && x < pair_end) x = ideal < (double)x ? x - 1 : x + 1;
    b.push_back(std::min<int64_t>((int64_t)p, std::max<int64_t>(b.back(), x)));
  }
  b.push_back((int64_t)p);
  std::vector<std::pair<int, int>> out;
  for (int k = 0; k < world; ++k) out.emplace_back((int)b[k], (int)b[k + 1]);
  return out;
}

// One frequency-parallel rank: partition, buffers and the piece schedule.
struct FreqRank {
  Comm* comm = nullptr;  // nullptr: a lockstep-emulated rank (qt_rank_freq_emulate)
  int rank = 0, world = 1, device = 0;
  uint64_t m = 0, n = 0, s = 0, p = 0;
  std::vector<std::pair<uint64_t, uint64_t>> arows, brows;  // row slabs of A/C and of B, per rank
  std::vector<std::pair<int, int>> ranges;                   // slot range per rank
  uint64_t a0 = 0, a1 = 0, b0 = 0, b1 = 0;
  int t0 = 0, t1 = 0;
  int algo = 0;
  // device buffers (each two CD planes, complex128):
  double2* ah = nullptr;  // (2, p, rows_a, n) K1 output, frequency-major
  double2* bh = nullptr;  // (2, p, rows_b, s)
  double2* ac = nullptr;  // (2, ns, m, n) compact slot tensors
  double2* bc = nullptr;  // (2, ns, n, s)
  double2* cc = nullptr;  // (2, ns, m, s)
  int* nonfinite = nullptr;
  uint64_t* sig = nullptr;  // kMaxWorld barrier slots (fused exchange), in buf so peers can address them
  void* buf = nullptr;
  // fused exchange (qt_rank_freq_set_peers): the peers' buffers mapped here,
  // device row tables of the routed transforms, the peers' signal slots
  bool fused = false;
  std::vector<void*> peer_buf;      // peer j's buffer as seen from this device (own: buf)
  std::vector<bool> peer_opened;    // opened through cudaIpcOpenMemHandle (closed at destroy)
  void* tables = nullptr;           // device: [A 2p][B 2p][C 2p] pointers, then world signal pointers
  uint64_t epoch = 0;

  uint64_t ra() const { return a1 - a0; }
  uint64_t rb() const { return b1 - b0; }
  int ns() const { return t1 - t0; }
};

// A piece of an exchange, semantically: the (slot, plane) block of rows
// [r0, r0 + rows) of the part's (m or n)-row dimension, to / from `peer`.
struct Sem {
  int peer, slot, plane;
  uint64_t r0, rows;
};
struct Piece {
  int peer;
  char* ptr;  // this side's buffer
  size_t bytes;
};

// The exchange schedules.  Both sides enumerate (slot, plane) per peer in the
// same order, so NCCL's in-order matching of the sends / receives between a
// pair of ranks lines every piece up (and the emulation pairs them the same
// way).  A / B: every rank sends its rows of each frequency slot to the slot's
// owner, which stores them at those rows of its compact slot tensor; C: the
// slot owner sends each row owner its rows of every owned slot.
enum class Part { A = 0, B = 1, C = 2 };
void schedule(const FreqRank& R, Part part, bool send, std::vector<Sem>& out) {
  out.clear();
  const bool from_rows = (part == Part::C) ? !send : send;  // this side holds rows of every slot
  if (from_rows) {
    const uint64_t r0 = part == Part::B ? R.b0 : R.a0, rows = part == Part::B ? R.rb() : R.ra();
    if (!rows) return;
    for (int j = 0; j < R.world; ++j)
      for (int t = R.ranges[j].first; t < R.ranges[j].second; ++t)
        for (int pl = 0; pl < 2; ++pl) out.push_back({j, t, pl, r0, rows});
  } else {  // this side owns slots [t0, t1): every row owner's block of them
    const auto& rows = part == Part::B ? R.brows : R.arows;
    for (int i = 0; i < R.world; ++i) {
      if (rows[i].second == rows[i].first) continue;
      for (int t = R.t0; t < R.t1; ++t)
        for (int pl = 0; pl < 2; ++pl) out.push_back({i, t, pl, rows[i].first, rows[i].second - rows[i].first});
    }
  }
}
// Device address of a piece on this side: the frequency-major K1 output /
// K3 input (rows of all p frequencies) or the compact slot tensors.
void pieces(const FreqRank& R, Part part, bool send, double2* c1, double2* c2, std::vector<Piece>& out) {
  std::vector<Sem> sem;
  schedule(R, part, send, sem);
  out.clear();
  const size_t cx = sizeof(double2);
  const bool from_rows = (part == Part::C) ? !send : send;
  const uint64_t width = part == Part::A ? R.n : R.s;
  for (const Sem& x : sem) {
    double2* ptr;
    if (from_rows) {
      const uint64_t k = (uint64_t)qtb::slot_frequency(x.slot, (int)R.p);
      if (part == Part::A) ptr = R.ah + (x.plane * R.p + k) * R.ra() * R.n;
      else if (part == Part::B) ptr = R.bh + (x.plane * R.p + k) * R.rb() * R.s;
      else ptr = (x.plane ? c2 : c1) + k * R.ra() * R.s;
    } else {
      double2* base = part == Part::A ? R.ac : part == Part::B ? R.bc : R.cc;
      const uint64_t height = part == Part::B ? R.n : R.m;
      ptr = base + ((x.plane * (uint64_t)R.ns() + (x.slot - R.t0)) * height + x.r0) * width;
    }
    out.push_back({x.peer, (char*)ptr, x.rows * width * cx});
  }
}

void partition(FreqRank& R, uint64_t m, uint64_t n, uint64_t s, uint64_t p, int rank, int world) {
  R.m = m;
  R.n = n;
  R.s = s;
  R.p = p;
  R.rank = rank;
  R.world = world;
  R.arows.clear();
  R.brows.clear();
  for (int r = 0; r < world; ++r) {
    uint64_t lo, hi;
    row_slab(m, world, r, &lo, &hi);
    R.arows.emplace_back(lo, hi);
    row_slab(n, world, r, &lo, &hi);
    R.brows.emplace_back(lo, hi);
  }
  R.ranges = slot_ranges(p, world);
  R.a0 = R.arows[rank].first;
  R.a1 = R.arows[rank].second;
  R.b0 = R.brows[rank].first;
  R.b1 = R.brows[rank].second;
  R.t0 = R.ranges[rank].first;
  R.t1 = R.ranges[rank].second;
}

constexpr int kMaxWorld = 64;

// Byte offsets of one rank's stage buffer (the same rule on every rank, so a
// rank can address a peer's compact slot tensors and signal slots).
struct Layout {
  size_t ah, bh, ac, bc, cc, nonfinite, sig, total;
};
Layout layout(const FreqRank& R) {
  const size_t cx = sizeof(double2);
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  Layout L;
  L.ah = 0;
  L.bh = L.ah + al(2 * R.p * R.ra() * R.n * cx);
  L.ac = L.bh + al(2 * R.p * R.rb() * R.s * cx);
  L.bc = L.ac + al(2 * (size_t)R.ns() * R.m * R.n * cx);
  L.cc = L.bc + al(2 * (size_t)R.ns() * R.n * R.s * cx);
  L.nonfinite = L.cc + al(2 * (size_t)R.ns() * R.m * R.s * cx);
  L.sig = L.nonfinite + 256;
  L.total = L.sig + kMaxWorld * sizeof(uint64_t);
  return L;
}

int setup(FreqRank& R, uint64_t m, uint64_t n, uint64_t s, uint64_t p, int rank, int world) {
  partition(R, m, n, s, p, rank, world);
  R.algo = qt_gemm_algo(m, n, s, p);
  const Layout L = layout(R);
  if (cudaMalloc(&R.buf, L.total) != cudaSuccess) {  // cudaMalloc: exportable through CUDA IPC
    cudaGetLastError();
    R.buf = nullptr;
    return QT_ENOMEM;
  }
  char* b = (char*)R.buf;
  R.ah = (double2*)(b + L.ah);
  R.bh = (double2*)(b + L.bh);
  R.ac = (double2*)(b + L.ac);
  R.bc = (double2*)(b + L.bc);
  R.cc = (double2*)(b + L.cc);
  R.nonfinite = (int*)(b + L.nonfinite);
  R.sig = (uint64_t*)(b + L.sig);
  return cudaMemset(b + L.nonfinite, 0, L.total - L.nonfinite) == cudaSuccess ? QT_OK : QT_ECUDA;
}

// ------------------------------------------------- fused (peer memory) exchange
// With every rank's stage buffer mapped (CUDA IPC over NVLink), the exchange
// needs no messages: K1 stores each frequency row of its rows of Â / B̂
// straight into the slot owner's compact tensor (qt_qfft3_conj_f64_device_routed:
// the last Stockham stage's store address comes from a per-(plane, frequency)
// row table), and K3 loads its rows of every frequency of Ĉ straight from the
// owners (qt_qifft3_conj_f64_device_routed).  The pieces land exactly where
// the NCCL exchange puts them, so the result is bitwise the same.  A device
// barrier (every rank release-stores an epoch into each peer's signal slot
// for it, then acquire-spins on its own slots) orders the phases: after K1
// (the pieces are in place) and after stage 2 (every Ĉ is complete and no rank
// still reads the Â / B̂ the next step's K1 overwrites); the next step's first
// barrier orders this step's K3 loads before any rank's next stage 2 rewrites
// its Ĉ.  Only for lengths whose transform is one launch (qt_fft_routable).
__global__ void peer_barrier_kernel(uint64_t* const* sig, int rank, int world, uint64_t epoch) {
  const int t = threadIdx.x;
  __threadfence_system();  // this rank's earlier peer stores before the signal
  if (t < world) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(sig[t] + rank), "l"(epoch) : "memory");
  if (t < world) {
    const uint64_t* mine = sig[rank] + t;
    uint64_t v = 0;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    } while (v < epoch);
  }
  __syncthreads();
  __threadfence_system();
}

// Row tables of rank R for the peers' buffers `bases` (each peer's own layout).
void build_tables(const FreqRank& R, const std::vector<char*>& bases, std::vector<void*>& tab) {
  const uint64_t p = R.p;
  tab.assign(6 * p + R.world, nullptr);
  std::vector<Layout> Ls(R.world);
  std::vector<FreqRank> P(R.world);
  for (int j = 0; j < R.world; ++j) {
    partition(P[j], R.m, R.n, R.s, R.p, j, R.world);
    Ls[j] = layout(P[j]);
  }
  std::vector<int> owner(p);
  for (int j = 0; j < R.world; ++j)
    for (int t = R.ranges[j].first; t < R.ranges[j].second; ++t) owner[t] = j;
  const size_t cx = sizeof(double2);
  for (uint64_t t = 0; t < p; ++t) {
    const uint64_t k = (uint64_t)qtb::slot_frequency((int)t, (int)p);
    const int j = owner[t];
    const uint64_t nsj = (uint64_t)P[j].ns(), tl = t - (uint64_t)P[j].t0;
    for (int pl = 0; pl < 2; ++pl) {
      tab[pl * p + k] = bases[j] + Ls[j].ac + (((pl * nsj + tl) * R.m + R.a0) * R.n) * cx;          // K1(A) stores
      tab[2 * p + pl * p + k] = bases[j] + Ls[j].bc + (((pl * nsj + tl) * R.n + R.b0) * R.s) * cx;  // K1(B) stores
      tab[4 * p + pl * p + k] = bases[j] + Ls[j].cc + (((pl * nsj + tl) * R.m + R.a0) * R.s) * cx;  // K3 loads
    }
  }
  for (int j = 0; j < R.world; ++j) tab[6 * p + j] = bases[j] + Ls[j].sig;
}

int upload_tables(FreqRank& R, const std::vector<void*>& tab) {
  if (!R.tables && cudaMalloc(&R.tables, tab.size() * sizeof(void*)) != cudaSuccess) return QT_ENOMEM;
  return cudaMemcpy(R.tables, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice) == cudaSuccess
             ? QT_OK
             : QT_ECUDA;
}

int k1_routed(FreqRank& R, const double* a1, const double* a2, const double* b1, const double* b2, cudaStream_t st) {
  double** T = (double**)R.tables;
  int rc = QT_OK;
  if (R.rb()) rc = qt_qfft3_conj_f64_device_routed(b1, b2, T + 2 * R.p, T + 3 * R.p, R.rb(), R.s, R.p, st);
  if (!rc && R.ra()) rc = qt_qfft3_conj_f64_device_routed(a1, a2, T, T + R.p, R.ra(), R.n, R.p, st);
  return rc;
}

int k3_routed(FreqRank& R, double* c1, double* c2, cudaStream_t st) {
  if (!R.ra()) return QT_OK;
  const double* const* T = (const double* const*)R.tables;
  return qt_qifft3_conj_f64_device_routed(T + 4 * R.p, T + 5 * R.p, c1, c2, R.ra(), R.s, R.p, st);
}

int barrier(FreqRank& R, cudaStream_t st) {
  if (R.world == 1) return QT_OK;
  ++R.epoch;
  peer_barrier_kernel<<<1, 64, 0, st>>>((uint64_t* const*)((void**)R.tables + 6 * R.p), R.rank, R.world, R.epoch);
  return cudaGetLastError() == cudaSuccess ? QT_OK : QT_ECUDA;
}

int k1(FreqRank& R, const double* a1, const double* a2, const double* b1, const double* b2, cudaStream_t st) {
  int rc = QT_OK;
  if (R.rb())
    rc = qt_qfft3_conj_f64_device(b1, b2, (double*)R.bh, (double*)(R.bh + R.p * R.rb() * R.s), R.rb(), R.s, R.p, st);
  if (!rc && R.ra())
    rc = qt_qfft3_conj_f64_device(a1, a2, (double*)R.ah, (double*)(R.ah + R.p * R.ra() * R.n), R.ra(), R.n, R.p, st);
  return rc;
}

int stage2(FreqRank& R, cudaStream_t st) {
  if (!R.ns() || !R.m || !R.s) return QT_OK;
  const uint64_t ns = R.ns();
  double* ac1 = (double*)R.ac;
  double* ac2 = (double*)(R.ac + ns * R.m * R.n);
  double* bc1 = (double*)R.bc;
  double* bc2 = (double*)(R.bc + ns * R.n * R.s);
  double* cc1 = (double*)R.cc;
  double* cc2 = (double*)(R.cc + ns * R.m * R.s);
  if (R.algo == QT_GEMM_INT8_EXACT) {
    void* h = nullptr;
    int rc = qt_int8_slots_create(bc1, bc2, R.n, R.s, R.p, R.t0, (int)ns, R.nonfinite, st, &h);
    if (rc) return rc;
    rc = qt_int8_slots_multiply(h, ac1, ac2, R.m, cc1, cc2, st);
    const int dr = qt_int8_slots_destroy(h, st);
    return rc ? rc : dr;
  }
  const cudaError_t e = qtb::dmma_spectral_gemm_slots((const double2*)ac1, (const double2*)ac2, (const double2*)bc1,
                                                      (const double2*)bc2, (double2*)cc1, (double2*)cc2, R.m, R.n,
                                                      R.s, R.p, R.t0, (int)ns, st, nullptr);
  return e == cudaSuccess ? QT_OK : QT_ECUDA;
}

// One exchange over NCCL: local pieces as device copies, the rest as one group
// of send/recv pairs on `st`.
int exchange(FreqRank& R, const std::vector<Piece>& snd, const std::vector<Piece>& rcv, cudaStream_t st) {
  std::vector<const Piece*> ls, lr;
  for (const Piece& x : snd)
    if (x.peer == R.rank) ls.push_back(&x);
  for (const Piece& x : rcv)
    if (x.peer == R.rank) lr.push_back(&x);
  if (ls.size() != lr.size()) return QT_EINVAL;
  for (size_t i = 0; i < ls.size(); ++i) {
    if (ls[i]->bytes != lr[i]->bytes) return QT_EINVAL;
    if (cudaMemcpyAsync(lr[i]->ptr, ls[i]->ptr, ls[i]->bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return QT_ECUDA;
  }
  if (R.world == 1) return QT_OK;
  NcclApi& api = qtb::nccl();
  if (api.GroupStart() != ncclSuccess) return QT_ENCCL;
  int rc = QT_OK;
  for (const Piece& x : snd)
    if (x.peer != R.rank && api.Send(x.ptr, x.bytes, ncclUint8, x.peer, R.comm->nc, st) != ncclSuccess) rc = QT_ENCCL;
  for (const Piece& x : rcv)
    if (x.peer != R.rank && api.Recv(x.ptr, x.bytes, ncclUint8, x.peer, R.comm->nc, st) != ncclSuccess) rc = QT_ENCCL;
  if (api.GroupEnd() != ncclSuccess) rc = QT_ENCCL;
  return rc;
}

int k3(FreqRank& R, double* c1, double* c2, cudaStream_t st) {
  if (!R.ra()) return QT_OK;
  return qt_qifft3_conj_f64_device(c1, c2, c1, c2, R.ra(), R.s, R.p, st);
}

}  // namespace

extern "C" {

int qt_comm_unique_id(void* id) {
  NcclApi& api = qtb::nccl();
  if (!id) return QT_EINVAL;
  if (!api.ok) return QT_ENCCL;
  ncclUniqueId u;
  if (api.GetUniqueId(&u) != ncclSuccess) return QT_ENCCL;
  memcpy(id, &u, sizeof(u));
  return QT_OK;
}

int qt_comm_init(const void* id, int rank, int world, int device, void** comm) {
  if (!id || !comm || world <= 0 || rank < 0 || rank >= world) return QT_EINVAL;
  *comm = nullptr;
  NcclApi& api = qtb::nccl();
  if (!api.ok) return QT_ENCCL;
  qtb::DeviceGuard guard;
  if (cudaSetDevice(device) != cudaSuccess) return QT_ECUDA;
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  Comm* c = new Comm;
  c->rank = rank;
  c->world = world;
  c->device = device;
  if (api.CommInitRank(&c->nc, world, u, rank) != ncclSuccess) {
    delete c;
    return QT_ENCCL;
  }
  int ver = 0;
  if (api.GetVersion) api.GetVersion(&ver);
  fprintf(stderr, "[qtensor_b200] NCCL %d.%d.%d communicator: rank %d of %d on cuda:%d\n", ver / 10000,
          (ver / 100) % 100, ver % 100, rank, world, device);
  *comm = c;
  return QT_OK;
}

int qt_comm_destroy(void* comm) {
  Comm* c = (Comm*)comm;
  if (!c) return QT_OK;
  NcclApi& api = qtb::nccl();
  const ncclResult_t r = api.ok ? api.CommDestroy(c->nc) : ncclSuccess;
  delete c;
  return r == ncclSuccess ? QT_OK : QT_ENCCL;
}

int qt_rank_partition(uint64_t m, uint64_t n, uint64_t p, int world, int rank, uint64_t* out6) {
  if (!out6 || world <= 0 || rank < 0 || rank >= world || p == 0) return QT_EINVAL;
  row_slab(m, world, rank, &out6[0], &out6[1]);
  row_slab(n, world, rank, &out6[2], &out6[3]);
  const auto r = slot_ranges(p, world);
  out6[4] = (uint64_t)r[rank].first;
  out6[5] = (uint64_t)r[rank].second;
  return QT_OK;
}

int qt_rank_freq_schedule(uint64_t m, uint64_t n, uint64_t s, uint64_t p, int world, int rank, int part, int send,
                          int64_t* out5, uint64_t cap, uint64_t* count) {
  if (world <= 0 || rank < 0 || rank >= world || p == 0 || part < 0 || part > 2 || !count) return QT_EINVAL;
  FreqRank R;
  partition(R, m, n, s, p, rank, world);
  std::vector<Sem> sem;
  schedule(R, (Part)part, send != 0, sem);
  *count = sem.size();
  if (!out5) return QT_OK;
  if (cap < sem.size()) return QT_EINVAL;
  for (size_t i = 0; i < sem.size(); ++i) {
    out5[5 * i + 0] = sem[i].peer;
    out5[5 * i + 1] = sem[i].slot;
    out5[5 * i + 2] = sem[i].plane;
    out5[5 * i + 3] = (int64_t)sem[i].r0;
    out5[5 * i + 4] = (int64_t)sem[i].rows;
  }
  return QT_OK;
}

int qt_rank_tprod_rows(void* comm, const double* a1, const double* a2, double* b1, double* b2, double* c1,
                       double* c2, uint64_t rows, uint64_t n, uint64_t s, uint64_t p, int root, void* stream) {
  Comm* c = (Comm*)comm;
  if (!c || root < 0 || root >= c->world || p == 0) return QT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (c->world > 1 && n && s) {
    NcclApi& api = qtb::nccl();
    const size_t count = 2 * n * s * p;  // doubles per plane
    if (api.GroupStart() != ncclSuccess) return QT_ENCCL;
    int rc = QT_OK;
    if (api.Broadcast(b1, b1, count, ncclFloat64, root, c->nc, st) != ncclSuccess ||
        api.Broadcast(b2, b2, count, ncclFloat64, root, c->nc, st) != ncclSuccess)
      rc = QT_ENCCL;
    if (api.GroupEnd() != ncclSuccess || rc) return QT_ENCCL;
  }
  if (!rows) return QT_OK;
  return qt_tprod_f64_device(a1, a2, b1, b2, c1, c2, rows, n, s, p, stream);
}

int qt_rank_freq_create(void* comm, uint64_t m, uint64_t n, uint64_t s, uint64_t p, void** plan) {
  Comm* c = (Comm*)comm;
  if (!c || !plan || p == 0 || p > 65534) return QT_EINVAL;
  *plan = nullptr;
  qtb::DeviceGuard guard;
  if (cudaSetDevice(c->device) != cudaSuccess) return QT_ECUDA;
  FreqRank* R = new FreqRank;
  R->comm = c;
  R->device = c->device;
  const int rc = setup(*R, m, n, s, p, c->rank, c->world);
  if (rc) {
    if (R->buf) cudaFree(R->buf);
    delete R;
    return rc;
  }
  *plan = R;
  return QT_OK;
}

int qt_rank_freq_step(void* plan, const double* a1, const double* a2, const double* b1, const double* b2, double* c1,
                      double* c2, void* stream) {
  FreqRank* R = (FreqRank*)plan;
  if (!R) return QT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (R->fused) {  // the exchange fused into K1's stores / K3's loads over peer memory
    int rc = k1_routed(*R, a1, a2, b1, b2, st);
    if (!rc) rc = barrier(*R, st);
    if (!rc) rc = stage2(*R, st);
    if (!rc) rc = barrier(*R, st);
    if (!rc) rc = k3_routed(*R, c1, c2, st);
    return rc;
  }
  if (!R->comm && R->world > 1) return QT_EINVAL;  // an IPC plan before qt_rank_freq_set_peers
  std::vector<Piece> snd, rcv;
  int rc = k1(*R, a1, a2, b1, b2, st);
  if (!rc) {
    pieces(*R, Part::B, true, nullptr, nullptr, snd);
    pieces(*R, Part::B, false, nullptr, nullptr, rcv);
    rc = exchange(*R, snd, rcv, st);
  }
  if (!rc) {
    pieces(*R, Part::A, true, nullptr, nullptr, snd);
    pieces(*R, Part::A, false, nullptr, nullptr, rcv);
    rc = exchange(*R, snd, rcv, st);
  }
  if (!rc) rc = stage2(*R, st);
  if (!rc) {
    pieces(*R, Part::C, true, nullptr, nullptr, snd);
    pieces(*R, Part::C, false, (double2*)c1, (double2*)c2, rcv);
    rc = exchange(*R, snd, rcv, st);
  }
  if (!rc) rc = k3(*R, c1, c2, st);
  return rc;
}

// A frequency-parallel plan without an NCCL communicator: its exchange goes
// through peer memory only (qt_rank_freq_ipc_handle / qt_rank_freq_set_peers).
int qt_rank_freq_create_ipc(int rank, int world, int device, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                            void** plan) {
  if (!plan || world <= 0 || world > kMaxWorld || rank < 0 || rank >= world || p == 0 || p > 65534) return QT_EINVAL;
  *plan = nullptr;
  qtb::DeviceGuard guard;
  if (cudaSetDevice(device) != cudaSuccess) return QT_ECUDA;
  FreqRank* R = new FreqRank;
  R->device = device;
  const int rc = setup(*R, m, n, s, p, rank, world);
  if (rc) {
    if (R->buf) cudaFree(R->buf);
    delete R;
    return rc;
  }
  *plan = R;
  return QT_OK;
}

int qt_rank_freq_ipc_handle(void* plan, void* out64) {
  FreqRank* R = (FreqRank*)plan;
  if (!R || !out64) return QT_EINVAL;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, R->buf) != cudaSuccess) {
    cudaGetLastError();
    return QT_ECUDA;
  }
  memcpy(out64, &h, sizeof(h));
  return QT_OK;
}

// handles: world x 64 bytes (every rank's qt_rank_freq_ipc_handle, in rank
// order).  Maps the peers' stage buffers, builds the routed transforms' row
// tables and switches the plan to the fused exchange (lengths whose transform
// is one launch; others keep the NCCL exchange, or fail for an IPC plan).
int qt_rank_freq_set_peers(void* plan, const void* handles) {
  FreqRank* R = (FreqRank*)plan;
  if (!R || !handles || R->world > kMaxWorld) return QT_EINVAL;  // (kMaxWorld signal slots per rank)
  if (!qt_fft_routable(R->p)) return R->comm ? QT_OK : QT_EINVAL;
  qtb::DeviceGuard guard;
  if (cudaSetDevice(R->device) != cudaSuccess) return QT_ECUDA;
  R->peer_buf.assign(R->world, nullptr);
  R->peer_opened.assign(R->world, false);
  std::vector<char*> bases(R->world);
  for (int j = 0; j < R->world; ++j) {
    if (j == R->rank) {
      R->peer_buf[j] = R->buf;
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, (const char*)handles + 64 * (size_t)j, sizeof(h));
      if (cudaIpcOpenMemHandle(&R->peer_buf[j], h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return QT_ECUDA;
      }
      R->peer_opened[j] = true;
    }
    bases[j] = (char*)R->peer_buf[j];
  }
  std::vector<void*> tab;
  build_tables(*R, bases, tab);
  const int rc = upload_tables(*R, tab);
  if (!rc) R->fused = true;
  return rc;
}

// One phase of the fused step without the device barriers, for callers that
// order the ranks themselves (the two-process test on one GPU: no kernel may
// wait on another process's kernel there): 0 = K1 with routed stores, 1 = stage
// 2 of the rank's slots, 2 = K3 with routed loads.
int qt_rank_freq_phase(void* plan, int phase, const double* a1, const double* a2, const double* b1, const double* b2,
                       double* c1, double* c2, void* stream) {
  FreqRank* R = (FreqRank*)plan;
  if (!R || !R->fused || phase < 0 || phase > 2) return QT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (phase == 0) return k1_routed(*R, a1, a2, b1, b2, st);
  if (phase == 1) return stage2(*R, st);
  return k3_routed(*R, c1, c2, st);
}

int qt_rank_freq_nonfinite(void* plan, int* out) {
  FreqRank* R = (FreqRank*)plan;
  if (!R || !out) return QT_EINVAL;
  return cudaMemcpy(out, R->nonfinite, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess ? QT_OK : QT_ECUDA;
}

int qt_rank_freq_destroy(void* plan) {
  FreqRank* R = (FreqRank*)plan;
  if (!R) return QT_OK;
  qtb::DeviceGuard guard;
  cudaSetDevice(R->device);
  for (size_t j = 0; j < R->peer_opened.size(); ++j)
    if (R->peer_opened[j]) cudaIpcCloseMemHandle(R->peer_buf[j]);
  if (R->tables) cudaFree(R->tables);
  const cudaError_t e = R->buf ? cudaFree(R->buf) : cudaSuccess;
  delete R;
  return e == cudaSuccess ? QT_OK : QT_ECUDA;
}

// G frequency-parallel ranks emulated in lockstep on the current device, every
// exchanged piece a device copy between the ranks' buffers (the same
// schedule the NCCL exchange follows): the single-GPU check of the
// decomposition.  a/b/c: whole device tensors (two planes each, slice-major);
// each rank reads its rows of A and B and writes its rows of C.
int qt_rank_freq_emulate(int world, int fused, const double* a1, const double* a2, const double* b1, const double* b2,
                         double* c1, double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, void* stream) {
  if (world <= 0 || world > kMaxWorld || p == 0 || p > 65534) return QT_EINVAL;
  if (fused && !qt_fft_routable(p)) return QT_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t cx = sizeof(double2);
  std::vector<FreqRank> R(world);
  std::vector<void*> abuf(world, nullptr), cbuf(world, nullptr);
  int rc = QT_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  for (int r = 0; r < world && !rc; ++r) {
    R[r].device = dev;
    rc = setup(R[r], m, n, s, p, r, world);
  }
  // per-rank input slabs (rows of A, B) and output slabs (rows of C), packed
  for (int r = 0; r < world && !rc; ++r) {
    const size_t ab = 2 * p * R[r].ra() * n * cx + 2 * p * R[r].rb() * s * cx, cb = 2 * p * R[r].ra() * s * cx;
    if (cudaMalloc(&abuf[r], ab + 16) != cudaSuccess || cudaMalloc(&cbuf[r], cb + 16) != cudaSuccess) rc = QT_ENOMEM;
    if (rc) break;
    double2* A = (double2*)abuf[r];
    double2* B = A + 2 * p * R[r].ra() * n;
    for (int pl = 0; pl < 2 && !rc; ++pl) {
      const double* as = pl ? a2 : a1;
      const double* bs = pl ? b2 : b1;
      if (R[r].ra() &&
          cudaMemcpy2DAsync(A + pl * p * R[r].ra() * n, R[r].ra() * n * cx, as + 2 * R[r].a0 * n, m * n * cx,
                            R[r].ra() * n * cx, p, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        rc = QT_ECUDA;
      if (R[r].rb() &&
          cudaMemcpy2DAsync(B + pl * p * R[r].rb() * s, R[r].rb() * s * cx, bs + 2 * R[r].b0 * s, n * s * cx,
                            R[r].rb() * s * cx, p, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        rc = QT_ECUDA;
    }
  }
  auto route = [&](Part part) {
    std::vector<std::vector<Piece>> snd(world), rcv(world);
    for (int r = 0; r < world; ++r) {
      double2* C = (double2*)cbuf[r];
      pieces(R[r], part, true, nullptr, nullptr, snd[r]);
      pieces(R[r], part, false, C, C + p * R[r].ra() * s, rcv[r]);
    }
    for (int dst = 0; dst < world; ++dst)
      for (int src = 0; src < world; ++src) {
        std::vector<const Piece*> from, into;
        for (const Piece& x : snd[src])
          if (x.peer == dst) from.push_back(&x);
        for (const Piece& x : rcv[dst])
          if (x.peer == src) into.push_back(&x);
        if (from.size() != into.size()) return QT_EINVAL;
        for (size_t i = 0; i < from.size(); ++i) {
          if (from[i]->bytes != into[i]->bytes) return QT_EINVAL;
          if (cudaMemcpyAsync(into[i]->ptr, from[i]->ptr, from[i]->bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return QT_ECUDA;
        }
      }
    return QT_OK;
  };
  if (fused && !rc) {  // every rank's row tables point into the other emulated ranks' buffers
    std::vector<char*> bases(world);
    for (int r = 0; r < world; ++r) bases[r] = (char*)R[r].buf;
    for (int r = 0; r < world && !rc; ++r) {
      std::vector<void*> tab;
      build_tables(R[r], bases, tab);
      rc = upload_tables(R[r], tab);
    }
  }
  for (int r = 0; r < world && !rc; ++r) {
    double2* A = (double2*)abuf[r];
    double2* B = A + 2 * p * R[r].ra() * n;
    const double *A1 = (double*)A, *A2 = (double*)(A + p * R[r].ra() * n);
    const double *B1 = (double*)B, *B2 = (double*)(B + p * R[r].rb() * s);
    rc = fused ? k1_routed(R[r], A1, A2, B1, B2, st) : k1(R[r], A1, A2, B1, B2, st);
  }
  if (!rc && !fused) rc = route(Part::B);
  if (!rc && !fused) rc = route(Part::A);
  for (int r = 0; r < world && !rc; ++r) rc = stage2(R[r], st);
  if (!rc && !fused) rc = route(Part::C);
  for (int r = 0; r < world && !rc; ++r) {
    double2* C = (double2*)cbuf[r];
    rc = fused ? k3_routed(R[r], (double*)C, (double*)(C + p * R[r].ra() * s), st)
               : k3(R[r], (double*)C, (double*)(C + p * R[r].ra() * s), st);
    for (int pl = 0; pl < 2 && !rc && R[r].ra(); ++pl)
      if (cudaMemcpy2DAsync((pl ? c2 : c1) + 2 * R[r].a0 * s, m * s * cx, C + pl * p * R[r].ra() * s,
                            R[r].ra() * s * cx, R[r].ra() * s * cx, p, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        rc = QT_ECUDA;
  }
  cudaStreamSynchronize(st);
  for (int r = 0; r < world; ++r) {
    if (R[r].tables) cudaFree(R[r].tables);
    if (R[r].buf) cudaFree(R[r].buf);
    if (abuf[r]) cudaFree(abuf[r]);
    if (cbuf[r]) cudaFree(cbuf[r]);
  }
  return rc;
}

}  // extern "C"
