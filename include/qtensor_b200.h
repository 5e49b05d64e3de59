/*
 * qtensor_b200.h — C-ABI of the B200-native quaternion-tensor T-product.
 *
 * This is the drop-in boundary for the reference's hot path
 *   qtensor::tprod_fast(a, b[, ws])      /root/reference/proj/include/qtensor/tproduct.hpp:45-46
 *                                        /root/reference/proj/src/tproduct.cpp:75-111
 * and for the two tube transforms it is built from
 *   qtensor::qfft3_conj(q)               transform.hpp:56-60, transform.cpp:151-158
 *   qtensor::qifft3_conj(qhat)           transform.hpp:62-64, transform.cpp:160-167
 *
 * Only plain pointers, sizes and status codes cross this boundary (no C++ or
 * torch types).  A quaternion tensor Q = t1 + t2*j of shape m x n x p is passed
 * as its two Cayley-Dickson planes t1, t2 (algebra.hpp:61-68), each an array of
 * m*n*p complex doubles stored as interleaved (re, im) pairs, slice-major:
 *     element (i, j, r) lives at complex index (r*m + i)*n + j
 * which is exactly CdTensor3's layout (transform.hpp:35-37), so
 * reinterpret_cast<const double*>(t.t1.data()) can be handed over unchanged.
 *
 * Error behaviour mirrors the reference: a shape the reference rejects with
 * std::invalid_argument returns QT_EINVAL (p == 0, transform.cpp:152); CUDA
 * failures return QT_ECUDA, allocation failures QT_ENOMEM, NCCL failures
 * QT_ENCCL.  qt_last_error() returns the calling thread's last message.
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point fails with QT_ENODEV.
 *
 * All compute entry points are reentrant (per-call stream-ordered workspace,
 * per-thread error state) and deterministic: identical inputs give bitwise
 * identical outputs, independent of the number of GPUs the rows are sharded
 * over.
 */
#ifndef QTENSOR_B200_H
#define QTENSOR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QT_B200_ABI_VERSION 2

enum qt_status {
  QT_OK = 0,
  QT_EINVAL = 1, /* reference throws std::invalid_argument            */
  QT_ECUDA = 2,  /* CUDA runtime / launch error                       */
  QT_ENOMEM = 3, /* device or pinned-host allocation failed            */
  QT_ENCCL = 4,  /* NCCL unavailable or failed (multi-GPU driver)      */
  QT_ENODEV = 5, /* no usable sm_100 device                            */
  /* QT3 file I/O: TensorIoErrorKind of tensor_io.hpp:22 (+ open/read/write) */
  QT_EBADMAGIC = 6,
  QT_ETRUNCATED = 7,
  QT_EDIMOVERFLOW = 8,
  QT_EIO = 9
};

/* ---- library ---------------------------------------------------------- */

/* ABI version (QT_B200_ABI_VERSION). */
int qt_abi_version(void);

/* Last error message of the calling thread ("" if none). */
const char* qt_last_error(void);

/* Number of CUDA kernels this library has launched in the process so far
 * (all devices).  Used by bench.py to report gpu_launches. */
uint64_t qt_kernel_launches(void);

/* Per-kernel device timing (CUDA events recorded on the launching stream
 * around each launch of a tagged kernel), for bench.py's roofline.  Off by
 * default; qt_prof_read synchronizes on the recorded events, returns the
 * summed milliseconds and launch count of one tag and clears it.  Tags:
 * "fft" (K1/K3 tube FFTs), "k2_dmma" (fp64 DMMA GEMM), "k2_int8_gemm"
 * (tcgen05 int8 modular GEMM), "k2_int8_residues", "k2_int8_crt". */
void qt_prof_enable(int on);
int qt_prof_read(const char* tag, double* ms, uint64_t* launches);
/* Timeline mode (qt_prof_enable(2)): every tagged launch is also kept in
 * order; qt_prof_timeline writes "tag stream start_ms end_ms" lines (times
 * from the enable call) into buf (NUL-terminated, truncated to cap), clears
 * them and returns the full text length (negative status on error). */
int qt_prof_timeline(char* buf, uint64_t cap);

/* ---- device-resident entry points (all pointers are device pointers) ---
 * stream is a cudaStream_t (NULL = legacy default stream).  Work is enqueued
 * on the stream; the call returns without synchronising.                  */

/* C = A *_T B (T-product).  A: m x n x p, B: n x s x p, C: m x s x p.
 * Replaces tprod_fast(a, b) / tprod_fast(a, b, ws), tproduct.hpp:45-46.
 * c1/c2 must not alias the inputs. */
int qt_tprod_f64_device(const double* a1, const double* a2,
                        const double* b1, const double* b2,
                        double* c1, double* c2,
                        uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                        void* stream);

/* Forward conjugate-fused tube transform, qfft3_conj (transform.hpp:56-60):
 *   y1 = fft_3(conj(x1)),  y2 = -fft_3(x2).  In-place (y == x) is allowed. */
int qt_qfft3_conj_f64_device(const double* x1, const double* x2,
                             double* y1, double* y2,
                             uint64_t m, uint64_t n, uint64_t p, void* stream);

/* Inverse, qifft3_conj (transform.hpp:62-64):
 *   y1 = conj(ifft_3(x1)),  y2 = -ifft_3(x2).  In-place is allowed. */
int qt_qifft3_conj_f64_device(const double* x1, const double* x2,
                              double* y1, double* y2,
                              uint64_t m, uint64_t n, uint64_t p, void* stream);

/* Routed forms of the two transforms for the frequency-parallel multi-GPU
 * driver: the exchange that follows K1 (or precedes K3) is fused into the
 * transform's own stores (loads).  rows1/rows2 are DEVICE arrays of p device
 * pointers, one per slice/frequency, each addressing m*n interleaved complex
 * doubles and possibly living in a peer GPU's memory (NVLink P2P):
 *   qfft3 routed:  frequency k of plane X is written to y{X}_rows[k][0..m*n)
 *   qifft3 routed: frequency k of plane X is read from x{X}_rows[k][0..m*n)
 * Same arithmetic as the plain forms (bitwise equal results).  Only lengths p
 * whose transform is one pass support routing (qt_fft_routable(p) == 1; all
 * p <= 512 and the smooth lengths below 1024); otherwise QT_EINVAL.
 * Replaces no reference entry point: the reference is single-process. */
int qt_fft_routable(uint64_t p);
int qt_qfft3_conj_f64_device_routed(const double* x1, const double* x2,
                                    double* const* y1_rows, double* const* y2_rows,
                                    uint64_t m, uint64_t n, uint64_t p, void* stream);
/* The forward routed transform with a broadcast fused into its stores:
 * y{X}_rows holds ndst tables of p pointers (destination d's table at
 * y{X}_rows + d * p), and frequency k of plane X is written to every
 * y{X}_rows[d * p + k] (the 2-D multi-GPU decomposition: a piece transformed
 * once by its owner, stored into every rank of its row / column group). */
int qt_qfft3_conj_f64_device_routed_n(const double* x1, const double* x2,
                                      double* const* y1_rows, double* const* y2_rows, int ndst,
                                      uint64_t m, uint64_t n, uint64_t p, void* stream);
int qt_qifft3_conj_f64_device_routed(const double* const* x1_rows, const double* const* x2_rows,
                                     double* y1, double* y2,
                                     uint64_t m, uint64_t n, uint64_t p, void* stream);

/* Stage 2 alone (the paired-frequency quaternion block GEMM, tproduct.cpp:90-104)
 * on already transformed operands: chat = ahat (.) bhat per frequency pair
 * (k, p-k).  Exposed for profiling and for callers that keep operands in the
 * transformed domain. */
int qt_spectral_product_f64_device(const double* ahat1, const double* ahat2,
                                   const double* bhat1, const double* bhat2,
                                   double* chat1, double* chat2,
                                   uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                   void* stream);

/* Stage 2 with explicit strides: B̂ rows at pitch ldb and slices bslice apart,
 * Ĉ rows at pitch ldc and slices cslice apart (all in complex elements).  A
 * column chunk of B̂ then writes straight into its columns of a wider Ĉ (pass
 * chat + column offset): the building block of the chunked-broadcast
 * multi-GPU pipeline (B arrives in column chunks, tproduct.cpp:90-104 per
 * chunk). */
int qt_spectral_product_f64_device_ld(const double* ahat1, const double* ahat2,
                                      const double* bhat1, const double* bhat2,
                                      double* chat1, double* chat2,
                                      uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                      uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice,
                                      void* stream);

/* Stage-2 algorithm for a product of this shape: QT_GEMM_DMMA (FP64 DMMA
 * tensor cores, mma.sync m8n8k4) or QT_GEMM_INT8_EXACT (exact integer
 * evaluation on the int8 tcgen05 tensor cores: 15 modular int8 GEMMs + CRT,
 * fp64-accurate).  Depends on (n, s) only and on
 * $QTB_OZAKI (0 never, 1 auto, 2 whenever n allows).  A caller that splits one
 * product into row slabs or column chunks passes the full-shape choice to
 * qt_spectral_product_f64_device_ld_algo so every piece uses the same
 * arithmetic (bitwise-identical results). */
#define QT_GEMM_AUTO (-1)
#define QT_GEMM_DMMA 0
#define QT_GEMM_INT8_EXACT 1
int qt_gemm_algo(uint64_t m, uint64_t n, uint64_t s, uint64_t p);
/* 1 if qt_tprod_f64_device runs a product of this shape as ONE launch (the
 * cluster kernel of csrc/qt_small.cu: K1, K2 and K3 exchanging through
 * distributed shared memory; p in {2, 4, 8, 16}, m, s <= 32, n <= 64, fp64 DMMA
 * stage 2; $QTB_SMALL=0 turns it off), else 0 (three or more launches).  The
 * result is bitwise the same either way.  Same role as qt_gemm_algo: an
 * introspection entry with no reference counterpart. */
int qt_small_fused(uint64_t m, uint64_t n, uint64_t s, uint64_t p);
int qt_spectral_product_f64_device_ld_algo(const double* ahat1, const double* ahat2,
                                           const double* bhat1, const double* bhat2,
                                           double* chat1, double* chat2,
                                           uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                           uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice,
                                           int algo, void* stream);

/* Accuracy guard of the int8 stage 2: before anything is
 * rounded every contraction index j of frequency pair (k, p-k) is balanced by
 * an exact power of two (row j of B̂ scaled to a maximum in [1/2, 1), column j
 * of Â by the inverse), and after the CRT each pair's rigorous error bound is
 * compared with its |Ĉ|: pairs whose relative Frobenius error cannot be
 * certified below 2^-42 ($QTB_OZAKI_GUARD_LOG2) are recomputed by the fp64
 * DMMA kernels.  This counter is the number of pairs sent to DMMA so far on
 * the current device (tests; $QTB_OZAKI_GUARD=force sends every pair). */
uint64_t qt_int8_guard_fallbacks(void);

/* Frequency slots (multi-GPU plumbing; no reference counterpart — the
 * reference's tprod_fast is single-process, tproduct.cpp:75-111).  Stage 2
 * visits frequencies in slots: slot 2j, 2j+1 hold the pair (j+1, p-j-1), the
 * self-paired 0 (and p/2 for even p) come last.  qt_slot_frequency maps a
 * slot to its frequency (-1 if slot >= p). */
int qt_slot_frequency(uint64_t p, uint64_t slot);

/* Exact int8 stage 2 on a compact slot range [slot0, slot0 + nslots) (the
 * frequency-parallel multi-GPU driver: one range per rank).  B̂ (nslots, n, s),
 * and the Â (nslots, m, n) / Ĉ (nslots, m, s) of every multiply, hold slice t
 * = slot slot0 + t (two complex128 planes each, dense).  Neither end of the
 * range may split a pair (an odd boundary below 2 * ((p - 1) / 2)).  B̂ must stay
 * valid until qt_int8_slots_destroy (the fp64 fallback reads it).  Non-finite
 * inputs and pairs the accuracy guard does not certify are recomputed by the
 * fp64 DMMA kernels on the compact tensors, as in the full-range product;
 * `nonfinite` (optional device int) receives 1 after a multiply whose Â or B̂
 * held an inf/NaN.  Bitwise identical to the same slots of a full-range int8
 * product. */
int qt_int8_slots_create(const double* bhat1, const double* bhat2, uint64_t n, uint64_t s, uint64_t p, int slot0,
                         int nslots, int* nonfinite, void* stream, void** handle);
int qt_int8_slots_multiply(void* handle, const double* ahat1, const double* ahat2, uint64_t m, double* chat1,
                           double* chat2, void* stream);
int qt_int8_slots_destroy(void* handle, void* stream);

/* Definitional product tprod_naive = fold(bcirc(A) . unfold(B))
 * (tproduct.hpp:23-25, tproduct.cpp:49-53) without materialising bcirc:
 * C_k = sum_r A_{(k-r) mod p} (.) B_r on FP64 DMMA.  16 m n s p^2 real
 * multiplications — the O(p^2) oracle the fast path is checked against. */
int qt_tprod_naive_f64_device(const double* a1, const double* a2,
                              const double* b1, const double* b2,
                              double* c1, double* c2,
                              uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                              void* stream);

/* ---- host-buffer entry points (what the C++ drop-in calls) ------------
 * All pointers are host pointers (pageable or pinned).  The call copies to
 * device `device`, computes, copies back and synchronises. */

int qt_tprod_f64_host(const double* a1, const double* a2,
                      const double* b1, const double* b2,
                      double* c1, double* c2,
                      uint64_t m, uint64_t n, uint64_t s, uint64_t p, int device);

/* tprod_fast that also returns Â, B̂, Ĉ (each m*n / n*s / m*s * p complex per
 * plane, host buffers): the reference's TProdWorkspace side effect
 * (tproduct.cpp:80-87, ws.ahat / ws.bhat / ws.chat), used by the drop-in when
 * $QTB_DROPIN_FILL_WS=1.  C equals qt_tprod_f64_host's. */
int qt_tprod_f64_host_spectra(const double* a1, const double* a2, const double* b1, const double* b2,
                              double* c1, double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, int device,
                              double* ahat1, double* ahat2, double* bhat1, double* bhat2,
                              double* chat1, double* chat2);

int qt_tprod_naive_f64_host(const double* a1, const double* a2,
                            const double* b1, const double* b2,
                            double* c1, double* c2,
                            uint64_t m, uint64_t n, uint64_t s, uint64_t p, int device);

int qt_qfft3_conj_f64_host(const double* x1, const double* x2,
                           double* y1, double* y2,
                           uint64_t m, uint64_t n, uint64_t p, int device);

int qt_qifft3_conj_f64_host(const double* x1, const double* x2,
                            double* y1, double* y2,
                            uint64_t m, uint64_t n, uint64_t p, int device);

/* ---- single-process multi-GPU driver -----------------------------------
 * Host buffers in, host buffers out.  Rows of A and C are sharded in
 * contiguous slabs of ceil(m/ndev) rows over devices[0..ndev); B is copied
 * to devices[0] once and broadcast to the others with NCCL over NVLink, then
 * every device runs the single-GPU product of its slab (csrc/qt_multi.cu).
 * ndev == 1 runs without NCCL.  Output is bitwise identical for every ndev;
 * the caller's current device is restored. */
int qt_tprod_f64_multi(const double* a1, const double* a2,
                       const double* b1, const double* b2,
                       double* c1, double* c2,
                       uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                       const int* devices, int ndev);

/* ---- one process per GPU (torchrun): per-rank multi-GPU drivers ---------
 * No reference counterpart (the reference is single-process,
 * tproduct.cpp:75-111).  The library owns the NCCL communicator (NCCL is
 * resolved at run time, csrc/qt_nccl.h); the launcher only moves the 128-byte
 * id: rank 0 calls qt_comm_unique_id, every rank qt_comm_init with it (prints
 * one "[qtensor_b200] NCCL x.y.z communicator: rank r of G on cuda:d" line).
 * All device pointers below live on the rank's device, which must be current.
 *
 * Row split (the north_star decomposition, csrc/qt_rank.cu): the rank owns
 * `rows` rows of A and C (a contiguous slab, qt_rank_partition); b1/b2 are
 * n*s*p complex planes on every rank, holding B on `root` — broadcast in
 * place (grouped ncclBroadcast per plane on `stream`), then the single-GPU
 * product of the slab.  Bitwise equal to the rows of the one-GPU product.
 *
 * Frequency-parallel split: rank r passes its rows [a0, a1) of A, its rows
 * [b0, b1) of B and receives its rows [a0, a1) of C (qt_rank_partition's
 * out6 = {a0, a1, b0, b1, slot0, slot1}); stage 2 of the frequency slots
 * [slot0, slot1) runs on this rank, the pieces move by NCCL send/recv.
 * Bitwise equal to the one-GPU product.  qt_rank_freq_emulate runs `world`
 * ranks in lockstep on the current device (pieces moved by device copies,
 * same schedule) over whole-tensor device buffers: the single-GPU test of the
 * decomposition. */
int qt_comm_unique_id(void* id128);
int qt_comm_init(const void* id128, int rank, int world, int device, void** comm);
int qt_comm_destroy(void* comm);
int qt_rank_partition(uint64_t m, uint64_t n, uint64_t p, int world, int rank, uint64_t* out6);
/* host only: the frequency-parallel exchange schedule of `rank` for part 0 (Â),
 * 1 (B̂) or 2 (Ĉ), its sends (send = 1) or receives, in transfer order: per
 * piece {peer, slot, plane, first row, rows} (rows of the m- or n-row
 * dimension).  count = number of pieces (out5 = NULL: count only). */
int qt_rank_freq_schedule(uint64_t m, uint64_t n, uint64_t s, uint64_t p, int world, int rank, int part, int send,
                          int64_t* out5, uint64_t cap, uint64_t* count);
int qt_rank_tprod_rows(void* comm, const double* a1, const double* a2, double* b1, double* b2,
                       double* c1, double* c2, uint64_t rows, uint64_t n, uint64_t s, uint64_t p,
                       int root, void* stream);
int qt_rank_freq_create(void* comm, uint64_t m, uint64_t n, uint64_t s, uint64_t p, void** plan);
int qt_rank_freq_step(void* plan, const double* a1, const double* a2, const double* b1, const double* b2,
                      double* c1, double* c2, void* stream);
int qt_rank_freq_nonfinite(void* plan, int* out);
int qt_rank_freq_destroy(void* plan);
int qt_rank_freq_emulate(int world, int fused, const double* a1, const double* a2, const double* b1,
                         const double* b2, double* c1, double* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                         void* stream);
/* Fused exchange over peer memory (NVLink): each rank exports its stage
 * buffer (qt_rank_freq_ipc_handle, 64 bytes), the launcher gathers all of them
 * in rank order and every rank calls qt_rank_freq_set_peers: from then on a
 * step's K1 stores each frequency row straight into its slot owner's buffer
 * and K3 loads its rows straight from the owners (routed transforms), with the
 * library's own device barrier between the phases — no messages.  Lengths
 * whose transform is one launch only (qt_fft_routable).  qt_rank_freq_create_ipc
 * makes a plan without an NCCL communicator (fused exchange only);
 * qt_rank_freq_phase runs phase 0 (routed K1), 1 (stage 2), 2 (routed K3)
 * without the device barriers, for callers that order the ranks themselves. */
int qt_rank_freq_create_ipc(int rank, int world, int device, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                            void** plan);
int qt_rank_freq_ipc_handle(void* plan, void* handle64);
int qt_rank_freq_set_peers(void* plan, const void* handles);
int qt_rank_freq_phase(void* plan, int phase, const double* a1, const double* a2, const double* b1,
                       const double* b2, double* c1, double* c2, void* stream);

/* ---- QT3 tensor files <-> device planes ---------------------------------
 * The reference's binary format (tensor_io.hpp:16-20): "QT3\0", m, n, p as
 * little-endian u64, then m*n*p records (w, x, y, z) little-endian doubles,
 * slice-major.  Reading streams the file through pinned staging into the two
 * device CD planes (a de-interleave kernel splits each 32-byte record);
 * writing is the reverse.  Both return after the data is on the device / in
 * the file, bit-exact.  Header errors follow parse_tensor
 * (tensor_io.cpp:56-80): QT_EBADMAGIC, QT_ETRUNCATED, QT_EDIMOVERFLOW;
 * open/read/write failures QT_EIO. */
int qt_qt3_probe(const char* path, uint64_t* m, uint64_t* n, uint64_t* p);

int qt_qt3_read_f64_device(const char* path, double* t1, double* t2,
                           uint64_t m, uint64_t n, uint64_t p, void* stream);

int qt_qt3_write_f64_device(const char* path, const double* t1, const double* t2,
                            uint64_t m, uint64_t n, uint64_t p, void* stream);

/* ---- seeded synthetic inputs (host) -----------------------------------
 * dist: QT_DIST_UNIFORM_SYM    all four components U[-1,1) — bitwise equal to
 *                              the reference's gen_random_tensor (rng.cpp:21-33)
 *       QT_DIST_NORMAL         all four components N(0, scale^2), Box-Muller
 *                              over the same mt19937_64 top-53 uniforms
 *       QT_DIST_PURE_UNIT      w = 0, (x, y, z) = U[0,1) (colour-video cfg4 A)
 * t1/t2 are host arrays of 2*m*n*p doubles. */
enum qt_dist { QT_DIST_UNIFORM_SYM = 0, QT_DIST_NORMAL = 1, QT_DIST_PURE_UNIT = 2 };

int qt_gen_tensor_f64(int dist, uint64_t m, uint64_t n, uint64_t p, uint64_t seed,
                      double scale, double* t1, double* t2);

/* derive_seed(base, stream) of rng.cpp:15-19 (splitmix64 chain). */
uint64_t qt_derive_seed(uint64_t base, uint64_t stream);

#ifdef __cplusplus
}
#endif

#endif /* QTENSOR_B200_H */
