// qt_internal.cuh — shared declarations of the sm_100a T-product kernels.
//
// Data layout in HBM: every quaternion tensor is two
// Cayley-Dickson planes (t1, t2), each m*n*p double2 (re, im), slice-major:
// element (i, j, r) at (r*m + i)*n + j.  A "tube" (i, j) is the stride-m*n
// sequence over r.  The transformed operands Â, B̂, Ĉ use the same layout, so
// per frequency k the slice k of each plane is a dense row-major matrix — the
// GEMM-friendly form the paired-frequency kernel reads.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>

namespace qtb {

// ---------------------------------------------------------------- tube FFT
// One "job" = one CD plane of one tensor.  The transform applied per tube is
//   y = scale * conj_out?( F( conj_in?(x) ) ),   F = unnormalised forward DFT
// which covers the four TubeOps of transform.cpp:116-147:
//   ConjInForward   (t1 of qfft3_conj)  : conj_in=1, conj_out=0, scale=+1
//   NegateForward   (t2 of qfft3_conj)  : conj_in=0, conj_out=0, scale=-1
//   InverseConjOut  (t1 of qifft3_conj) : conj_in=1, conj_out=0, scale=+1/p
//   NegateInverse   (t2 of qifft3_conj) : conj_in=1, conj_out=1, scale=-1/p
// (conj(ifft(x)) = F(conj x)/p and -ifft(x) = -conj(F(conj x))/p.)
struct TubeJob {
  const double2* in;
  double2* out;
  uint64_t ntubes;  // m*n of the tensor (tubes per plane)
  int conj_in;
  int conj_out;
  double scale;
  int stream_out = 0;  // 1: evict-first stores (final pass of the split FFT: keep its L2 scratch resident)
  // Routed rows (single-pass transforms only): input row r (slice r, ntubes
  // complex) is read from in_rows[r] instead of in + r*ntubes, output row k
  // is written to out_rows[k] — device pointer tables, possibly pointing into
  // peer GPUs' memory, so a transform can scatter its frequency rows straight
  // to the ranks that own them (or gather them) over NVLink.
  const double2* const* in_rows = nullptr;
  double2* const* out_rows = nullptr;
  // several destinations per output row (a broadcast fused into the stores):
  // destination d's table at out_rows + d * out_rows_stride
  int out_ndst = 1;
  int out_rows_stride = 0;
};

constexpr int kMaxJobs = 4;
constexpr int kMaxStages = 40;

struct TubeBatch {
  TubeJob job[kMaxJobs];
  int njobs;
};

struct FftPlan {
  int p;
  int nstages;
  int radix[kMaxStages];
};

// Radix schedule for length p (8s first, then 4, 2, then odd primes).
FftPlan make_fft_plan(int p);

// Device twiddle table W_p[k] = exp(-2 pi i k / p), k in [0, p), cached per
// (device, p).  Returns nullptr on failure (error recorded).
const double2* twiddles_for(int device, int p, cudaStream_t stream);

// Enqueue the tube transform of every job in `batch` (all jobs share p).
// Returns cudaSuccess or the launch error.
cudaError_t launch_tube_fft(const TubeBatch& batch, int p, cudaStream_t stream, int device);
// The length-p transform runs as one pass (so routed rows are supported).
bool fft_single_pass(int p);
// The length-p transform runs as the two-pass four-step split.
bool fft_split_length(int p);

// ------------------------------------------------------ paired spectral GEMM
// chat[k] for all k from ahat, bhat (slice-major CD planes), tproduct.cpp:90-104.
cudaError_t launch_spectral_gemm(const double2* ah1, const double2* ah2,
                                 const double2* bh1, const double2* bh2,
                                 double2* ch1, double2* ch2,
                                 uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                 cudaStream_t stream, int algo = -1);

// Same with explicit leading dimensions: B̂ rows at pitch ldb (slice stride
// bslice), Ĉ rows at pitch ldc (slice stride cslice) — lets a column chunk of
// B̂ write straight into its columns of a wider Ĉ (multi-GPU chunked broadcast).
cudaError_t launch_spectral_gemm_ld(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                    double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                    uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice,
                                    cudaStream_t stream, int algo = -1);

// Frequency slots of the stage-2 schedule: slot 2j, 2j+1 hold the pair
// (j+1, p-j-1); the self-paired 0 and p/2 come last.
__host__ __device__ __forceinline__ int slot_frequency(int slot, int p) {
  const int npairs = (p - 1) / 2;
  if (slot < 2 * npairs) return (slot & 1) ? p - (slot / 2 + 1) : slot / 2 + 1;
  return slot == 2 * npairs ? 0 : p / 2;
}
// Units of a slot range [s0, s0 + ns) that keeps pairs whole: the pairs
// (2j, 2j+1) below pair_end first, then the self-paired slots (one each).
__host__ __device__ __forceinline__ int slot_units(int s0, int ns, int p) {
  const int pe = 2 * ((p - 1) / 2);
  const int lo = s0 < pe ? s0 : pe, hi = s0 + ns < pe ? s0 + ns : pe;
  const int np = (hi - lo) / 2;
  const int from = s0 > pe ? s0 : pe;
  return np + (s0 + ns > from ? s0 + ns - from : 0);
}
__host__ __device__ __forceinline__ void unit_slots(int u, int s0, int ns, int p, int& sa, int& sb) {
  const int pe = 2 * ((p - 1) / 2);
  const int lo = s0 < pe ? s0 : pe, hi = s0 + ns < pe ? s0 + ns : pe;
  const int np = (hi - lo) / 2;
  if (u < np) {
    sa = s0 + 2 * u;
    sb = sa + 1;
  } else {
    sa = sb = (s0 > pe ? s0 : pe) + (u - np);
  }
}

// Exact int8 tensor-core (Ozaki-II / CRT) evaluation of the same product
// (qt_ozaki.cu).  `flag` is a device int array of int8_flag_ints(p) entries,
// zeroed by the caller: flag[0] is set to 1 if the inputs hold a non-finite
// value (C is then left untouched), flag[1 + min(k, p - k)] to 1 if the
// accuracy guard could not certify pair k (C of that pair is then to be
// recomputed by dmma_spectral_gemm with only_if = flag).
enum GemmAlgo { kAlgoAuto = -1, kAlgoDmma = 0, kAlgoOzaki = 1 };
inline uint64_t int8_flag_ints(uint64_t p) { return p / 2 + 2; }
bool ozaki_supported(uint64_t n, uint64_t s, uint64_t p);
// the algorithm a product of this shape uses (callers that split one product
// into row slabs or column chunks decide once, on the full shape)
inline int choose_gemm_algo(uint64_t n, uint64_t s, uint64_t p) {
  return ozaki_supported(n, s, p) ? kAlgoOzaki : kAlgoDmma;
}
cudaError_t launch_spectral_gemm_ozaki(const double2* ah1, const double2* ah2, const double2* bh1,
                                       const double2* bh2, double2* ch1, double2* ch2, uint64_t m, uint64_t n,
                                       uint64_t s, uint64_t p, uint64_t ldb, uint64_t ldc, uint64_t bslice,
                                       uint64_t cslice, int* flag, cudaStream_t stream);
// Two-phase form for row-slab streaming: B' residues prepared once for every
// frequency (require_all) or per A batch, then any number of A row slabs.
struct OzakiB {
  uint8_t* res = nullptr;
  int* eB = nullptr;
  double* yl1 = nullptr;  // L1 norms of the scaled B' columns (accuracy guard)
  int* bdel = nullptr;    // contraction balancing exponents, [p][n] by frequency
  int* bmin = nullptr;    // smallest column exponent per B' slot (accuracy guard weights)
  uint64_t n = 0, s = 0, p = 0, ldb = 0, bslice = 0;
  int nslots = 0;
  bool all = false;
  int s0 = 0, ns = 0, cbase = -1;  // slot range; cbase >= 0: compact operand tensors (slot - cbase)
  // all && !ready: B' is built batch by batch inside the first multiply (its
  // residues pipelined beside the GEMMs of earlier batches) from bh1/bh2
  bool ready = false;
  const double2* bh1 = nullptr;
  const double2* bh2 = nullptr;
};
// lazy: with B' kept for every slot, defer its residues into the first
// multiply's batch pipeline (B̂ must stay valid until then)
cudaError_t ozaki_prepare_b(const double2* bh1, const double2* bh2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                            uint64_t ldb, uint64_t bslice, int* flag, bool require_all, OzakiB* out,
                            cudaStream_t stream, bool lazy = false);
cudaError_t ozaki_multiply(OzakiB& B, const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                           uint64_t m, double2* ch1, double2* ch2, uint64_t ldc, uint64_t cslice, int* flag,
                           cudaStream_t stream);
cudaError_t ozaki_release(OzakiB& B, cudaStream_t stream);
cudaError_t ozaki_prepare_b_slots(const double2* bh1, const double2* bh2, uint64_t n, uint64_t s, uint64_t p, int s0,
                                  int ns, int* flag, OzakiB* out, cudaStream_t stream);
// pairs the accuracy guard has sent to the DMMA kernels since load (all devices' counters summed: this device's)
uint64_t int8_guard_fallbacks();
// DMMA kernels that run only if *only_if != 0 (nullptr: always); with an
// int8 flag array (see above) a CTA of pair k runs if flag[0] or flag[1 + k]
cudaError_t dmma_spectral_gemm(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                               double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                               uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice, cudaStream_t stream,
                               const int* only_if);
// the same on compact slot tensors (slice t = frequency slot s0 + t, the
// slot range keeping pairs whole; qt_int8_slots_*)
cudaError_t dmma_spectral_gemm_slots(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                     double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                     int s0, int ns, cudaStream_t stream, const int* only_if);

// $QTB_DEBUG_NO_REFLECT=1: sigma(k) = k in stage 2 (the parity tests' negative control)
bool debug_noreflect();
bool dmma_gauss();
// One-launch T-product for small products (qt_small.cu): eligibility and launch.
bool small_fused_eligible(uint64_t m, uint64_t n, uint64_t s, uint64_t p);
cudaError_t launch_small_tprod(const double2* a1, const double2* a2, const double2* b1, const double2* b2,
                               double2* c1, double2* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                               cudaStream_t stream, int device);

// Definitional product C_k = sum_r A_{(k-r) mod p} (.) B_r (qt_naive.cu).
cudaError_t launch_naive_tprod(const double2* a1, const double2* a2, const double2* b1, const double2* b2,
                               double2* c1, double2* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                               cudaStream_t stream);

// QT3 file I/O (qt_io.cu); status codes of qtensor_b200.h, message in *err.
int qt3_probe(const char* path, uint64_t* m, uint64_t* n, uint64_t* p, std::string* err);
int qt3_read_device(const char* path, double* t1, double* t2, uint64_t m, uint64_t n, uint64_t p,
                    cudaStream_t stream, std::string* err);
int qt3_write_device(const char* path, const double* t1, const double* t2, uint64_t m, uint64_t n, uint64_t p,
                     cudaStream_t stream, std::string* err);

// Kernel attributes (e.g. the dynamic shared-memory opt-in) are per device:
// run `fn` once for every device a launcher is used on (thread-safe).
template <class F>
cudaError_t once_per_device(std::mutex& mu, uint64_t& done_mask, F fn) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && ((done_mask >> dev) & 1ull)) return cudaSuccess;
  e = fn();
  if (e == cudaSuccess && dev < 64) done_mask |= 1ull << dev;
  return e;
}

// Launch accounting (qt_kernel_launches).
void count_launches(uint64_t k);

// Per-kernel event timing (qt_prof_enable / qt_prof_read): a ProfScope
// records a start event on construction and a stop event in stop(); both are
// no-ops unless profiling is on.
bool prof_on();
struct ProfScope {
  const char* tag;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  cudaEvent_t t0 = nullptr;  // timeline twin of e0 (qt_prof_enable(2))
  ProfScope(const char* t, cudaStream_t s);
  void stop();
};

}  // namespace qtb
