// qt_fft.cu — K1/K3: batched mode-3 tube FFT over the CD planes (sm_100a).
//
// Replaces transform_tubes/fft_rec (/root/reference/proj/src/transform.cpp:12-68,
// 116-147).  The reference gathers each stride-m*n tube into a heap vector and
// runs a recursive smallest-prime-factor DIT with per-call twiddles.  Here a
// CTA owns T consecutive tubes of one CD plane (consecutive tubes are
// consecutive in memory, so every access is a T*16-byte coalesced row) and
// runs a mixed-radix Stockham FFT: radix-8/4/2 register butterflies, generic
// direct-DFT stages for odd prime factors (the same O(p^2) fallback the
// reference takes for prime lengths, transform.cpp:48).  The first stage reads
// HBM directly and the last stage writes HBM directly with the conj/negate/
// scale of the TubeOp fused in, so a 64-point tube costs one HBM read, one
// shared-memory round trip and one HBM write.
//
// Long tubes (p*T*16 B does not fit shared memory with T >= 8, e.g. p = 4096)
// use a two-pass four-step split p = p1*p2: pass A transforms the p1-point
// stride-p2 sub-tubes and applies the W_p^(n2*k1) twiddle, pass B transforms the
// p2-point contiguous sub-tubes and writes the transposed result; both passes
// keep T = 32-tube coalesced rows.  Lengths with no usable split (large primes)
// use one generic stage per launch over global memory.
//
// Bytes per tube element: 16 B read + 16 B written per CD plane (x2 for the
// two-pass split) — HBM-bound.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "qt_fft_reg.cuh"
#include "qt_internal.cuh"

namespace qtb {

// ------------------------------------------------------------------ planning
FftPlan make_fft_plan(int p) {
  FftPlan pl{};
  pl.p = p;
  int rest = p, ns = 0;
  while (rest % 8 == 0 && ns < kMaxStages) { pl.radix[ns++] = 8; rest /= 8; }
  while (rest % 4 == 0 && ns < kMaxStages) { pl.radix[ns++] = 4; rest /= 4; }
  while (rest % 2 == 0 && ns < kMaxStages) { pl.radix[ns++] = 2; rest /= 2; }
  for (int f = 3; rest > 1 && ns < kMaxStages;) {
    if ((long long)f * f > rest) { pl.radix[ns++] = rest; rest = 1; break; }
    if (rest % f == 0) { pl.radix[ns++] = f; rest /= f; }
    else f += 2;
  }
  pl.nstages = ns;
  return pl;
}

// ------------------------------------------------------------------ twiddles
namespace {
std::mutex g_tw_mu;
std::map<std::pair<int, int>, double2*> g_tw;  // (device, p) -> table
}  // namespace

const double2* twiddles_for(int device, int p, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_pair(device, p);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) return it->second;
  // exp(-2 pi i k/p) evaluated in x87 long double (64-bit mantissa) and
  // rounded once to double; exact at the quarter points.
  std::vector<double2> h(p);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int k = 0; k < p; ++k) {
    long double ang = two_pi * (long double)k / (long double)p;
    h[k].x = (double)cosl(ang);
    h[k].y = (double)(-sinl(ang));
  }
  h[0] = make_double2(1.0, 0.0);
  if (p % 2 == 0) h[p / 2] = make_double2(-1.0, 0.0);
  if (p % 4 == 0) { h[p / 4] = make_double2(0.0, -1.0); h[3 * p / 4] = make_double2(0.0, 1.0); }
  double2* d = nullptr;
  if (cudaMalloc(&d, sizeof(double2) * p) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), sizeof(double2) * p, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  (void)stream;
  g_tw[key] = d;
  return d;
}

// complex arithmetic and the radix-2/4/8 register butterflies: qt_fft_reg.cuh

__host__ __device__ __forceinline__ bool is_reg_radix(int R) { return R == 2 || R == 4 || R == 8; }

// Row geometry of one launch.  A CTA in group g transforms, for each of its T
// tubes, the L elements at rows  g*ig + i*is  (i < L) and writes output k to
// row  g*og + k*os, optionally multiplied by W_p^(g*k) (four-step twiddle).
// W_L^e is read from the length-p table as tw[e * tws], tws = p / L.
struct FftGeom {
  int L, ig, is, og, os, post_tw, tws;
};

// Row base pointers (tube t0 of row r), plain or routed through the job's row
// tables.  Routed launches use only the single-pass geometry (rows = slices).
template <bool ROUTED>
__device__ __forceinline__ const double2* in_row(const TubeJob& job, int row, uint64_t t0) {
  if (ROUTED && job.in_rows) return job.in_rows[row] + t0;
  return job.in + (uint64_t)row * job.ntubes + t0;
}
template <bool ROUTED>
__device__ __forceinline__ double2* out_row(const TubeJob& job, int row, uint64_t t0) {
  if (ROUTED && job.out_rows) return job.out_rows[row] + t0;
  return job.out + (uint64_t)row * job.ntubes + t0;
}

// One Stockham stage of radix R over an L x T smem tile (tube index fastest).
// src/dst element (r, t) at [r*T + t].  Ns = product of earlier radices.
template <int R>
__device__ __forceinline__ void stage_reg(const double2* __restrict__ src, double2* __restrict__ dst,
                                          const double2* __restrict__ tw, const FftGeom& G, int logT, int Ns) {
  const int T = 1 << logT;
  const int L = G.L;
  const int pR = L / R;
  const int twmul = (L / (Ns * R)) * G.tws;
  for (int b = threadIdx.x; b < (pR << logT); b += blockDim.x) {
    const int j = b >> logT, t = b & (T - 1);
    const int jm = j % Ns;
    const int step = jm * twmul;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[((j + r * pR) << logT) + t];
    if (step != 0) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[r * step]));
    }
    dft_reg<R>(v);
    const int idxD = (j - jm) * R + jm;
#pragma unroll
    for (int k = 0; k < R; ++k) dst[((idxD + k * Ns) << logT) + t] = v[k];
  }
}

// Generic radix-R stage: one output per thread iteration, direct R-point DFT
// folded with the stage twiddle into one table lookup.
__device__ __forceinline__ void stage_generic(const double2* __restrict__ src, double2* __restrict__ dst,
                                              const double2* __restrict__ tw, const FftGeom& G, int logT, int Ns,
                                              int R) {
  const int T = 1 << logT;
  const int L = G.L;
  const int pR = L / R;
  const int twmul = L / (Ns * R);
  for (int b = threadIdx.x; b < (L << logT); b += blockDim.x) {
    const int o = b >> logT, t = b & (T - 1);
    const int j = o / R, k = o - j * R;
    const int jm = j % Ns;
    const int base = jm * twmul + k * pR;  // < L
    double2 acc = src[(j << logT) + t];
    int e = 0;
    for (int r = 1; r < R; ++r) {
      e += base;
      if (e >= L) e -= L;
      const double2 x = src[((j + r * pR) << logT) + t];
      const double2 w = __ldg(&tw[e * G.tws]);
      acc.x = fma(x.x, w.x, fma(-x.y, w.y, acc.x));
      acc.y = fma(x.x, w.y, fma(x.y, w.x, acc.y));
    }
    const int idxD = (j - jm) * R + jm;
    dst[((idxD + k * Ns) << logT) + t] = acc;
  }
}

__device__ __forceinline__ void stage_smem(const double2* src, double2* dst, const double2* __restrict__ tw,
                                           const FftGeom& G, int logT, int Ns, int R) {
  if (R == 8) stage_reg<8>(src, dst, tw, G, logT, Ns);
  else if (R == 4) stage_reg<4>(src, dst, tw, G, logT, Ns);
  else if (R == 2) stage_reg<2>(src, dst, tw, G, logT, Ns);
  else stage_generic(src, dst, tw, G, logT, Ns, R);
}

// output store with the four-step twiddle, conj-out and scale fused
template <bool ROUTED>
__device__ __forceinline__ void store_out(const TubeJob& job, uint64_t t0, const FftGeom& G,
                                          const double2* __restrict__ tw, int g, int kk, int t, double2 v) {
  if (G.post_tw && g != 0) v = cmul(v, __ldg(&tw[g * kk]));
  const double sc = job.scale;
  const double sci = job.conj_out ? -sc : sc;
  const double2 o = make_double2(v.x * sc, v.y * sci);
  const int row = g * G.og + kk * G.os;
  if (ROUTED && job.out_rows) {
    for (int d = 0; d < job.out_ndst; ++d) job.out_rows[d * job.out_rows_stride + row][t0 + t] = o;
  } else {
    out_row<ROUTED>(job, row, t0)[t] = o;
  }
}

// stage 0: HBM -> registers -> smem (Ns = 1, so no twiddles)
template <int R, bool ROUTED>
__device__ __forceinline__ void stage_first_global(const TubeJob& job, const FftGeom& G, int g, uint64_t t0,
                                                   int tcount, double2* __restrict__ dst, int logT) {
  const int T = 1 << logT;
  const int pR = G.L / R;
  for (int b = threadIdx.x; b < (pR << logT); b += blockDim.x) {
    const int j = b >> logT, t = b & (T - 1);
    double2 v[R];
    const bool ok = t < tcount;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = g * G.ig + (j + r * pR) * G.is;
      v[r] = ok ? __ldcs(&in_row<ROUTED>(job, row, t0)[t]) : make_double2(0.0, 0.0);
      if (job.conj_in) v[r].y = -v[r].y;
    }
    dft_reg<R>(v);
#pragma unroll
    for (int k = 0; k < R; ++k) dst[((j * R + k) << logT) + t] = v[k];
  }
}

// last stage: smem -> registers -> HBM with the output ops fused
template <int R, bool ROUTED>
__device__ __forceinline__ void stage_last_global(const double2* __restrict__ src, const TubeJob& job,
                                                  const FftGeom& G, int g, uint64_t t0, int tcount,
                                                  const double2* __restrict__ tw, int logT, int Ns) {
  const int T = 1 << logT;
  const int pR = G.L / R;
  const int twmul = (G.L / (Ns * R)) * G.tws;
  for (int b = threadIdx.x; b < (pR << logT); b += blockDim.x) {
    const int j = b >> logT, t = b & (T - 1);
    const int jm = j % Ns;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[((j + r * pR) << logT) + t];
    const int step = jm * twmul;
    if (step != 0) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[r * step]));
    }
    dft_reg<R>(v);
    if (t < tcount) {
      const int idxD = (j - jm) * R + jm;
#pragma unroll
      for (int k = 0; k < R; ++k) store_out<ROUTED>(job, t0, G, tw, g, idxD + k * Ns, t, v[k]);
    }
  }
}

// single-stage transform (L in {2, 4, 8}): HBM -> registers -> HBM
template <int R, bool ROUTED>
__device__ __forceinline__ void stage_only_global(const TubeJob& job, const FftGeom& G, int g, uint64_t t0,
                                                  int tcount, const double2* __restrict__ tw, int logT) {
  const int T = 1 << logT;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    if (t >= tcount) continue;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      v[r] = __ldcs(&in_row<ROUTED>(job, g * G.ig + r * G.is, t0)[t]);
      if (job.conj_in) v[r].y = -v[r].y;
    }
    dft_reg<R>(v);
#pragma unroll
    for (int k = 0; k < R; ++k) store_out<ROUTED>(job, t0, G, tw, g, k, t, v[k]);
  }
}

// K1 / K3 kernel: grid = (tube tiles, jobs, groups), T = 1 << logT tubes per CTA.
template <bool ROUTED>
__global__ void __launch_bounds__(256) tube_fft_kernel(TubeBatch batch, FftPlan plan, FftGeom G,
                                                       const double2* __restrict__ tw, int logT) {
  extern __shared__ double2 sm[];
  const TubeJob job = batch.job[blockIdx.y];
  const int g = blockIdx.z;
  const int T = 1 << logT;
  const uint64_t t0 = (uint64_t)blockIdx.x << logT;
  if (t0 >= job.ntubes) return;
  const int L = G.L;
  const int S = plan.nstages;
  const int tcount = (int)min((uint64_t)T, job.ntubes - t0);

  if (S == 0) {  // L == 1: the transform is the identity, ops only
    const double2* __restrict__ in = in_row<ROUTED>(job, g * G.ig, t0);
    for (int t = threadIdx.x; t < tcount; t += blockDim.x) {
      double2 v = __ldcs(&in[t]);
      if (job.conj_in) v.y = -v.y;
      store_out<ROUTED>(job, t0, G, tw, g, 0, t, v);
    }
    return;
  }
  const int R0 = plan.radix[0];
  if (S == 1 && is_reg_radix(R0)) {
    if (R0 == 8) stage_only_global<8, ROUTED>(job, G, g, t0, tcount, tw, logT);
    else if (R0 == 4) stage_only_global<4, ROUTED>(job, G, g, t0, tcount, tw, logT);
    else stage_only_global<2, ROUTED>(job, G, g, t0, tcount, tw, logT);
    return;
  }

  double2* cbuf = sm;                        // holds the current data
  double2* obuf = sm + ((size_t)L << logT);  // other ping-pong buffer
  int s = 0, Ns = 1;
  if (is_reg_radix(R0)) {
    if (R0 == 8) stage_first_global<8, ROUTED>(job, G, g, t0, tcount, cbuf, logT);
    else if (R0 == 4) stage_first_global<4, ROUTED>(job, G, g, t0, tcount, cbuf, logT);
    else stage_first_global<2, ROUTED>(job, G, g, t0, tcount, cbuf, logT);
    s = 1;
    Ns = R0;
  } else {  // explicit coalesced tile load, conj fused
    for (int idx = threadIdx.x; idx < (L << logT); idx += blockDim.x) {
      const int r = idx >> logT, t = idx & (T - 1);
      double2 v = make_double2(0.0, 0.0);
      if (t < tcount) v = __ldcs(&in_row<ROUTED>(job, g * G.ig + r * G.is, t0)[t]);
      if (job.conj_in) v.y = -v.y;
      cbuf[idx] = v;
    }
  }
  __syncthreads();
  const int last_reg = is_reg_radix(plan.radix[S - 1]) ? 1 : 0;
  for (; s < S - last_reg; ++s) {
    stage_smem(cbuf, obuf, tw, G, logT, Ns, plan.radix[s]);
    __syncthreads();
    double2* tmp = cbuf;
    cbuf = obuf;
    obuf = tmp;
    Ns *= plan.radix[s];
  }
  if (last_reg) {
    const int R = plan.radix[S - 1];
    if (R == 8) stage_last_global<8, ROUTED>(cbuf, job, G, g, t0, tcount, tw, logT, Ns);
    else if (R == 4) stage_last_global<4, ROUTED>(cbuf, job, G, g, t0, tcount, tw, logT, Ns);
    else stage_last_global<2, ROUTED>(cbuf, job, G, g, t0, tcount, tw, logT, Ns);
  } else {  // generic last stage already ran into cbuf: explicit store
    for (int idx = threadIdx.x; idx < (L << logT); idx += blockDim.x) {
      const int r = idx >> logT, t = idx & (T - 1);
      if (t < tcount) store_out<ROUTED>(job, t0, G, tw, g, r, t, cbuf[idx]);
    }
  }
}

// Two-stage specialisation (L = R0*R1 with R0, R1 in {2, 4, 8}: p = 16, 32, 64
// and the 64-point halves of the four-step split — every BASELINE config):
// radices, the sub-FFT length and the stage-1 twiddle stride are compile-time,
// so the index math has no divisions and the kernel needs few registers
// (higher occupancy for the small, latency-bound launches).  Arithmetic per
// tube is the same Stockham formula as tube_fft_kernel.
template <int R0, int R1, bool ROUTED>
__global__ void __launch_bounds__(256) tube_fft2_kernel(TubeBatch batch, FftGeom G, const double2* __restrict__ tw,
                                                        int logT) {
  constexpr int L = R0 * R1;
  constexpr int P0 = L / R0, P1 = L / R1;
  extern __shared__ double2 sm[];
  const TubeJob job = batch.job[blockIdx.y];
  const int g = blockIdx.z;
  const int T = 1 << logT;
  const uint64_t t0 = (uint64_t)blockIdx.x << logT;
  if (t0 >= job.ntubes) return;
  const int tcount = (int)min((uint64_t)T, job.ntubes - t0);
  const uint64_t nt = job.ntubes;
  const double2* __restrict__ in = job.in + t0 + (uint64_t)(g * G.ig) * nt;
  const uint64_t istr = (uint64_t)G.is * nt;
  // stage 0: HBM -> registers -> smem (no twiddles)
  for (int b = threadIdx.x; b < (P0 << logT); b += blockDim.x) {
    const int j = b >> logT, t = b & (T - 1);
    double2 v[R0];
    const bool ok = t < tcount;
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      v[r] = ok ? __ldcs(ROUTED && job.in_rows ? &job.in_rows[j + r * P0][t0 + t] : &in[(uint64_t)(j + r * P0) * istr + t])
                : make_double2(0.0, 0.0);
      if (job.conj_in) v[r].y = -v[r].y;
    }
    dft_reg<R0>(v);
#pragma unroll
    for (int k = 0; k < R0; ++k) sm[((j * R0 + k) << logT) + t] = v[k];
  }
  __syncthreads();
  // stage 1 (Ns = R0): smem -> registers -> HBM, output ops fused
  double2* __restrict__ out = job.out + t0 + (uint64_t)(g * G.og) * nt;
  const uint64_t ostr = (uint64_t)G.os * nt;
  const double sc = job.scale;
  const double sci = job.conj_out ? -sc : sc;
  for (int b = threadIdx.x; b < (P1 << logT); b += blockDim.x) {
    const int j = b >> logT, t = b & (T - 1);
    const int jm = j % R0;
    double2 v[R1];
#pragma unroll
    for (int r = 0; r < R1; ++r) v[r] = sm[((j + r * P1) << logT) + t];
    if (jm != 0) {
#pragma unroll
      for (int r = 1; r < R1; ++r) v[r] = cmul(v[r], __ldg(&tw[r * jm * G.tws]));
    }
    dft_reg<R1>(v);
    if (t < tcount) {
      const int idxD = (j - jm) * R1 + jm;
#pragma unroll
      for (int k = 0; k < R1; ++k) {
        const int kk = idxD + k * R0;
        double2 y = v[k];
        if (G.post_tw && g != 0) y = cmul(y, __ldg(&tw[g * kk]));
        const double2 o = make_double2(y.x * sc, y.y * sci);
        if (ROUTED && job.out_rows) {
          for (int d = 0; d < job.out_ndst; ++d) job.out_rows[d * job.out_rows_stride + kk][t0 + t] = o;
        } else {
          double2* dst = &out[(uint64_t)kk * ostr + t];
          if (job.stream_out) __stcs(dst, o);
          else *dst = o;
        }
      }
    }
  }
}

// Fallback for long tubes with no usable split: one generic Stockham stage per
// launch over global memory (element (r, tube) at [r*ntubes + tube]).
__global__ void tube_fft_global_stage_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                                             uint64_t ntubes, int p, int Ns, int R,
                                             const double2* __restrict__ tw, int conj_in, int conj_out,
                                             double scale) {
  const uint64_t total = (uint64_t)p * ntubes;
  const int pR = p / R;
  const int twmul = p / (Ns * R);
  const double sci = conj_out ? -scale : scale;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < total;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t o = b / ntubes, t = b - o * ntubes;
    const int j = (int)(o / R), k = (int)(o - (uint64_t)j * R);
    const int jm = j % Ns;
    const int base = jm * twmul + k * pR;
    double2 acc = src[(uint64_t)j * ntubes + t];
    if (conj_in) acc.y = -acc.y;
    int e = 0;
    for (int r = 1; r < R; ++r) {
      e += base;
      if (e >= p) e -= p;
      double2 x = src[(uint64_t)(j + r * pR) * ntubes + t];
      if (conj_in) x.y = -x.y;
      const double2 w = __ldg(&tw[e]);
      acc.x = fma(x.x, w.x, fma(-x.y, w.y, acc.x));
      acc.y = fma(x.x, w.y, fma(x.y, w.x, acc.y));
    }
    const int idxD = (j - jm) * R + jm;
    dst[(uint64_t)(idxD + k * Ns) * ntubes + t] = make_double2(acc.x * scale, acc.y * sci);
  }
}

// ------------------------------------------------------------------ launch
namespace {
constexpr int kFftThreads = 256;
constexpr size_t kSmemBudget = 96 * 1024;  // two CTAs per SM
constexpr size_t kSmemMax = 224 * 1024;    // one CTA per SM

bool batch_routed(const TubeBatch& b) {
  for (int i = 0; i < b.njobs; ++i)
    if (b.job[i].in_rows || b.job[i].out_rows) return true;
  return false;
}

// shared-memory buffers the kernel needs for a plan (host mirror of the
// control flow above)
int fft_smem_buffers(const FftPlan& pl) {
  const int S = pl.nstages;
  if (S == 0) return 0;
  const bool r0 = is_reg_radix(pl.radix[0]);
  const bool rl = is_reg_radix(pl.radix[S - 1]);
  if (S == 1 && r0) return 0;
  const int smem_stages = S - (r0 ? 1 : 0) - (rl ? 1 : 0);
  return smem_stages == 0 ? 1 : 2;
}

cudaError_t ensure_smem_attr(int device) {
  static std::mutex mu;
  static bool attr_set[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device >= 0 && device < 64 && !attr_set[device]) {
    cudaError_t e =
        cudaFuncSetAttribute(tube_fft_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tube_fft_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
    if (e != cudaSuccess) return e;
    attr_set[device] = true;
  }
  return cudaSuccess;
}

// tile width: ~2048 elements (32 KB) per tile, >= 8 tubes (128-byte rows)
// when it fits, fewer for tiny jobs; returns -1 if even T = 1 does not fit.
int choose_logT(const FftPlan& pl, int L, uint64_t maxtubes, int njobs, uint64_t groups, size_t* smem) {
  const size_t per_tube = (size_t)fft_smem_buffers(pl) * sizeof(double2) * (size_t)L;
  if (per_tube > kSmemMax) return -1;
  int logT = 0;
  while (logT < 6 && ((size_t)L << (logT + 1)) <= 2048 && (per_tube << (logT + 1)) <= kSmemBudget) ++logT;
  if (logT < 3 && (per_tube << 3) <= kSmemBudget) logT = 3;
  while (logT > 0 && (uint64_t(1) << (logT - 1)) >= maxtubes) --logT;
  while (logT > 3 && (maxtubes >> logT) * (uint64_t)njobs * groups < 296) --logT;
  *smem = per_tube << logT;
  return logT;
}

template <int R0, int R1>
cudaError_t launch_fft2(const TubeBatch& batch, const FftGeom& G, const double2* tw, uint64_t maxtubes, int groups,
                        int njobs, cudaStream_t stream) {
  constexpr int L = R0 * R1;
  // stage 0 has exactly one butterfly per thread at full width (T = 256*R0/L)
  int logT = 0;
  while ((1 << logT) < 256 * R0 / L) ++logT;
  while (logT > 0 && (uint64_t(1) << (logT - 1)) >= maxtubes) --logT;           // tiny jobs
  while (logT > 3 && (maxtubes >> logT) * (uint64_t)njobs * groups < 296) --logT;  // >= 2 CTAs/SM
  const size_t smem = sizeof(double2) * ((size_t)L << logT);
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t attr = once_per_device(mu, done, [] {
    cudaError_t r =
        cudaFuncSetAttribute(tube_fft2_kernel<R0, R1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(tube_fft2_kernel<R0, R1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kSmemMax);
    return r;
  });
  if (attr != cudaSuccess) return attr;
  const uint64_t tiles = (maxtubes + (uint64_t(1) << logT) - 1) >> logT;
  dim3 grid((unsigned)tiles, njobs, groups);
  ProfScope ps("fft", stream);
  if (batch_routed(batch)) tube_fft2_kernel<R0, R1, true><<<grid, kFftThreads, smem, stream>>>(batch, G, tw, logT);
  else tube_fft2_kernel<R0, R1, false><<<grid, kFftThreads, smem, stream>>>(batch, G, tw, logT);
  ps.stop();
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_pass(const TubeBatch& batch, const FftPlan& pl, const FftGeom& G, const double2* tw,
                        uint64_t maxtubes, int groups, int logT, size_t smem, cudaStream_t stream) {
  if (pl.nstages == 2) {
    const int r0 = pl.radix[0], r1 = pl.radix[1];
    if (r0 == 8 && r1 == 8) return launch_fft2<8, 8>(batch, G, tw, maxtubes, groups, batch.njobs, stream);
    if (r0 == 8 && r1 == 4) return launch_fft2<8, 4>(batch, G, tw, maxtubes, groups, batch.njobs, stream);
    if (r0 == 8 && r1 == 2) return launch_fft2<8, 2>(batch, G, tw, maxtubes, groups, batch.njobs, stream);
    if (r0 == 4 && r1 == 2) return launch_fft2<4, 2>(batch, G, tw, maxtubes, groups, batch.njobs, stream);
  }
  const uint64_t tiles = (maxtubes + (uint64_t(1) << logT) - 1) >> logT;
  dim3 grid((unsigned)tiles, batch.njobs, groups);
  ProfScope ps("fft", stream);
  if (batch_routed(batch)) tube_fft_kernel<true><<<grid, kFftThreads, smem, stream>>>(batch, pl, G, tw, logT);
  else tube_fft_kernel<false><<<grid, kFftThreads, smem, stream>>>(batch, pl, G, tw, logT);
  ps.stop();
  count_launches(1);
  return cudaGetLastError();
}

// balanced split p = p1 * p2 (p1 >= p2 > 1) from the prime factors; 0 if prime
void split_length(int p, int* p1, int* p2) {
  std::vector<int> f;
  int r = p;
  for (int d = 2; (long long)d * d <= r; ++d)
    while (r % d == 0) { f.push_back(d); r /= d; }
  if (r > 1) f.push_back(r);
  *p1 = *p2 = 0;
  if (f.size() < 2) return;
  std::sort(f.rbegin(), f.rend());
  long long a = 1, b = 1;
  for (int x : f) (a <= b ? a : b) *= x;
  *p1 = (int)std::max(a, b);
  *p2 = (int)std::min(a, b);
}
}  // namespace

bool fft_single_pass(int p) {
  if (p <= 0) return false;
  const FftPlan plan = make_fft_plan(p);
  const size_t per_tube = (size_t)fft_smem_buffers(plan) * sizeof(double2) * (size_t)p;
  if (per_tube > kSmemMax) return false;
  const bool narrow = (per_tube << 3) > kSmemMax;
  int p1 = 0, p2 = 0;
  if (narrow) split_length(p, &p1, &p2);
  return !(narrow && p1 > 1 && p2 > 1 && p1 <= 2048);
}

bool fft_split_length(int p) {
  if (p <= 0 || fft_single_pass(p)) return false;
  const FftPlan plan = make_fft_plan(p);
  const size_t per_tube = (size_t)fft_smem_buffers(plan) * sizeof(double2) * (size_t)p;
  const bool narrow = per_tube > kSmemMax || (per_tube << 3) > kSmemMax;
  int p1 = 0, p2 = 0;
  if (narrow) split_length(p, &p1, &p2);
  if (!(p1 > 1 && p2 > 1 && p1 <= 2048)) return false;
  const FftPlan pl1 = make_fft_plan(p1), pl2 = make_fft_plan(p2);
  size_t sm = 0;
  return choose_logT(pl1, p1, 1, 1, 1, &sm) >= 0 && choose_logT(pl2, p2, 1, 1, 1, &sm) >= 0;
}

cudaError_t launch_tube_fft(const TubeBatch& batch, int p, cudaStream_t stream, int device) {
  if (batch.njobs == 0) return cudaSuccess;
  uint64_t maxtubes = 0;
  for (int i = 0; i < batch.njobs; ++i) maxtubes = std::max(maxtubes, batch.job[i].ntubes);
  if (maxtubes == 0) return cudaSuccess;
  const double2* tw = twiddles_for(device, p, stream);
  if (!tw) return cudaErrorMemoryAllocation;
  cudaError_t e = ensure_smem_attr(device);
  if (e != cudaSuccess) return e;

  // 1) single pass when a >= 8-tube tile fits in shared memory.  The choice
  // between single pass and split depends on p ONLY (never on the number of
  // tubes), so every tube is transformed with the same arithmetic whatever the
  // batch — results stay bitwise identical across row/column shardings.
  const FftPlan plan = make_fft_plan(p);
  size_t smem = 0;
  int logT = choose_logT(plan, p, maxtubes, batch.njobs, 1, &smem);
  const size_t per_tube = (size_t)fft_smem_buffers(plan) * sizeof(double2) * (size_t)p;
  const bool narrow = per_tube > kSmemMax || (per_tube << 3) > kSmemMax;  // no 8-tube tile fits
  int p1 = 0, p2 = 0;
  if (narrow) split_length(p, &p1, &p2);
  const bool split_ok = p1 > 1 && p2 > 1 && p1 <= 2048;
  if (logT >= 0 && !(narrow && split_ok)) {
    const FftGeom G{p, 0, 1, 0, 1, 0, 1};
    return launch_pass(batch, plan, G, tw, maxtubes, 1, logT, smem, stream);
  }
  // routed rows exist for the single-pass transform only
  if (batch_routed(batch)) return cudaErrorNotSupported;

  // 2) four-step split p = p1 * p2 through a scratch plane per job
  if (split_ok) {
    const FftPlan pl1 = make_fft_plan(p1), pl2 = make_fft_plan(p2);
    size_t sm1 = 0, sm2 = 0;
    const int lt1 = choose_logT(pl1, p1, maxtubes, batch.njobs, p2, &sm1);
    const int lt2 = choose_logT(pl2, p2, maxtubes, batch.njobs, p1, &sm2);
    if (lt1 >= 0 && lt2 >= 0) {
      uint64_t total = 0;
      for (int i = 0; i < batch.njobs; ++i) total += batch.job[i].ntubes * (uint64_t)p;
      double2* scratch = nullptr;
      if ((e = cudaMallocAsync(&scratch, total * sizeof(double2), stream)) != cudaSuccess) return e;
      TubeBatch A = batch, B = batch;
      uint64_t off = 0;
      for (int i = 0; i < batch.njobs; ++i) {
        const TubeJob& J = batch.job[i];
        // pass A: conj-in, no output ops, into scratch
        A.job[i].out = scratch + off;
        A.job[i].conj_out = 0;
        A.job[i].scale = 1.0;
        // pass B: from scratch, output ops of the job; its output streams past L2
        B.job[i].in = scratch + off;
        B.job[i].conj_in = 0;
        B.job[i].out = J.out;
        B.job[i].stream_out = 1;
        off += J.ntubes * (uint64_t)p;
      }
      const FftGeom GA{p1, 1, p2, 1, p2, 1, p2};  // rows g + p2*i -> g + p2*k, twiddle W_p^(g*k)
      const FftGeom GB{p2, p2, 1, 1, p1, 0, p1};  // rows p2*g + i -> g + p1*k
      e = launch_pass(A, pl1, GA, tw, maxtubes, p2, lt1, sm1, stream);
      if (e == cudaSuccess) e = launch_pass(B, pl2, GB, tw, maxtubes, p1, lt2, sm2, stream);
      cudaError_t fe = cudaFreeAsync(scratch, stream);
      return e != cudaSuccess ? e : fe;
    }
  }
  if (logT >= 0) {  // narrow tile but no split: still correct
    const FftGeom G{p, 0, 1, 0, 1, 0, 1};
    return launch_pass(batch, plan, G, tw, maxtubes, 1, logT, smem, stream);
  }

  // 3) global multi-pass path (long prime-ish lengths): one launch per stage per job
  for (int i = 0; i < batch.njobs; ++i) {
    const TubeJob& J = batch.job[i];
    if (J.ntubes == 0) continue;
    const size_t bytes = sizeof(double2) * (size_t)p * J.ntubes;
    double2* scratch = nullptr;
    e = cudaMallocAsync(&scratch, 2 * bytes, stream);
    if (e != cudaSuccess) return e;
    double2* bufs[2] = {scratch, scratch + (size_t)p * J.ntubes};
    const double2* src = J.in;
    int Ns = 1;
    for (int s = 0; s < plan.nstages; ++s) {
      const bool first = s == 0, last = s == plan.nstages - 1;
      // a single in-place stage must not write the buffer it is reading
      const bool bounce = last && first && J.in == J.out;
      double2* dst = (last && !bounce) ? J.out : bufs[s & 1];
      const uint64_t tot = (uint64_t)p * J.ntubes;
      const unsigned blocks = (unsigned)std::min<uint64_t>((tot + 255) / 256, 148ull * 16);
      ProfScope ps("fft", stream);
      tube_fft_global_stage_kernel<<<blocks, 256, 0, stream>>>(src, dst, J.ntubes, p, Ns, plan.radix[s], tw,
                                                               first ? J.conj_in : 0, last ? J.conj_out : 0,
                                                               last ? J.scale : 1.0);
      ps.stop();
      count_launches(1);
      if (bounce) {
        cudaError_t ce = cudaMemcpyAsync(J.out, dst, bytes, cudaMemcpyDeviceToDevice, stream);
        if (ce != cudaSuccess) return ce;
      }
      src = dst;
      Ns *= plan.radix[s];
    }
    e = cudaFreeAsync(scratch, stream);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace qtb
