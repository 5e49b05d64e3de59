// qt_gemm.cu — K2: paired-frequency quaternion block GEMM on FP64 DMMA (sm_100a).
//
// Replaces the slice loop of tprod_fast (/root/reference/proj/src/tproduct.cpp:90-104),
// which for every frequency i (ri = slice_reflect(i, p) = (p - i) % p) runs
//     C1_i = Â1_i·B̂1_i − conj(Â2_ri)·B̂2_i
//     C2_i = conj(Â1_ri)·B̂2_i + Â2_i·B̂1_i
// as four i-k-j complex MAC loops (slice_gemm_acc, tproduct.cpp:57-71).
//
// Here one CTA owns a BM x BN tile of the output for the frequency PAIR
// (k, σk), σk = (p - k) % p.  The four Â slices Â1_k, Â2_k, Â1_σk, Â2_σk are
// staged once per K-step and feed both frequencies:
//     C1_k  = Â1_k ·B̂1_k  − conj(Â2_σk)·B̂2_k      C2_k  = conj(Â1_σk)·B̂2_k  + Â2_k ·B̂1_k
//     C1_σk = Â1_σk·B̂1_σk − conj(Â2_k) ·B̂2_σk     C2_σk = conj(Â1_k) ·B̂2_σk + Â2_σk·B̂1_σk
// Self-paired frequencies (k = 0 and k = p/2 for even p) run the SELF variant
// that computes one frequency.  Each complex product is four real products
// issued as `mma.sync.m8n8k4.f64` (SASS DMMA.8x8x4, the FP64 tensor pipe —
// tcgen05 has no f64 kind); conjugation and the minus signs are sign-bit XORs
// on the B fragments (ALU pipe), so the FP64 pipe only ever sees DMMA.
//
// Two tile shapes: the main one (64 x 16 tile, 8 warps, 2 CTAs/SM) for
// GEMM-sized slices, and a small one (16 x 16 tile, whole K <= 16 per stage,
// 4 warps) for many tiny slices (long tubes, e.g. m = n = s = 16, p = 4096).
//
// Determinism: no split-K, no atomics; each accumulator adds its four terms in
// a fixed order for K-steps 0..n-1, independent of the M/N tiling and of the
// tile shape, so results are bitwise reproducible and identical across row
// shardings.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "qt_dmma_tile.cuh"
#include "qt_internal.cuh"

namespace qtb {

namespace {

template <class C, bool SELF>
__device__ __forceinline__ void pair_tile(const PairArgs& P, int row0, int col0, int m, int n, int s, int ldb,
                                          int ldc) {
  extern __shared__ double2 smem[];
  constexpr int NC = SELF ? 4 : 8;  // accumulated real components
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp % C::WM, wn = warp / C::WM;

  double acc[NC][C::RB][2];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb) acc[c][rb][0] = acc[c][rb][1] = 0.0;

  const int ktiles = (n + C::BK - 1) / C::BK;
#pragma unroll
  for (int st = 0; st < C::STAGES - 1; ++st) {
    if (st < ktiles) load_stage<C, SELF>(smem + st * C::STAGE_ELEMS, P, st, row0, col0, m, n, s, ldb);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + C::STAGES - 1;
      if (nk < ktiles) load_stage<C, SELF>(smem + (nk % C::STAGES) * C::STAGE_ELEMS, P, nk, row0, col0, m, n, s, ldb);
      cp_async_commit();
    }
    const double2* sa = smem + (kt % C::STAGES) * C::STAGE_ELEMS;
    mma_stage<C, SELF>(sa, sa + 4 * C::A_PLANE, acc, wm, wn, g, q);
  }
  cp_async_wait<0>();
  store_tile<C, SELF>(P, acc, row0, col0, m, s, ldc, wm, wn, g, q);
}

__device__ __forceinline__ PairArgs pair_args(const double2* ah1, const double2* ah2, const double2* bh1,
                                              const double2* bh2, double2* ch1, double2* ch2, int k, int sg,
                                              size_t amn, size_t bns, size_t cms) {
  PairArgs P;
  P.a[0] = ah1 + k * amn;
  P.a[1] = ah2 + k * amn;
  P.a[2] = ah1 + sg * amn;
  P.a[3] = ah2 + sg * amn;
  P.b[0] = bh1 + k * bns;
  P.b[1] = bh2 + k * bns;
  P.b[2] = bh1 + sg * bns;
  P.b[3] = bh2 + sg * bns;
  P.c[0] = ch1 + k * cms;
  P.c[1] = ch2 + k * cms;
  P.c[2] = ch1 + sg * cms;
  P.c[3] = ch2 + sg * cms;
  return P;
}

// Persistent variant for many tiny slices whose whole K fits one stage
// (n <= BK, e.g. m = n = s = 16 with p = 4096): each CTA walks work items
// (pair, tile) with a two-deep cp.async ring ACROSS items, so the loads of item
// i+1 overlap the DMMAs of item i and there is no wave-quantisation tail.
// Self-paired frequencies run the general formulas with σk = k, which
// evaluate the same operands in the same order as the SELF variant and store
// the same values twice to the same place (bitwise identical to pair_tile).
template <class C>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
    paired_small_persistent_kernel(const double2* __restrict__ ah1, const double2* __restrict__ ah2,
                                   const double2* __restrict__ bh1, const double2* __restrict__ bh2,
                                   double2* __restrict__ ch1, double2* __restrict__ ch2, int m, int n, int s, int p,
                                   int ldb, int ldc, long long bslice, long long cslice) {
  extern __shared__ double2 smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp % C::WM, wn = warp / C::WM;
  const int ntm = (m + C::BM - 1) / C::BM, ntn = (s + C::BN - 1) / C::BN;
  const long long tiles = (long long)ntm * ntn;
  const long long items = (long long)(p / 2 + 1) * tiles;
  const size_t amn = (size_t)m * n;
  auto item_args = [&](long long w, int* row0, int* col0) {
    const int k = (int)(w / tiles);
    const int t = (int)(w - (long long)k * tiles);
    *row0 = (t % ntm) * C::BM;
    *col0 = (t / ntm) * C::BN;
    return pair_args(ah1, ah2, bh1, bh2, ch1, ch2, k, (p - k) % p, amn, (size_t)bslice, (size_t)cslice);
  };
  long long w = blockIdx.x;
  if (w >= items) return;
  int r0, c0;
  PairArgs P = item_args(w, &r0, &c0);
  load_stage<C, false>(smem, P, 0, r0, c0, m, n, s, ldb);
  cp_async_commit();
  for (int it = 0; w < items; ++it, w += gridDim.x) {
    const long long wn_ = w + gridDim.x;
    int nr0 = 0, nc0 = 0;
    if (wn_ < items) {
      const PairArgs Pn = item_args(wn_, &nr0, &nc0);
      load_stage<C, false>(smem + ((it + 1) & 1) * C::STAGE_ELEMS, Pn, 0, nr0, nc0, m, n, s, ldb);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double acc[8][C::RB][2];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int rb = 0; rb < C::RB; ++rb) acc[c][rb][0] = acc[c][rb][1] = 0.0;
    const double2* sa = smem + (it & 1) * C::STAGE_ELEMS;
    mma_stage<C, false>(sa, sa + 4 * C::A_PLANE, acc, wm, wn, g, q);
    store_tile<C, false>(P, acc, r0, c0, m, s, ldc, wm, wn, g, q);
    __syncthreads();  // buffer (it & 1) is refilled by the next iteration's prefetch
    if (wn_ < items) {
      P = item_args(wn_, &r0, &c0);
    }
  }
  cp_async_wait<0>();
}

// Tile rasterisation: a CTA's linear index walks GROUP_M row tiles fastest
// inside a band of the output, so the ~300 co-resident CTAs cover a squarish
// GROUP_M x ~37 block of tiles and share both their Â rows and their B̂
// columns through L2 (the plain column-fastest order re-reads B̂ from HBM once
// per row tile: 146 GB vs 67 GB of DRAM reads per launch on config 5).
constexpr int GROUP_M = 8;

template <class C>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
    paired_spectral_gemm_kernel(const double2* __restrict__ ah1, const double2* __restrict__ ah2,
                                const double2* __restrict__ bh1, const double2* __restrict__ bh2,
                                double2* __restrict__ ch1, double2* __restrict__ ch2, int m, int n, int s, int p,
                                int pair0, int ldb, int ldc, long long bslice, long long cslice) {
  const int k = pair0 + blockIdx.y;
  const int sg = (p - k) % p;
  const int ntm = (m + C::BM - 1) / C::BM, ntn = (s + C::BN - 1) / C::BN;
  const int bid = blockIdx.x;
  const int per_group = GROUP_M * ntn;
  const int grp = bid / per_group;
  const int first_m = grp * GROUP_M;
  const int gsz = min(GROUP_M, ntm - first_m);
  const int w = bid - grp * per_group;
  const int tm = first_m + w % gsz, tn = w / gsz;
  const size_t amn = (size_t)m * n, bns = (size_t)bslice, cms = (size_t)cslice;
  const PairArgs P = pair_args(ah1, ah2, bh1, bh2, ch1, ch2, k, sg, amn, bns, cms);
  const int row0 = tm * C::BM, col0 = tn * C::BN;
  if (sg == k) pair_tile<C, true>(P, row0, col0, m, n, s, ldb, ldc);
  else pair_tile<C, false>(P, row0, col0, m, n, s, ldb, ldc);
}

template <class C>
cudaError_t launch_cfg(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2, double2* ch1,
                       double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, uint64_t ldb, uint64_t ldc,
                       uint64_t bslice, uint64_t cslice, cudaStream_t stream) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(paired_spectral_gemm_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)C::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const uint64_t npairs = p / 2 + 1;
  const uint64_t tiles = ((m + C::BM - 1) / C::BM) * ((s + C::BN - 1) / C::BN);
  // a K that fits one stage (e.g. n <= 16 on the small tile) needs one buffer only
  const uint64_t ktiles = (n + C::BK - 1) / C::BK;
  const size_t smem = (size_t)std::min<uint64_t>(C::STAGES, std::max<uint64_t>(1, ktiles)) * C::STAGE_ELEMS * 16;
  if (tiles > 0x7fffffffULL) return cudaErrorInvalidConfiguration;
  for (uint64_t k0 = 0; k0 < npairs; k0 += 65535) {
    const unsigned chunk = (unsigned)std::min<uint64_t>(65535, npairs - k0);
    dim3 grid((unsigned)tiles, chunk);
    paired_spectral_gemm_kernel<C><<<grid, C::NTHREADS, smem, stream>>>(
        ah1, ah2, bh1, bh2, ch1, ch2, (int)m, (int)n, (int)s, (int)p, (int)k0, (int)ldb, (int)ldc, (long long)bslice,
        (long long)cslice);
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_small_persistent(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                    double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                    uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice,
                                    cudaStream_t stream) {
  using C = SmallCfg;
  auto kern = paired_small_persistent_kernel<C>;
  const size_t smem = 2 * (size_t)C::STAGE_ELEMS * 16;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  static int per_sm = 1, sms = 148;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (attr_err == cudaSuccess)
      attr_err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NTHREADS, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const uint64_t tiles = ((m + C::BM - 1) / C::BM) * ((s + C::BN - 1) / C::BN);
  const uint64_t items = (p / 2 + 1) * tiles;
  const uint64_t grid = std::min<uint64_t>(items, (uint64_t)std::max(1, per_sm) * sms);
  kern<<<(unsigned)grid, C::NTHREADS, smem, stream>>>(ah1, ah2, bh1, bh2, ch1, ch2, (int)m, (int)n, (int)s, (int)p,
                                                       (int)ldb, (int)ldc, (long long)bslice, (long long)cslice);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_spectral_gemm_ld(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                    double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                    uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice, cudaStream_t stream) {
  if (m == 0 || s == 0 || p == 0) return cudaSuccess;
  // Small slices (m, s <= 32): the 64-row tile would waste >= half its DMMAs
  // and its two-deep K pipeline would be all latency; use the 16 x 16 tile.
  if (m <= 32 && s <= 32) {
    if (n <= (uint64_t)SmallCfg::BK)
      return launch_small_persistent(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream);
    return launch_cfg<SmallCfg>(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream);
  }
  return launch_cfg<BigCfg>(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream);
}

cudaError_t launch_spectral_gemm(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                 double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                 cudaStream_t stream) {
  return launch_spectral_gemm_ld(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, s, s, n * s, m * s, stream);
}

}  // namespace qtb
