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
#include <cstdlib>
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

// ---------------------------------------------------------------------------
// Gauss's 3-multiplication complex product on the DMMA pipe.  For a term
// s * op(X) * Y with op(X) = xr + i*sig*xi (sig = -1 for conj) and Y = yr + i*yi:
//     T1 += s*xr*yr,  T2 += s*(sig*xi)*yi,  T3 += s*(xr + sig*xi)*(yr + yi)
// and at the end  Re = T1 - T2,  Im = T3 - T1 - T2.  Both complex products of
// every output (e.g. C1_k = Â1_k B̂1_k - conj(Â2_σ) B̂2_k) accumulate into the
// same three sums, so each output costs 6 DMMAs per K-step instead of 8: 24
// instead of 32 per frequency pair and 8-row block.  The operand sums
// (xr +- xi, yr + yi) are 12 DADDs per 24 DMMAs on the shared FP64 pipe.  The
// flop count the metric uses stays the reference's (32 m n s p); the kernel
// executes 24 m n s p (+ the DADDs).
template <class C, bool SELF>
__device__ __forceinline__ void mma_stage_3m(const double2* sa, const double2* sb,
                                             double (&T)[SELF ? 6 : 12][C::RB][2], int wm, int wn, int g, int q) {
#pragma unroll
  for (int ks = 0; ks < C::BK / 4; ++ks) {
    const int kb = ks * 4 + q;
    const int jb = (wn * 8 + g) ^ (q << 1);
    double br[4], bi[4], bp[4];
#pragma unroll
    for (int pl = 0; pl < (SELF ? 2 : 4); ++pl) {
      const double2 v = sb[pl * C::B_PLANE + kb * C::BN + jb];
      br[pl] = v.x;
      bi[pl] = v.y;
      bp[pl] = v.x + v.y;
    }
    // planes: 0 B1k, 1 B2k, 2 B1s, 3 B2s
    const double nb2k_r = dneg(br[1]), nb2k_i = dneg(bi[1]), nb2k_p = dneg(bp[1]);
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb) {
      const int i = wm * (C::RB * 8) + rb * 8 + g;
      const int ca = (ks * 4 + q) ^ ((i & 1) << 2);
      double ar[4], ai[4], ap[4], am[4];  // planes: 0 A1k, 1 A2k, 2 A1s, 3 A2s
#pragma unroll
      for (int pl = 0; pl < (SELF ? 2 : 4); ++pl) {
        const double2 v = sa[pl * C::A_PLANE + i * C::BK + ca];
        ar[pl] = v.x;
        ai[pl] = v.y;
        ap[pl] = v.x + v.y;
        am[pl] = v.x - v.y;
      }
      if (SELF) {
        ar[2] = ar[0]; ai[2] = ai[0]; ap[2] = ap[0]; am[2] = am[0];
        ar[3] = ar[1]; ai[3] = ai[1]; ap[3] = ap[1]; am[3] = am[1];
      }
      // Term order per T set is fixed (first product, then second), but the
      // 12 independent sets are interleaved so consecutive DMMAs never depend
      // on each other.  Sets: C1_k = A1k B1k - conj(A2s) B2k (0..2),
      // C2_k = conj(A1s) B2k + A2k B1k (3..5), C1_s = A1s B1s - conj(A2k) B2s
      // (6..8), C2_s = conj(A1k) B2s + A2s B1s (9..11); each (T1, T2, T3).
      constexpr int NT = SELF ? 6 : 12;
      dmma(T[0][rb], ar[0], br[0]);
      dmma(T[1][rb], ai[0], bi[0]);
      dmma(T[2][rb], ap[0], bp[0]);
      dmma(T[3][rb], ar[2], br[1]);
      dmma(T[4][rb], ai[2], nb2k_i);
      dmma(T[5][rb], am[2], bp[1]);
      if (!SELF) {
        dmma(T[6 % NT][rb], ar[2], br[2]);
        dmma(T[7 % NT][rb], ai[2], bi[2]);
        dmma(T[8 % NT][rb], ap[2], bp[2]);
        dmma(T[9 % NT][rb], ar[0], br[3]);
        dmma(T[10 % NT][rb], ai[0], dneg(bi[3]));
        dmma(T[11 % NT][rb], am[0], bp[3]);
      }
      dmma(T[0][rb], ar[3], nb2k_r);
      dmma(T[1][rb], ai[3], bi[1]);
      dmma(T[2][rb], am[3], nb2k_p);
      dmma(T[3][rb], ar[1], br[0]);
      dmma(T[4][rb], ai[1], bi[0]);
      dmma(T[5][rb], ap[1], bp[0]);
      if (!SELF) {
        dmma(T[6 % NT][rb], ar[1], dneg(br[3]));
        dmma(T[7 % NT][rb], ai[1], bi[3]);
        dmma(T[8 % NT][rb], am[1], dneg(bp[3]));
        dmma(T[9 % NT][rb], ar[3], br[2]);
        dmma(T[10 % NT][rb], ai[3], bi[2]);
        dmma(T[11 % NT][rb], ap[3], bp[2]);
      }
    }
  }
}

// epilogue of the 3M variant: Re = T1 - T2, Im = T3 - T1 - T2 per output
template <class C, bool SELF>
__device__ __forceinline__ void store_tile_3m(const PairArgs& P, const double (&T)[SELF ? 6 : 12][C::RB][2],
                                              int row0, int col0, int m, int s, int ldc, int wm, int wn, int g,
                                              int q) {
  constexpr int NT = SELF ? 6 : 12;
  const int col = col0 + wn * 8 + 2 * q;
#pragma unroll
  for (int o = 0; o < (SELF ? 2 : 4); ++o) {
    double2* Cp = P.c[o];  // outputs in P.c order: C1_k, C2_k, C1_s, C2_s
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb) {
      const int row = row0 + wm * (C::RB * 8) + rb * 8 + g;
      if (row < m) {
        double2* dst = Cp + (size_t)row * ldc + col;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double t1 = T[(3 * o) % NT][rb][e], t2 = T[(3 * o + 1) % NT][rb][e], t3 = T[(3 * o + 2) % NT][rb][e];
          if (col + e < s) dst[e] = make_double2(t1 - t2, t3 - t1 - t2);
        }
      }
    }
  }
}

template <class C, bool SELF>
__device__ __forceinline__ void pair_tile_3m(const PairArgs& P, int row0, int col0, int m, int n, int s, int ldb,
                                             int ldc) {
  extern __shared__ double2 smem[];
  constexpr int NT = SELF ? 6 : 12;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp % C::WM, wn = warp / C::WM;
  double T[NT][C::RB][2];
#pragma unroll
  for (int c = 0; c < NT; ++c)
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb) T[c][rb][0] = T[c][rb][1] = 0.0;
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
    mma_stage_3m<C, SELF>(sa, sa + 4 * C::A_PLANE, T, wm, wn, g, q);
  }
  cp_async_wait<0>();
  store_tile_3m<C, SELF>(P, T, row0, col0, m, s, ldc, wm, wn, g, q);
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

// Work unit u of a launch -> the slices of its pair (ka, kb; ka == kb for a
// self-paired frequency) and its flag key min(k, p - k).  Frequency mode
// (s0 < 0): u = k in [0, p/2], slices are frequencies.  Compact mode: the
// operands hold the frequency slots [s0, s0 + ns) (slice t = slot s0 + t) and
// u walks that range's pair / self-paired units (qt_int8_slots_*).
// noreflect: the negative control of the parity tests ($QTB_DEBUG_NO_REFLECT=1):
// sigma(k) = k instead of slice_reflect (tproduct.hpp:27-29), i.e. the
// quaternion product treated as if j commuted with the complex scalars —
// every frequency then runs as its own "pair" and parity must fail.
struct PairMap {
  int s0 = -1, ns = 0;
  int noreflect = 0;
};
__device__ __forceinline__ void map_unit(int u, const PairMap& M, int p, int& ka, int& kb, int& key) {
  if (M.noreflect) {
    ka = kb = key = u;
    return;
  }
  if (M.s0 < 0) {
    ka = u;
    kb = (p - u) % p;
    key = u;
    return;
  }
  int sa, sb;
  unit_slots(u, M.s0, M.ns, p, sa, sb);
  ka = sa - M.s0;
  kb = sb - M.s0;
  const int f = slot_frequency(sa, p);
  key = min(f, p - f);
}
// int8 fallback: the CTA's pair runs only if the inputs were non-finite or the
// accuracy guard flagged it (only_if[0] / only_if[1 + key]); nullptr: always
__device__ __forceinline__ bool skip_unit(const int* only_if, int key) {
  return only_if != nullptr && only_if[0] == 0 && only_if[1 + key] == 0;
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
                                   int ldb, int ldc, long long bslice, long long cslice, const int* only_if,
                                   PairMap map, int units) {
  extern __shared__ double2 smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp % C::WM, wn = warp / C::WM;
  const int ntm = (m + C::BM - 1) / C::BM, ntn = (s + C::BN - 1) / C::BN;
  const long long tiles = (long long)ntm * ntn;
  const long long items = (long long)units * tiles;
  const size_t amn = (size_t)m * n;
  auto item_args = [&](long long w, int* row0, int* col0) {
    const int u = (int)(w / tiles);
    const int t = (int)(w - (long long)u * tiles);
    *row0 = (t % ntm) * C::BM;
    *col0 = (t / ntm) * C::BN;
    int ka, kb, key;
    map_unit(u, map, p, ka, kb, key);
    return pair_args(ah1, ah2, bh1, bh2, ch1, ch2, ka, kb, amn, (size_t)bslice, (size_t)cslice);
  };
  // int8 fallback: only the flagged pairs' items run (the others are skipped
  // wholesale; the ring then just prefetches fewer items)
  auto live = [&](long long w) {
    if (only_if == nullptr) return true;
    int ka, kb, key;
    map_unit((int)(w / tiles), map, p, ka, kb, key);
    return !skip_unit(only_if, key);
  };
  constexpr int D = C::STAGES;  // ring depth: items prefetched D - 1 ahead
  const long long G = gridDim.x;
  long long w = blockIdx.x;
  if (w >= items) return;
#pragma unroll
  for (int d = 0; d < D - 1; ++d) {
    const long long wd = w + d * G;
    if (wd < items && live(wd)) {
      int lr, lc;
      const PairArgs Pd = item_args(wd, &lr, &lc);
      load_stage<C, false>(smem + d * C::STAGE_ELEMS, Pd, 0, lr, lc, m, n, s, ldb);
    }
    cp_async_commit();
  }
  for (int it = 0; w < items; ++it, w += G) {
    {
      const long long wp = w + (D - 1) * G;
      if (wp < items && live(wp)) {
        int lr, lc;
        const PairArgs Pp = item_args(wp, &lr, &lc);
        load_stage<C, false>(smem + ((it + D - 1) % D) * C::STAGE_ELEMS, Pp, 0, lr, lc, m, n, s, ldb);
      }
      cp_async_commit();
    }
    cp_async_wait<D - 1>();
    __syncthreads();
    if (!live(w)) {  // (block-uniform) nothing was loaded for this item
      __syncthreads();
      continue;
    }
    int r0, c0;
    const PairArgs P = item_args(w, &r0, &c0);
    const double2* sa = smem + (it % D) * C::STAGE_ELEMS;
    if constexpr (C::GAUSS) {
      double T[12][C::RB][2];
#pragma unroll
      for (int c = 0; c < 12; ++c)
#pragma unroll
        for (int rb = 0; rb < C::RB; ++rb) T[c][rb][0] = T[c][rb][1] = 0.0;
      mma_stage_3m<C, false>(sa, sa + 4 * C::A_PLANE, T, wm, wn, g, q);
      store_tile_3m<C, false>(P, T, r0, c0, m, s, ldc, wm, wn, g, q);
    } else {
      double acc[8][C::RB][2];
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int rb = 0; rb < C::RB; ++rb) acc[c][rb][0] = acc[c][rb][1] = 0.0;
      mma_stage<C, false>(sa, sa + 4 * C::A_PLANE, acc, wm, wn, g, q);
      store_tile<C, false>(P, acc, r0, c0, m, s, ldc, wm, wn, g, q);
    }
    __syncthreads();  // buffer (it % D) is refilled by a later iteration's prefetch
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
                                int pair0, int ldb, int ldc, long long bslice, long long cslice, const int* only_if,
                                PairMap map) {
  int k, sg, key;
  map_unit(pair0 + blockIdx.y, map, p, k, sg, key);
  if (skip_unit(only_if, key)) return;  // int8 path certified this pair (qt_ozaki.cu)
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
  if constexpr (C::GAUSS) {
    if (sg == k) pair_tile_3m<C, true>(P, row0, col0, m, n, s, ldb, ldc);
    else pair_tile_3m<C, false>(P, row0, col0, m, n, s, ldb, ldc);
  } else {
    if (sg == k) pair_tile<C, true>(P, row0, col0, m, n, s, ldb, ldc);
    else pair_tile<C, false>(P, row0, col0, m, n, s, ldb, ldc);
  }
}

template <class C>
cudaError_t launch_cfg(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2, double2* ch1,
                       double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p, uint64_t ldb, uint64_t ldc,
                       uint64_t bslice, uint64_t cslice, cudaStream_t stream, const int* only_if = nullptr,
                       PairMap map = PairMap{}) {
  static std::mutex mu;
  static uint64_t done = 0;
  const cudaError_t attr_err = once_per_device(mu, done, [] {
    return cudaFuncSetAttribute(paired_spectral_gemm_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)C::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const uint64_t npairs =
      map.noreflect ? p : map.s0 < 0 ? p / 2 + 1 : (uint64_t)slot_units(map.s0, map.ns, (int)p);
  const uint64_t tiles = ((m + C::BM - 1) / C::BM) * ((s + C::BN - 1) / C::BN);
  // a K that fits one stage (e.g. n <= 16 on the small tile) needs one buffer only
  const uint64_t ktiles = (n + C::BK - 1) / C::BK;
  const size_t smem = (size_t)std::min<uint64_t>(C::STAGES, std::max<uint64_t>(1, ktiles)) * C::STAGE_ELEMS * 16;
  if (tiles > 0x7fffffffULL) return cudaErrorInvalidConfiguration;
  for (uint64_t k0 = 0; k0 < npairs; k0 += 65535) {
    const unsigned chunk = (unsigned)std::min<uint64_t>(65535, npairs - k0);
    dim3 grid((unsigned)tiles, chunk);
    ProfScope ps(only_if ? "k2_dmma_guard" : "k2_dmma", stream);
    paired_spectral_gemm_kernel<C><<<grid, C::NTHREADS, smem, stream>>>(
        ah1, ah2, bh1, bh2, ch1, ch2, (int)m, (int)n, (int)s, (int)p, (int)k0, (int)ldb, (int)ldc, (long long)bslice,
        (long long)cslice, only_if, map);
    ps.stop();
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Every tile shape uses the same complex-product algorithm, so each element of
// C is computed with the same arithmetic whatever m, s or the sharding: Gauss
// 3M by default; $QTB_GEMM=4m selects the 4-multiplication kernels everywhere.
bool gauss_enabled() {
  static const bool on = [] {
    const char* e = getenv("QTB_GEMM");
    return !(e && (e[0] == '4'));
  }();
  return on;
}

template <class C>
cudaError_t launch_small_persistent(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                    double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                    uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice,
                                    cudaStream_t stream, const int* only_if = nullptr, PairMap map = PairMap{}) {
  auto kern = paired_small_persistent_kernel<C>;
  const size_t smem = (size_t)C::STAGES * C::STAGE_ELEMS * 16;
  static std::mutex mu;
  static uint64_t done = 0;
  static int per_sm = 1, sms = 148;  // identical on every B200
  const cudaError_t attr_err = once_per_device(mu, done, [&] {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NTHREADS, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return e;
  });
  if (attr_err != cudaSuccess) return attr_err;
  const uint64_t tiles = ((m + C::BM - 1) / C::BM) * ((s + C::BN - 1) / C::BN);
  const uint64_t units =
      map.noreflect ? p : map.s0 < 0 ? p / 2 + 1 : (uint64_t)slot_units(map.s0, map.ns, (int)p);
  const uint64_t items = units * tiles;
  if (items == 0) return cudaSuccess;
  const uint64_t grid = std::min<uint64_t>(items, (uint64_t)std::max(1, per_sm) * sms);
  ProfScope ps(only_if ? "k2_dmma_guard" : "k2_dmma", stream);
  kern<<<(unsigned)grid, C::NTHREADS, smem, stream>>>(ah1, ah2, bh1, bh2, ch1, ch2, (int)m, (int)n, (int)s, (int)p,
                                                       (int)ldb, (int)ldc, (long long)bslice, (long long)cslice,
                                                       only_if, map, (int)units);
  ps.stop();
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Warp-specialised persistent variant for tiny slices that are whole tiles
// (m, s <= 16, n <= 16, contiguous slices: e.g. config 3, 16 x 16 x 16 with
// p = 4096 -> 2049 pair products of 32 KB operands each).  The cp.async ring
// of paired_small_persistent_kernel keeps one item in flight per CTA and all
// 128 threads issue its 2048 16-byte copies; here ONE producer warp streams
// each item's eight operand slices (four of Â, four of B̂, each one contiguous
// m*n or n*s block) with bulk copies (cp.async.bulk, mbarrier complete_tx)
// into a kTinyStages-deep ring, and three groups of four consumer warps take
// turns on the items, so several items' loads are in flight while up to three
// are on the DMMA pipe.  Operands sit in shared memory unswizzled (each slice
// as it is in HBM; padded rows through per-row copies were measured 2.6x
// slower: 128 small bulk copies per item starve the consumers); out-of-range
// rows / K / columns read +0, as the zero-filled cp.async tiles.  Every accumulator gets exactly mma_stage_3m's DMMA sequence (sets
// 0-11, K-steps of 4 over the 16-wide K tile), and the epilogue is
// store_tile_3m's, so results are bitwise those of the other kernels.
constexpr int kTinyStages = 6;
constexpr int kTinySlice = 256;                    // double2 per operand slice (16 x 16 max)
constexpr int kTinyItem = 8 * kTinySlice;          // 32 KB per item
constexpr int kTinyGroups = 3;
constexpr int kTinyConsumers = 4 * kTinyGroups;    // warps 0-11: three groups of four
constexpr int kTinyThreads = 32 * (kTinyConsumers + 1);  // + warp 8: producer
constexpr size_t kTinySmem = (size_t)kTinyStages * kTinyItem * sizeof(double2);

__device__ __forceinline__ void tiny_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tiny_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tiny_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tiny_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tiny_bulk_load(double2* dst, const double2* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(kTinyThreads, 1)
    paired_tiny_ws_kernel(const double2* __restrict__ ah1, const double2* __restrict__ ah2,
                          const double2* __restrict__ bh1, const double2* __restrict__ bh2, double2* __restrict__ ch1,
                          double2* __restrict__ ch2, int m, int n, int s, int p, const int* only_if, PairMap map,
                          int units) {
  extern __shared__ double2 smem[];
  __shared__ __align__(8) uint64_t full[kTinyStages], empty[kTinyStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t amn = (size_t)m * n, bns = (size_t)n * s, cms = (size_t)m * s;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kTinyStages; ++st) {
      tiny_mbar_init(&full[st], 1);
      tiny_mbar_init(&empty[st], 4);  // the four warps of the consuming group
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  if (warp == kTinyConsumers) {  // ---- producer
    if (lane == 0) {
      const uint32_t abytes = (uint32_t)(amn * 16), bbytes = (uint32_t)(bns * 16);
      for (int i = 0;; ++i) {
        const int w = blockIdx.x + i * G;
        if (w >= units) break;
        const int st = i % kTinyStages;
        tiny_mbar_wait(&empty[st], ((i / kTinyStages) & 1) ^ 1);
        int ka, kb, key;
        map_unit(w, map, p, ka, kb, key);
        if (skip_unit(only_if, key)) {  // nothing to load: complete the phase empty
          tiny_mbar_expect_tx(&full[st], 0);
          continue;
        }
        tiny_mbar_expect_tx(&full[st], 4 * abytes + 4 * bbytes);
        double2* d = smem + (size_t)st * kTinyItem;
        // A1_k, A2_k, A1_s, A2_s | B1_k, B2_k, B1_s, B2_s  (qt_dmma_tile.cuh PairArgs order)
        tiny_bulk_load(d + 0 * kTinySlice, ah1 + ka * amn, abytes, &full[st]);
        tiny_bulk_load(d + 1 * kTinySlice, ah2 + ka * amn, abytes, &full[st]);
        tiny_bulk_load(d + 2 * kTinySlice, ah1 + kb * amn, abytes, &full[st]);
        tiny_bulk_load(d + 3 * kTinySlice, ah2 + kb * amn, abytes, &full[st]);
        tiny_bulk_load(d + 4 * kTinySlice, bh1 + ka * bns, bbytes, &full[st]);
        tiny_bulk_load(d + 5 * kTinySlice, bh2 + ka * bns, bbytes, &full[st]);
        tiny_bulk_load(d + 6 * kTinySlice, bh1 + kb * bns, bbytes, &full[st]);
        tiny_bulk_load(d + 7 * kTinySlice, bh2 + kb * bns, bbytes, &full[st]);
      }
    }
    return;
  }
  // ---- consumers: group gr takes the CTA's items gr, gr + 2, ...
  const int gr = warp >> 2, wq = warp & 3;
  const int wm = wq & 1, wn = wq >> 1;  // the warp's 8 x 8 block of the 16 x 16 tile
  const int g = lane >> 2, q = lane & 3;
  const int i_row = wm * 8 + g, j_col = wn * 8 + g;
  for (int i = gr;; i += kTinyGroups) {
    const int w = blockIdx.x + i * G;
    if (w >= units) break;
    const int st = i % kTinyStages;
    tiny_mbar_wait(&full[st], (i / kTinyStages) & 1);
    int ka, kb, key;
    map_unit(w, map, p, ka, kb, key);
    if (!skip_unit(only_if, key)) {
      const double2* sa = smem + (size_t)st * kTinyItem;
      const double2* sb = sa + 4 * kTinySlice;
      double T[12][2];
#pragma unroll
      for (int c = 0; c < 12; ++c) T[c][0] = T[c][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {  // K tile of 16 (SmallGaussCfg::BK), zero-padded beyond n
        const int k = ks * 4 + q;
        double br[4], bi[4], bp[4];
        const bool bok = k < n && j_col < s;
#pragma unroll
        for (int pl = 0; pl < 4; ++pl) {
          const double2 v = bok ? sb[pl * kTinySlice + k * s + j_col] : make_double2(0.0, 0.0);
          br[pl] = v.x;
          bi[pl] = v.y;
          bp[pl] = v.x + v.y;
        }
        const double nb2k_r = dneg(br[1]), nb2k_i = dneg(bi[1]), nb2k_p = dneg(bp[1]);
        const bool aok = k < n && i_row < m;
        double ar[4], ai[4], ap[4], am[4];
#pragma unroll
        for (int pl = 0; pl < 4; ++pl) {
          const double2 v = aok ? sa[pl * kTinySlice + i_row * n + k] : make_double2(0.0, 0.0);
          ar[pl] = v.x;
          ai[pl] = v.y;
          ap[pl] = v.x + v.y;
          am[pl] = v.x - v.y;
        }
        // mma_stage_3m's sequence (non-SELF; a self-paired unit has sigma k = k)
        dmma(T[0], ar[0], br[0]);
        dmma(T[1], ai[0], bi[0]);
        dmma(T[2], ap[0], bp[0]);
        dmma(T[3], ar[2], br[1]);
        dmma(T[4], ai[2], nb2k_i);
        dmma(T[5], am[2], bp[1]);
        dmma(T[6], ar[2], br[2]);
        dmma(T[7], ai[2], bi[2]);
        dmma(T[8], ap[2], bp[2]);
        dmma(T[9], ar[0], br[3]);
        dmma(T[10], ai[0], dneg(bi[3]));
        dmma(T[11], am[0], bp[3]);
        dmma(T[0], ar[3], nb2k_r);
        dmma(T[1], ai[3], bi[1]);
        dmma(T[2], am[3], nb2k_p);
        dmma(T[3], ar[1], br[0]);
        dmma(T[4], ai[1], bi[0]);
        dmma(T[5], ap[1], bp[0]);
        dmma(T[6], ar[1], dneg(br[3]));
        dmma(T[7], ai[1], bi[3]);
        dmma(T[8], am[1], dneg(bp[3]));
        dmma(T[9], ar[3], br[2]);
        dmma(T[10], ai[3], bi[2]);
        dmma(T[11], ap[3], bp[2]);
      }
      // operands consumed: hand the stage back before the (global) stores
      __syncwarp();
      if (lane == 0) tiny_mbar_arrive(&empty[st]);
      double2* cp[4] = {ch1 + ka * cms, ch2 + ka * cms, ch1 + kb * cms, ch2 + kb * cms};
      const int row = i_row, col = wn * 8 + 2 * q;
      if (row < m) {
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          double2* dst = cp[o] + (size_t)row * s + col;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double t1 = T[3 * o][e], t2 = T[3 * o + 1][e], t3 = T[3 * o + 2][e];
            if (col + e < s) dst[e] = make_double2(t1 - t2, t3 - t1 - t2);
          }
        }
      }
    } else {
      __syncwarp();
      if (lane == 0) tiny_mbar_arrive(&empty[st]);
    }
  }
}

bool tiny_enabled() {
  static const bool on = [] {
    const char* e = getenv("QTB_TINY");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t launch_tiny_ws(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                           double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                           cudaStream_t stream, const int* only_if, PairMap map) {
  static std::mutex mu;
  static uint64_t done = 0;
  static int sms = 148;
  const cudaError_t attr_err = once_per_device(mu, done, [&] {
    cudaError_t e = cudaFuncSetAttribute(paired_tiny_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kTinySmem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return e;
  });
  if (attr_err != cudaSuccess) return attr_err;
  const uint64_t units = map.noreflect ? p : map.s0 < 0 ? p / 2 + 1 : (uint64_t)slot_units(map.s0, map.ns, (int)p);
  if (units == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<uint64_t>(units, (uint64_t)sms);
  ProfScope ps(only_if ? "k2_dmma_guard" : "k2_dmma", stream);
  paired_tiny_ws_kernel<<<grid, kTinyThreads, kTinySmem, stream>>>(ah1, ah2, bh1, bh2, ch1, ch2, (int)m, (int)n,
                                                                   (int)s, (int)p, only_if, map, (int)units);
  ps.stop();
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

// the complex-product algorithm every DMMA tile uses (the one-launch small
// product, qt_small.cu, must evaluate the same one)
bool dmma_gauss() { return gauss_enabled(); }

// DMMA (fp64 tensor-core) paired product; with an int8 flag array in only_if
// a CTA runs only for the pairs the int8 path did not certify (qt_ozaki.cu).
static cudaError_t dmma_impl(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                             double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                             uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice, cudaStream_t stream,
                             const int* only_if, PairMap map) {
  // Small slices (m, s <= 32): the 64-row tile would waste >= half its DMMAs
  // and its two-deep K pipeline would be all latency; use the 16 x 16 tile.
  const bool gauss = gauss_enabled();
  if (m <= 32 && s <= 32) {
    // whole-slice tiles with contiguous slices: the warp-specialised ring
    if (gauss && tiny_enabled() && m <= 16 && s <= 16 && n <= 16 && ldb == s && ldc == s && bslice == n * s &&
        cslice == m * s)
      return launch_tiny_ws(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, stream, only_if, map);
    if (n <= (uint64_t)SmallCfg::BK)
      return gauss ? launch_small_persistent<SmallGaussCfg>(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc,
                                                            bslice, cslice, stream, only_if, map)
                   : launch_small_persistent<SmallCfg>(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice,
                                                       cslice, stream, only_if, map);
    return gauss ? launch_cfg<SmallGaussCfg>(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice,
                                             stream, only_if, map)
                 : launch_cfg<SmallCfg>(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream,
                                        only_if, map);
  }
  if (gauss)
    return launch_cfg<GaussCfg>(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream, only_if,
                                map);
  return launch_cfg<BigCfg>(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream, only_if, map);
}

bool debug_noreflect() {
  static const bool on = [] {
    const char* e = getenv("QTB_DEBUG_NO_REFLECT");
    return e && e[0] == '1';
  }();
  return on;
}

cudaError_t dmma_spectral_gemm(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                               double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                               uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice, cudaStream_t stream,
                               const int* only_if) {
  PairMap map;
  map.noreflect = (only_if == nullptr && debug_noreflect()) ? 1 : 0;
  return dmma_impl(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream, only_if, map);
}

cudaError_t dmma_spectral_gemm_slots(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                     double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                     int s0, int ns, cudaStream_t stream, const int* only_if) {
  PairMap map;
  map.s0 = s0;
  map.ns = ns;
  return dmma_impl(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, s, s, n * s, m * s, stream, only_if, map);
}

cudaError_t launch_spectral_gemm_ld(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                    double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                    uint64_t ldb, uint64_t ldc, uint64_t bslice, uint64_t cslice, cudaStream_t stream,
                                    int algo) {
  if (m == 0 || s == 0 || p == 0) return cudaSuccess;
  if (algo == kAlgoAuto) algo = choose_gemm_algo(n, s, p);
  if (algo == kAlgoOzaki && (n % 32 != 0 || n > 8192 || p > 65534)) return cudaErrorInvalidValue;
  if (algo != kAlgoOzaki)
    return dmma_spectral_gemm(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream, nullptr);
  // exact int8 tensor-core path (qt_ozaki.cu); the DMMA kernels run only if
  // the inputs held a non-finite value
  int* flag = nullptr;
  const size_t fb = int8_flag_ints(p) * sizeof(int);
  cudaError_t e = cudaMallocAsync(&flag, fb, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(flag, 0, fb, stream);
  if (e == cudaSuccess)
    e = launch_spectral_gemm_ozaki(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, flag, stream);
  if (e == cudaErrorMemoryAllocation) {
    // not enough free HBM for the residue workspace: the fp64 kernels
    // recompute the whole product unconditionally (always correct)
    cudaGetLastError();
    e = cudaMemsetAsync(flag, 0xff, sizeof(int), stream);
  }
  if (e == cudaSuccess)
    e = dmma_spectral_gemm(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, ldb, ldc, bslice, cslice, stream, flag);
  const cudaError_t fe = cudaFreeAsync(flag, stream);
  return e != cudaSuccess ? e : fe;
}

cudaError_t launch_spectral_gemm(const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                                 double2* ch1, double2* ch2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                                 cudaStream_t stream, int algo) {
  return launch_spectral_gemm_ld(ah1, ah2, bh1, bh2, ch1, ch2, m, n, s, p, s, s, n * s, m * s, stream, algo);
}

}  // namespace qtb
