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

#include "qt_internal.cuh"

namespace qtb {

namespace {

// Tile configuration.  Warps are laid out WM x WN; a warp owns RB 8-row blocks
// x one 8-column block of the tile, for all 8 (or 4, SELF) real components.
template <int BM_, int BN_, int BK_, int WM_, int WN_, int RB_, int STAGES_, int MINB_>
struct TileCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, RB = RB_, STAGES = STAGES_;
  static constexpr int MINB = MINB_;
  static constexpr int NTHREADS = 32 * WM * WN;
  // smem tile geometry (double2 units); XOR swizzles make every fragment load
  // a conflict-free LDS.128 without padding:
  //   A plane: [BM][BK], element (i, c) at i*BK + (c ^ ((i & 1) << 2))
  //   B plane: [BK][BN], element (k, j) at k*BN + (j ^ ((k & 3) << 1))
  static constexpr int A_PLANE = BM * BK;
  static constexpr int B_PLANE = BK * BN;
  static constexpr int STAGE_ELEMS = 4 * A_PLANE + 4 * B_PLANE;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_ELEMS * 16;
  static_assert(BM == WM * RB * 8 && BN == WN * 8, "warp layout must tile the CTA tile");
  static_assert(BK % 8 == 0 && BN % 8 == 0, "swizzles need BK, BN multiples of 8");
};
using BigCfg = TileCfg<64, 16, 8, 4, 2, 2, 2, 2>;     // 256 threads, 80 KB smem
using SmallCfg = TileCfg<16, 16, 16, 2, 2, 1, 2, 4>;  // 128 threads, 64 KB smem

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;  // zero-fill out-of-range chunks
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double dneg(double x) {
  // sign flip on the integer pipe (keeps the FP64 pipe for DMMA only)
  long long b = __double_as_longlong(x) ^ (long long)0x8000000000000000ULL;
  return __longlong_as_double(b);
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

struct PairArgs {
  const double2* a[4];  // Â1_k, Â2_k, Â1_σ, Â2_σ   (m x n each)
  const double2* b[4];  // B̂1_k, B̂2_k, B̂1_σ, B̂2_σ   (n x s each)
  double2* c[4];        // Ĉ1_k, Ĉ2_k, Ĉ1_σ, Ĉ2_σ   (m x s each)
};

template <class C, bool SELF>
__device__ __forceinline__ void load_stage(double2* st, const PairArgs& P, int kt, int row0, int col0, int m, int n,
                                           int s, int ldb) {
  constexpr int NP = SELF ? 2 : 4;
  const int tid = threadIdx.x;
  const int k0 = kt * C::BK;
  // plane index is static in every loop (no local-memory pointer indexing)
#pragma unroll
  for (int pl = 0; pl < NP; ++pl) {
#pragma unroll
    for (int id = tid; id < C::A_PLANE; id += C::NTHREADS) {
      const int c = id % C::BK;
      const int i = id / C::BK;
      const int gr = row0 + i, gc = k0 + c;
      const bool ok = gr < m && gc < n;
      const double2* src = P.a[pl] + (ok ? (size_t)gr * n + gc : 0);
      double2* dst = st + pl * C::A_PLANE + i * C::BK + (c ^ ((i & 1) << 2));
      cp_async16(smem_u32(dst), src, ok);
    }
  }
  double2* sb = st + 4 * C::A_PLANE;
#pragma unroll
  for (int pl = 0; pl < NP; ++pl) {
#pragma unroll
    for (int id = tid; id < C::B_PLANE; id += C::NTHREADS) {
      const int j = id % C::BN;
      const int k = id / C::BN;
      const int gk = k0 + k, gj = col0 + j;
      const bool ok = gk < n && gj < s;
      const double2* src = P.b[pl] + (ok ? (size_t)gk * ldb + gj : 0);
      double2* dst = sb + pl * C::B_PLANE + k * C::BN + (j ^ ((k & 3) << 1));
      cp_async16(smem_u32(dst), src, ok);
    }
  }
}

// One staged K-slice (BK complex columns of Â, BK rows of B̂) through the DMMAs.
template <class C, bool SELF>
__device__ __forceinline__ void mma_stage(const double2* sa, const double2* sb, double (&acc)[SELF ? 4 : 8][C::RB][2],
                                          int wm, int wn, int g, int q) {
  constexpr int NC = SELF ? 4 : 8;
  constexpr int RB = C::RB;
#pragma unroll
  for (int ks = 0; ks < C::BK / 4; ++ks) {
    // B fragments: element (k = ks*4 + q, j = wn*8 + g); swizzle j ^ (q << 1)
    const int kb = ks * 4 + q;
    const int jb = (wn * 8 + g) ^ (q << 1);
    double br[4], bi[4];
#pragma unroll
    for (int pl = 0; pl < (SELF ? 2 : 4); ++pl) {
      const double2 v = sb[pl * C::B_PLANE + kb * C::BN + jb];
      br[pl] = v.x;
      bi[pl] = v.y;
    }
    const double nb1k_i = dneg(bi[0]);
    const double nb2k_r = dneg(br[1]);
    const double nb2k_i = dneg(bi[1]);
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
      const int i = wm * (RB * 8) + rb * 8 + g;
      const int ca = (ks * 4 + q) ^ ((i & 1) << 2);
      double ar[4], ai[4];
#pragma unroll
      for (int pl = 0; pl < (SELF ? 2 : 4); ++pl) {
        const double2 v = sa[pl * C::A_PLANE + i * C::BK + ca];
        ar[pl] = v.x;
        ai[pl] = v.y;
      }
      if (SELF) {  // A1s = A1k, A2s = A2k
        ar[2] = ar[0]; ai[2] = ai[0]; ar[3] = ar[1]; ai[3] = ai[1];
      }
      // C1_k = A1k B1k - conj(A2s) B2k
      dmma(acc[0][rb], ar[0], br[0]);
      dmma(acc[0][rb], ai[0], nb1k_i);
      dmma(acc[0][rb], ar[3], nb2k_r);
      dmma(acc[0][rb], ai[3], nb2k_i);
      dmma(acc[1][rb], ar[0], bi[0]);
      dmma(acc[1][rb], ai[0], br[0]);
      dmma(acc[1][rb], ar[3], nb2k_i);
      dmma(acc[1][rb], ai[3], br[1]);
      // C2_k = conj(A1s) B2k + A2k B1k
      dmma(acc[2][rb], ar[2], br[1]);
      dmma(acc[2][rb], ai[2], bi[1]);
      dmma(acc[2][rb], ar[1], br[0]);
      dmma(acc[2][rb], ai[1], nb1k_i);
      dmma(acc[3][rb], ar[2], bi[1]);
      dmma(acc[3][rb], ai[2], nb2k_r);
      dmma(acc[3][rb], ar[1], bi[0]);
      dmma(acc[3][rb], ai[1], br[0]);
      if (!SELF) {
        const double nb1s_i = dneg(bi[2]);
        const double nb2s_r = dneg(br[3]);
        const double nb2s_i = dneg(bi[3]);
        // C1_σ = A1s B1s - conj(A2k) B2s
        dmma(acc[4 % NC][rb], ar[2], br[2]);
        dmma(acc[4 % NC][rb], ai[2], nb1s_i);
        dmma(acc[4 % NC][rb], ar[1], nb2s_r);
        dmma(acc[4 % NC][rb], ai[1], nb2s_i);
        dmma(acc[5 % NC][rb], ar[2], bi[2]);
        dmma(acc[5 % NC][rb], ai[2], br[2]);
        dmma(acc[5 % NC][rb], ar[1], nb2s_i);
        dmma(acc[5 % NC][rb], ai[1], br[3]);
        // C2_σ = conj(A1k) B2s + A2s B1s
        dmma(acc[6 % NC][rb], ar[0], br[3]);
        dmma(acc[6 % NC][rb], ai[0], bi[3]);
        dmma(acc[6 % NC][rb], ar[3], br[2]);
        dmma(acc[6 % NC][rb], ai[3], nb1s_i);
        dmma(acc[7 % NC][rb], ar[0], bi[3]);
        dmma(acc[7 % NC][rb], ai[0], nb2s_r);
        dmma(acc[7 % NC][rb], ar[3], bi[2]);
        dmma(acc[7 % NC][rb], ai[3], br[2]);
      }
    }
  }
}

// epilogue: (re, im) pairs of C[row][col], col = 2q, 2q+1 of the 8-wide block
template <class C, bool SELF>
__device__ __forceinline__ void store_tile(const PairArgs& P, const double (&acc)[SELF ? 4 : 8][C::RB][2], int row0,
                                           int col0, int m, int s, int ldc, int wm, int wn, int g, int q) {
  constexpr int NC = SELF ? 4 : 8;
  const int col = col0 + wn * 8 + 2 * q;
#pragma unroll
  for (int f = 0; f < (SELF ? 1 : 2); ++f) {
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      double2* Cp = P.c[f * 2 + part];
      const int cr = f * 4 + part * 2;
#pragma unroll
      for (int rb = 0; rb < C::RB; ++rb) {
        const int row = row0 + wm * (C::RB * 8) + rb * 8 + g;
        if (row < m) {
          double2* dst = Cp + (size_t)row * ldc + col;
          if (col < s) dst[0] = make_double2(acc[cr % NC][rb][0], acc[(cr + 1) % NC][rb][0]);
          if (col + 1 < s) dst[1] = make_double2(acc[cr % NC][rb][1], acc[(cr + 1) % NC][rb][1]);
        }
      }
    }
  }
}

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
