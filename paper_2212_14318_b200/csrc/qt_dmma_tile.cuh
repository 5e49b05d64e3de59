// qt_dmma_tile.cuh — shared FP64-DMMA tile machinery of the spectral GEMM
// (qt_gemm.cu) and the definitional product (qt_naive.cu): tile shapes,
// cp.async staging with XOR-swizzled conflict-free shared-memory layouts, the
// m8n8k4.f64 fragment loop of the paired-frequency product and the epilogue.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace qtb {
namespace {

// Tile configuration.  Warps are laid out WM x WN; a warp owns RB 8-row blocks
// x one 8-column block of the tile, for all 8 (or 4, SELF) real components.
template <int BM_, int BN_, int BK_, int WM_, int WN_, int RB_, int STAGES_, int MINB_, int GAUSS_ = 0>
struct TileCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, RB = RB_, STAGES = STAGES_;
  static constexpr int MINB = MINB_;
  static constexpr bool GAUSS = GAUSS_ != 0;  // 3-multiplication complex products (qt_gemm.cu)
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
// Gauss 3M variant: 12 accumulator sets per 8x8 block need ~170 registers, so
// 4 warps (32 x 16 tile) and 3 CTAs per SM; 3-deep cp.async ring (72 KB)
using GaussCfg = TileCfg<32, 16, 8, 2, 2, 2, 3, 3, 1>;
using SmallGaussCfg = TileCfg<16, 16, 16, 2, 2, 1, 2, 4, 1>;
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
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
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

}  // namespace
}  // namespace qtb
