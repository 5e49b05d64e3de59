// qt_ozaki.cu — K2 on the int8 tensor cores: exact modular (Ozaki-II / CRT)
// evaluation of the paired-frequency product (sm_100a, tcgen05 + TMA + TMEM).
//
// What is computed is the same stage 2 as qt_gemm.cu (tproduct.cpp:89-106):
//     [C1_k; C2_k] = X_k Y_k,  X_k = [[A1_k, -conj A2_sk], [A2_k, conj A1_sk]],  Y_k = [B1_k; B2_k]
// (sk = (p - k) mod p, SURVEY §8(a) paired form).  In real form
//     [Re C | Im C] = [Re X | Im X] . [[Re Y, Im Y], [-Im Y, Re Y]]      (2m x 4n) . (4n x 2s)
// FP64 has no tcgen05 path on B200 (DMMA peaks at 37 TF/s), so the product is
// evaluated EXACTLY in integers and rounded once:
//   1. scale: every row of X_k and every column of Y_k gets a power of two so
//      that its largest |re|, |im| stays below 2^53 and its Euclidean norm below
//      2^T (T = 58), and is rounded to integers X', Y' (the only approximation:
//      <= 2^-53 of the row/column maximum, i.e. fp64 input precision, whenever
//      the norm bound is not the tighter one — max/rms > sqrt(4n)/32 — and at
//      most ~1 bit less otherwise);
//   2. residues: X' and Y' mod each of Q = 15 pairwise-coprime moduli <= 256, as
//      uint8 in [0, p) (K2r kernels, K-major, ready for TMA);
//   3. int8 GEMMs: for each modulus, X'_q Y'_q on tcgen05.mma.kind::i8 (u8 x u8)
//      with an int32 TMEM accumulator (exact: sum < 255^2 * 4n < 2^31 for
//      n <= 8192), reduced mod p_q in the epilogue and stored as one byte per
//      real output (K2g kernel);
//   4. CRT: the 15 residues give X'Y' exactly (Cauchy-Schwarz: |x'.y'| <=
//      ||x'|| ||y'|| < 2^116 < M/2 = 2^116.6),
//      reconstructed as a 96-bit fixed-point fraction X'Y'/M, converted to
//      double once and scaled back by 2^-(eX + eY) (K2c kernel).
// The integer product is exact, so the result does not depend on tiling,
// K order, row shards or column chunks — bitwise — and its error is the fp64
// rounding of the scaled inputs plus one final rounding: measured below the
// DMMA path's error against the definitional product.
//
// Non-finite inputs cannot be represented in integers: K2r raises a device
// flag, K2c then leaves C alone and the DMMA kernel (qt_gemm.cu) recomputes
// the product on the GPU (its launch is conditional on the flag).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "qt_internal.cuh"

namespace qtb {
namespace oz {

constexpr int kQ = 15;
constexpr int kBits = 53;
// pairwise coprime, <= 256; product M = 2^117.6
constexpr int kModuli[kQ] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197};

struct ModTable {
  uint32_t p[kQ];
  uint32_t magic[kQ];  // floor(2^32 / p): quotient estimate off by at most one
  uint32_t magic37[kQ];  // ceil(2^37 / p): exact quotient umulhi(v, .) >> 5 for v < 2^28
  uint32_t negp[kQ];     // -p mod 2^32 (r = v + q (-p): one IMAD, no negation)
  uint32_t wlo[kQ];    // bytes 256^b mod p, b = 0..3 (dp4a weights of the low word)
  uint32_t whi[kQ];    // bytes 256^b mod p, b = 4..6 (and 0 for b = 7)
  uint32_t cofs[kQ];   // p - (2^55 mod p): removes the 2^55 offset, keeps the sum non-negative
  uint32_t w[kQ][3];   // round(2^96 * y_q / p_q) mod 2^96, y_q = (M/p_q)^-1 mod p_q (CRT weights)
  double M;            // prod p_q (rounded)
  int ebound;          // T = floor((log2 M - 1) / 2) - margin: ||x'||, ||y'|| < 2^T keeps |x'.y'| < M/2
};
__constant__ ModTable c_mod;

// ------------------------------------------------------------------ tiles
constexpr int BM = 128;        // output rows per CTA (TMEM lanes)
constexpr int BNC = 128;       // complex output columns per CTA (Re + Im = 256 TMEM columns)
constexpr int BN = 2 * BNC;    // real B' rows per tile
constexpr int BK = 128;        // K bytes per stage (one 128-byte swizzle row)
constexpr int STAGES = 4;
constexpr int A_STAGE = BM * BK;  // 16 KB
constexpr int B_STAGE = BN * BK;  // 32 KB
constexpr int GEMM_THREADS = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr size_t GEMM_SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) + 1024;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T, int8 x int8 -> int32
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// K-major operand, 128-byte swizzle: 8-row groups 1024 B apart (SBO), version 1
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: s32 accumulator, u8 x u8, K-major A and B, M = 128, N = 256
constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// v mod p for any 32-bit v: the magic quotient is exact or one short
__device__ __forceinline__ uint32_t mod_u32(uint32_t v, uint32_t p, uint32_t magic) {
  const uint32_t r = v - __umulhi(v, magic) * p;
  return r >= p ? r - p : r;
}

// --------------------------------------------------------------- K2g GEMM
struct GemmParams {
  uint8_t* R;        // residues out: [Q][F * Mp][Sp] x (re, im) bytes
  int Q, mt, Mp, Sp, KB, F;
  int bslot0;        // slot of this batch's first frequency in the B' buffer
  int nt, fcur;      // n tiles, slots in this batch (persistent pair kernel)
  int aslot0;        // slot of this batch's first frequency in the X' buffer
  int slot0;         // absolute frequency slot of the batch's first slot
  int share_end;     // slots below this share X': an odd one reads its even partner's (0: off)
};

// The odd slot 2j+1 (frequency sk) of a pair reuses the X' of its partner 2j
// (frequency k): X_sk's rows are X_k's with the row halves swapped, the K
// quarters permuted and some signs flipped (X_sk top = M(X_k bottom), X_sk
// bottom = -M(X_k top), M[q0 q1 q2 q3] = [q1 -q0 -q3 q2]), so
//   X_sk . Y_sk = [X_k bottom . Y''; -(X_k top . Y'')],  Y'' = M*(Y_sk),
// M*[q0 q1 q2 q3] = [-q1 q0 q3 -q2] applied to every Y row.  The residue
// kernels then write each X' row once instead of twice, the odd slot's B'
// holds Y'' instead of Y, and its CRT reads the R rows in swapped order with
// the top half negated — every integer is the same, so results are bitwise
// the same as with a separate X_sk.
__device__ __forceinline__ bool shares_x(int slot, int share_end) { return slot < share_end && (slot & 1); }

// (slot, modulus) of the persistent GEMM's fq-th (slot, modulus) plane.  With
// shared X' the two slots of a pair take turns per modulus, (2j, q), (2j+1, q),
// (2j, q+1), ..., so the X' plane both read is still in L2 for the second;
// otherwise slot-major.  (Batches start at an even slot: pairs stay together.)
__device__ __forceinline__ void item_slot_mod(int fq, const GemmParams& P, int& f, int& q) {
  const int fe = P.share_end > P.slot0 ? min(P.fcur, P.share_end - P.slot0) & ~1 : 0;  // shared slots of the batch
  if (fq < fe * P.Q) {
    const int pr = fq / (2 * P.Q), rem = fq - pr * 2 * P.Q;
    q = rem >> 1;
    f = 2 * pr + (rem & 1);
  } else {
    const int r = fq - fe * P.Q;
    f = fe + r / P.Q;
    q = r % P.Q;
  }
}

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   GemmParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mtile = blockIdx.x % P.mt, ntile = blockIdx.x / P.mt, f = blockIdx.y;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      const int af = f - (shares_x(P.slot0 + f, P.share_end) ? 1 : 0);
      const int arow = (P.aslot0 + af) * P.Mp + mtile * BM, brow = (P.bslot0 + f) * 2 * P.Sp + ntile * BN;
      uint32_t it = 0;
      for (int q = 0; q < P.Q; ++q)
        for (int kb = 0; kb < P.KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], A_STAGE + B_STAGE);
          tma_load_3d(sA + s * A_STAGE, &mapA, &full[s], kb * BK, arow, q);
          tma_load_3d(sB + s * B_STAGE, &mapB, &full[s], kb * BK, brow, q);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      uint32_t it = 0;
      for (int q = 0; q < P.Q; ++q) {
        const int b = q & 1;
        mbar_wait(&tempty[b], ((q >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + b * BN;
        for (int kb = 0; kb < P.KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * A_STAGE), b0 = smem_u32(sB + s * B_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            mma_i8(d, smem_desc_sw128(a0 + kk * 32), smem_desc_sw128(b0 + kk * 32), kIdesc, (kb | kk) != 0);
          tc_commit(&empty[s]);  // smem stage free once these MMAs have read it
        }
        tc_commit(&tfull[b]);  // accumulator b complete
      }
    }
  } else {  // ---- epilogue: TMEM -> mod p -> bytes
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const size_t plane = (size_t)P.F * P.Mp * P.Sp * 2;
    uint8_t* out0 = P.R + ((size_t)(f * P.Mp + mtile * BM + row) * P.Sp + (size_t)ntile * BNC) * 2;
    for (int q = 0; q < P.Q; ++q) {
      const int b = q & 1;
      mbar_wait(&tfull[b], (q >> 1) & 1);
      tc_fence_after();
      const uint32_t pq = c_mod.p[q], mg = c_mod.magic[q];
      uint8_t* out = out0 + (size_t)q * plane;
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + b * BN;
#pragma unroll 1
      for (int c = 0; c < BNC / 32; ++c) {
        uint32_t re[32], im[32];
        tmem_ld32(tbase + c * 32, re);
        tmem_ld32(tbase + BNC + c * 32, im);
        tmem_wait_ld();
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t r0 = mod_u32(re[2 * j], pq, mg), i0 = mod_u32(im[2 * j], pq, mg);
          const uint32_t r1 = mod_u32(re[2 * j + 1], pq, mg), i1 = mod_u32(im[2 * j + 1], pq, mg);
          w[j] = r0 | (i0 << 8) | (r1 << 16) | (i1 << 24);
        }
        uint4* o = reinterpret_cast<uint4*>(out + c * 64);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ----------------------------------------------- K2g GEMM, CTA pair (2SM)
// The same product on tcgen05.mma.cta_group::2: a cluster of two CTAs on a
// TPC computes a 256 x 256 tile (M = 256 rows of X', N = 128 complex output
// columns).  Each CTA stages its own 128 rows of A and HALF of the 256 B' rows,
// so per SM the L2->SMEM operand traffic per MMA drops from 12 KB to 8 KB; the
// even CTA issues the MMAs (its descriptors address the same offsets in the
// odd CTA's shared memory) into both CTAs' TMEM.  Barriers: TMA bytes of both
// CTAs land on the even CTA's full[s]; MMA commits multicast to both CTAs'
// empty[s] / tfull[b]; both epilogues arrive on the even CTA's tempty[b].
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the even CTA's copy
constexpr int B2_STAGE = (BN / 2) * BK;  // 16 KB: this CTA's half of the B' tile
constexpr size_t gemm2_smem(int stages) { return (size_t)stages * (A_STAGE + B2_STAGE) + 1024; }
constexpr uint32_t kIdesc2 = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ void tma_load_3d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_commit_2sm(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mma_i8_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int STAGES2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    oz_gemm2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    GemmParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * A_STAGE;
  __shared__ __align__(8) uint64_t full[STAGES2], empty[STAGES2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  // persistent: cluster c takes work items c, c + nclusters, ... in the order
  // (slot, modulus, n tile, m tile), so the clusters in flight share one
  // (slot, modulus) plane of X' and Y' (~67 MB at config 5): each operand
  // byte comes from DRAM about once instead of once per wave
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int mt2 = P.mt / 2;  // 256-row tiles
  const int tiles = mt2 * P.nt;
  const int nitems = P.fcur * P.Q * tiles;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote use
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs)
      uint32_t it = 0;
      for (int item = cl; item < nitems; item += ncl) {
        const int t = item % tiles;
        int f, q;
        item_slot_mod(item / tiles, P, f, q);
        const int mtile2 = t % mt2, ntile = t / mt2;
        const int af = f - (shares_x(P.slot0 + f, P.share_end) ? 1 : 0);
        const int arow = (P.aslot0 + af) * P.Mp + mtile2 * 256 + rank * BM;
        const int brow = (P.bslot0 + f) * 2 * P.Sp + ntile * BN + rank * (BN / 2);
        for (int kb = 0; kb < P.KB; ++kb, ++it) {
          const int s = it % STAGES2;
          mbar_wait(&empty[s], ((it / STAGES2) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * (A_STAGE + B2_STAGE));
          tma_load_3d_2sm(sA + s * A_STAGE, &mapA, &full[s], kb * BK, arow, q);
          tma_load_3d_2sm(sB + s * B2_STAGE, &mapB, &full[s], kb * BK, brow, q);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {  // ---- MMA issuer (even CTA)
      uint32_t it = 0;
      for (int item = cl, li = 0; item < nitems; item += ncl, ++li) {
        const int b = li & 1;
        mbar_wait(&tempty[b], ((li >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + b * BN;
        for (int kb = 0; kb < P.KB; ++kb, ++it) {
          const int s = it % STAGES2;
          mbar_wait(&full[s], (it / STAGES2) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * A_STAGE), b0 = smem_u32(sB + s * B2_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            mma_i8_2sm(d, smem_desc_sw128(a0 + kk * 32), smem_desc_sw128(b0 + kk * 32), kIdesc2, (kb | kk) != 0);
          tc_commit_2sm(&empty[s]);
        }
        tc_commit_2sm(&tfull[b]);
      }
    }
  } else {  // ---- epilogue (both CTAs, own TMEM rows)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const size_t plane = (size_t)P.F * P.Mp * P.Sp * 2;
    for (int item = cl, li = 0; item < nitems; item += ncl, ++li) {
      const int t = item % tiles;
      int f, q;
      item_slot_mod(item / tiles, P, f, q);
      const int mtile2 = t % mt2, ntile = t / mt2;
      const int b = li & 1;
      mbar_wait(&tfull[b], (li >> 1) & 1);
      tc_fence_after();
      const uint32_t pq = c_mod.p[q], mg = c_mod.magic[q];
      uint8_t* out = P.R + (size_t)q * plane +
                     ((size_t)(f * P.Mp + mtile2 * 256 + rank * BM + row) * P.Sp + (size_t)ntile * BNC) * 2;
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + b * BN;
#pragma unroll 1
      for (int c = 0; c < BNC / 32; ++c) {
        uint32_t re[32], im[32];
        tmem_ld32(tbase + c * 32, re);
        tmem_ld32(tbase + BNC + c * 32, im);
        tmem_wait_ld();
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t r0 = mod_u32(re[2 * j], pq, mg), i0 = mod_u32(im[2 * j], pq, mg);
          const uint32_t r1 = mod_u32(re[2 * j + 1], pq, mg), i1 = mod_u32(im[2 * j + 1], pq, mg);
          w[j] = r0 | (i0 << 8) | (r1 << 16) | (i1 << 24);
        }
        uint4* o = reinterpret_cast<uint4*>(out + c * 64);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(&tempty[b]) & kPeerMask)
                     : "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------- K2r residues
// Frequencies are processed in slots: slot 2j, 2j+1 hold the pair (j+1,
// p-j-1); the self-paired 0 and p/2 come last.  A batch is a run of slots with
// an even start, so a pair never straddles two batches.
__device__ __forceinline__ int slot_freq(int slot, int p) { return slot_frequency(slot, p); }

// Slice of a frequency slot in the operand tensors: the frequency itself, or
// (compact tensors holding slots [cbase, ...) in slot order) slot - cbase.
__device__ __forceinline__ int slot_slice(int slot, int p, int cbase) {
  return cbase < 0 ? slot_freq(slot, p) : slot - cbase;
}

// x * 2^e, exact for the finite values scaled here (one multiply in range)
__device__ __forceinline__ double scale2(double x, int e) {
  if (e >= -1022 && e <= 1023) return x * __longlong_as_double((long long)(e + 1023) << 52);
  return ldexp(x, e);
}

// An integer-valued double |x| <= 2^53, offset by 2^55 to a non-negative
// integer < 2^56: its seven bytes, as the low and high 32-bit words
struct Limbs {
  uint32_t lo, hi;
};
__device__ __forceinline__ Limbs to_limbs(double x, int e) {
  const long long v = __double2ll_rn(scale2(x, e)) + (1ll << 55);
  return Limbs{(uint32_t)v, (uint32_t)(v >> 32)};
}
// x mod p_q in [0, p_q); q is a compile-time index after unrolling, so the
// table entries are constant-bank operands.  x + 2^55 = sum_b byte_b 256^b, so
// x = sum_b byte_b (256^b mod p) - 2^55 (mod p): two byte dot products (dp4a)
// plus the offset correction give s < 7 * 255^2 + 256 < 2^19, reduced exactly
// by the 37-bit reciprocal (valid below 2^28).
__device__ __forceinline__ uint32_t res_of(const Limbs& l, int q) {
  if (q == 0) return l.lo & 0xffu;  // p_0 = 256 divides 2^55: the low byte
  const uint32_t v = __dp4a(l.lo, c_mod.wlo[q], __dp4a(l.hi, c_mod.whi[q], c_mod.cofs[q]));
  return v + (__umulhi(v, c_mod.magic37[q]) >> 5) * c_mod.negp[q];
}
// four bytes (each < 256) into one little-endian word (3 PRMT)
__device__ __forceinline__ uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}
__device__ __forceinline__ uint32_t neg_res(uint32_t r, uint32_t p) { return r ? p - r : 0u; }
// -r mod p for an MMA operand byte: p - r in [1, p] (p itself stands for 0: the
// GEMM only needs the value mod p, and 255^2 * 4n still bounds its sums), and
// for p = 256 the packed low byte of 256 - r is -r mod 256.  One operation.
__device__ __forceinline__ uint32_t neg_op(uint32_t r, uint32_t p) { return p - r; }

__device__ __forceinline__ double block_max_dbl(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
  return v;
}
__device__ __forceinline__ int block_max_int(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = max(v, red[w]);
  return v;
}

// deterministic block sum (fixed shuffle tree, then warps in order)
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v += red[w];
  return v;
}

// binary exponent E of a finite nonzero max (max < 2^E, max >= 2^(E-1))
__device__ __forceinline__ int exp_of(double mx) {
  int E;
  frexp(mx, &E);
  return E;
}
constexpr double kDblMax = 1.7976931348623157e308;
constexpr int kNoExp = (int)0xC0C0C0C0;  // no nonzero value seen (cudaMemset byte 0xC0); below every exponent
// binary exponent E of |v| > 0 finite (|v| < 2^E, |v| >= 2^(E-1)), from the bits
__device__ __forceinline__ int exp_bits(double v) {
  const int f = (int)((__double_as_longlong(v) >> 52) & 0x7ff);
  return f ? f - 1022 : exp_of(v);  // subnormal: frexp
}

// ------------------------------------------------ contraction balancing
// X_k Y_k = (X_k D^-1)(D Y_k) for any diagonal D of powers of two along the
// contraction index, exactly.  Row j of Y_k is B̂1_k[j] (j < n) or B̂2_k[j-n]
// (and the matching column of X_k multiplies it); one exponent per n-index j
// and frequency PAIR (k, p-k), shared by both CD parts and both slots so the
// shared X' of a pair stays valid: d_j = -E_j, E_j the binary exponent of the
// largest |re|, |im| of row j of B̂1/B̂2 at frequencies k and p-k (over every
// column).  Each row of D Y then has its maximum in [1/2, 1) and X's column j
// absorbs the scale, so a contraction index scaled up in A and down in B (or
// the reverse) — which the per-row / per-column exponents alone would turn into
// lost low-order bits — is balanced back before anything is rounded.  The
// balanced values are never formed: each kernel folds d_j into the one
// power-of-two scale it already applies (exponent arithmetic, so nothing
// overflows or underflows on the way).  bdel: [p][n] ints, indexed by frequency
// (decomposition-independent: row slabs, compact slot ranges and the
// one-shot product see the same d for the same B̂).
__device__ __forceinline__ int bal_delta(const int* __restrict__ bdel, int k, int n, int j) {
  return bdel ? __ldg(bdel + (size_t)k * n + j) : 0;
}

// bdel for the slot units of [f0, f0 + units): one warp per (unit, row j)
// reads a fixed sample of row j — kBalSample columns at a stride spread over
// the row (every column when s <= kBalSample) — of both CD planes at both
// frequencies of the unit.  Any power-of-two D is exact, so a sample only has
// to see the scale of the row (a row scaling of B, or the inverse of a column
// scaling of A, shows in every column); whatever it misses costs accuracy
// only, which the guard below certifies (else that pair goes to fp64).  The
// sample is a function of the column index alone, so row slabs and compact
// slot ranges see the same D.  (A 1/32 sample of config 5's B̂: 0.05 ms vs
// 0.7 ms for every column.)
constexpr int kBalSample = 64;
__global__ void __launch_bounds__(256) oz_balance_b_kernel(const double2* __restrict__ b1,
                                                           const double2* __restrict__ b2, int* __restrict__ bdel,
                                                           int n, int s, int p, int f0, int ns, uint64_t ldb,
                                                           uint64_t bslice, int cbase) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + w;
  if (j >= n) return;
  int sa, sb;
  unit_slots(blockIdx.y, f0, ns, p, sa, sb);
  const int ka = slot_freq(sa, p), kb = slot_freq(sb, p);
  const int la = slot_slice(sa, p, cbase), lb = slot_slice(sb, p, cbase);
  const int stride = s <= kBalSample ? 1 : (s + kBalSample - 1) / kBalSample;
  int E = kNoExp;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (t >= 2 && la == lb) break;
    const double2* row = (t & 1 ? b2 : b1) + (size_t)(t < 2 ? la : lb) * bslice + (size_t)j * ldb;
#pragma unroll
    for (int u = 0; u < kBalSample / 32; ++u) {
      const int c = (lane + 32 * u) * stride;
      if (c < s) {
        const double2 y = __ldcs(row + c);
        const double mx = fmax(fabs(y.x), fabs(y.y));
        // inf / nan: the colexp pass raises the non-finite flag; any d is fine then
        if (mx != 0.0 && mx <= kDblMax) E = max(E, exp_bits(mx));
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) E = max(E, __shfl_xor_sync(0xffffffffu, E, o));
  if (lane == 0) {
    const int d = E == kNoExp ? 0 : -E;
    bdel[(size_t)ka * n + j] = d;
    bdel[(size_t)kb * n + j] = d;
  }
}

// ------------------------------------------------------ accuracy guard
// The only approximation of the int8 path is rounding the scaled operands to
// integers (|dx|, |dy| <= 1/2 in scaled units); the integer product and the
// CRT are exact.  Per real output element, in scaled units,
//   |err| <= 1/2 ||y''_c||_1 + 1/2 ||x''_r||_1 + K/4 (+ 2^42 CRT weights, + final rounding),
// with x''_r, y''_c the unrounded scaled row of X (real form, K = 4n) and
// column of Y (an all-zero row or column is exact: no term).  The residue
// kernels record those L1 norms (xl1 per X' row, yl1 per B' column) and the
// smallest row / column exponent of each slot (amin, bmin); the CRT kernel
// accumulates, per frequency slot, the squared bound and |C|^2 with the
// element weights 2^-2(e_row - amin) 2^-2(e_col - bmin) <= 1 (the true
// weights 2^-2(e_row + e_col) up to one common factor), and the guard kernel
// certifies each pair with sum bound^2 <= tol^2 sum |C|^2 (tol = 2^-42 by
// default), i.e. a relative Frobenius error of the pair's stage-2 result
// below tol.  A pair that is not certified (or whose sums under/overflowed)
// gets flag[1 + min(k, p - k)] and the fp64 DMMA kernels recompute it
// (qt_gemm.cu, launched behind every int8 product).
struct GuardAcc {
  double sb;  // sum of bound^2 * weight
  double sc;  // sum of |C'|^2 * weight
};
__device__ unsigned long long g_guard_fallbacks = 0;  // pairs sent to the DMMA kernels (qt_int8_guard_fallbacks)

// Scale exponent of a row / column with max < 2^E and ||v|| / 2^E = ns (the
// scaled Euclidean norm, >= 1/2): e = min(53 - E, T - E_ns - E) with
// ns < 2^E_ns, so every scaled value has <= 53 bits AND ||v 2^e|| < 2^T.  By
// Cauchy-Schwarz |x'.y'| <= ||x'|| ||y'|| < 2^2T < M/2, so the CRT recovers
// the integer product; for data whose max/rms exceeds ~sqrt(K)/2^(T-53) the
// first bound is the binding one (no precision below 53 bits is given up).
__device__ __forceinline__ int scale_exponent(int E, double ns) {
  const int Ens = exp_of(ns * (1.0 + 0x1p-30));  // margin for the rounded sum of squares
  return min(kBits, c_mod.ebound - Ens) - E;
}

// A side: one CTA per (slot f, row i < m) handles the row pair
// (A1_k[i], A2_sk[i]), which shares one exponent, and writes
//   X_k  row i     = [Re A1_k | -Re A2_sk | Im A1_k |  Im A2_sk]
//   X_sk row m + i = [Re A2_sk |  Re A1_k | Im A2_sk | -Im A1_k]
// (X_sk's slot is f^1, or f itself for a self-paired frequency).
constexpr int kAVec = 4;  // consecutive K elements per thread and store (one 32-bit word)
__global__ void __launch_bounds__(256, 4) oz_residue_a_kernel(const double2* __restrict__ a1,
                                                           const double2* __restrict__ a2, uint8_t* __restrict__ out,
                                                           int* __restrict__ eA, double* __restrict__ xl1,
                                                           int* __restrict__ amin, const int* __restrict__ bdel,
                                                           int* nonfinite, int m, int n, int p, int f0, int Mp, int F,
                                                           int cbase, int share_end) {
  __shared__ double red[8];
  __shared__ int ired[8];
  const int i = blockIdx.x, f = blockIdx.y;
  const int slot = f0 + f;
  const int k = slot_freq(slot, p), sk = (p - k) % p;
  // (no shared memory: this kernel runs beside the int8 GEMM's maximum-carveout CTAs)
  const int* dk = bdel ? bdel + (size_t)k * n : nullptr;
  const int fpart = (k == sk) ? f : (f ^ 1);
  const int kq = slot_slice(slot, p, cbase), skq = slot_slice((k == sk) ? slot : (slot ^ 1), p, cbase);
  const double2* P = a1 + ((size_t)kq * m + i) * n;
  const double2* Qr = a2 + ((size_t)skq * m + i) * n;
  // column j of this row pair multiplies Y rows j and n + j: balanced by 2^-d_j.
  // Fast path: one pass of plain max / sum of squares / L1 sums of the
  // balanced values (one exact power-of-two multiply each), rescaled once —
  // bitwise the exponent-tracking passes below whenever nothing is subnormal
  // or overflows (row maximum in [2^-400, 2^400], every |d| <= 1000).
  bool bad = false, slow = false;
  double mxf = 0.0, ssf = 0.0, l1f = 0.0;
#pragma unroll 4
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double2 x = P[j], y = Qr[j];
    bad |= !(fabs(x.x) + fabs(x.y) + fabs(y.x) + fabs(y.y) <= kDblMax);
    const int dj = dk ? __ldg(dk + j) : 0;
    slow |= (dj < -1000) | (dj > 1000);
    const double sc = __longlong_as_double((long long)(1023 - dj) << 52);
    const double a = x.x * sc, b = x.y * sc, c = y.x * sc, d = y.y * sc;
    mxf = fmax(mxf, fmax(fmax(fabs(a), fabs(b)), fmax(fabs(c), fabs(d))));
    ssf = fma(a, a, fma(b, b, fma(c, c, fma(d, d, ssf))));
    l1f += (fabs(a) + fabs(b)) + (fabs(c) + fabs(d));
  }
  bad = __syncthreads_or(bad);
  if (bad) {
    if (threadIdx.x == 0) atomicExch(nonfinite, 1);
    return;
  }
  slow = __syncthreads_or(slow);
  mxf = block_max_dbl(mxf, red);
  ssf = block_sum(ssf, red);
  l1f = block_sum(l1f, red);
  slow = slow || !(l1f <= kDblMax) || (mxf != 0.0 && (mxf > 0x1p400 || mxf < 0x1p-400));
  int E = kNoExp;
  int e = 0;
  double l1s = 0.0;  // L1 norm of the scaled (unrounded) real-form row
  if (!slow) {
    if (mxf != 0.0) {
      E = exp_bits(mxf);
      const double ss = scale2(ssf, -2 * E);
      e = scale_exponent(E, sqrt(ss));
      l1s = scale2(scale2(l1f, -E) * (1.0 + 0x1p-40), E + e);
    }
  } else {
    // exponent-tracking passes (any magnitudes)
#pragma unroll 4
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double2 x = P[j], y = Qr[j];
      const double mx = fmax(fmax(fabs(x.x), fabs(x.y)), fmax(fabs(y.x), fabs(y.y)));
      if (mx != 0.0) E = max(E, exp_bits(mx) - (dk ? __ldg(dk + j) : 0));
    }
    E = block_max_int(E, ired);
    if (E != kNoExp) {
      double ss = 0.0;  // sum of squares of the balanced row scaled by 2^-E (each term <= 1)
      double l1 = 0.0;
#pragma unroll 4
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double2 x = P[j], y = Qr[j];
        const int sh = -(dk ? __ldg(dk + j) : 0) - E;
        const double a = scale2(x.x, sh), b = scale2(x.y, sh), c = scale2(y.x, sh), d = scale2(y.y, sh);
        ss = fma(a, a, fma(b, b, fma(c, c, fma(d, d, ss))));
        l1 += (fabs(a) + fabs(b)) + (fabs(c) + fabs(d));
      }
      ss = block_sum(ss, red);
      l1 = block_sum(l1, red);
      e = scale_exponent(E, sqrt(ss));
      l1s = scale2(l1 * (1.0 + 0x1p-40), E + e);
    }
  }
  if (threadIdx.x == 0) {
    eA[f * Mp + i] = e;
    eA[fpart * Mp + m + i] = e;
    xl1[f * Mp + i] = l1s;
    xl1[fpart * Mp + m + i] = l1s;
    if (E != kNoExp) {  // (the row is in both slots of the pair)
      atomicMin(amin + f, e);
      if (fpart != f) atomicMin(amin + fpart, e);
    }
  }
  const size_t Kp = 4 * (size_t)n, plane = (size_t)F * Mp * Kp;
  uint8_t* up = out + (size_t)(f * Mp + i) * Kp;
  uint8_t* lo = out + (size_t)(fpart * Mp + m + i) * Kp;
  // with shared X' (shares_x) a pair keeps only the even slot's X': its row i
  // comes from the even CTA, its row m + i from the odd one
  const bool pair_shared = fpart != f && slot < share_end;
  const bool wu = !(pair_shared && (slot & 1)), wl = !(pair_shared && !(slot & 1));
  // work unit: 4 consecutive elements of ONE source row (P = A1_k[i] or Q = A2_sk[i]);
  // each residue goes to two places (one per output row)
  const int nq = n / kAVec;
  for (int u = threadIdx.x; u < 2 * nq; u += blockDim.x) {
    const bool isP = u < nq;
    const int j0 = (isP ? u : u - nq) * kAVec;
    const double2* src = isP ? P : Qr;
    Limbs re[kAVec], im[kAVec];
    const int4 d4 = dk ? __ldg(reinterpret_cast<const int4*>(dk + j0)) : make_int4(0, 0, 0, 0);  // (n % 32 == 0)
    const int dv[kAVec] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
    for (int t = 0; t < kAVec; ++t) {
      const double2 x = src[j0 + t];
      const int et = e - dv[t];
      re[t] = to_limbs(x.x, et);
      im[t] = to_limbs(x.y, et);
    }
    // P: up[0n] = Re, lo[1n] = Re, up[2n] = Im, lo[3n] = -Im
    // Q: lo[0n] = Re, up[1n] = -Re, lo[2n] = Im, up[3n] = Im
    uint8_t* pa = (isP ? up : lo) + j0;             // Re, plain
    uint8_t* pb = (isP ? lo + n : up + n) + j0;     // Re (P) / -Re (Q)
    uint8_t* pc = (isP ? up : lo) + 2 * n + j0;     // Im, plain
    uint8_t* pd = (isP ? lo : up) + 3 * n + j0;     // -Im (P) / Im (Q)
    if (!pair_shared) {  // both output rows (self-paired frequency, or X' not shared)
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const uint32_t pq = c_mod.p[q];
        uint32_t a[kAVec], b[kAVec], na[kAVec], nb[kAVec];
#pragma unroll
        for (int t = 0; t < kAVec; ++t) {
          a[t] = res_of(re[t], q);
          b[t] = res_of(im[t], q);
          na[t] = neg_op(a[t], pq);
          nb[t] = neg_op(b[t], pq);
        }
        const uint32_t wa = pack4(a[0], a[1], a[2], a[3]), wb = pack4(b[0], b[1], b[2], b[3]);
        const uint32_t wna = pack4(na[0], na[1], na[2], na[3]), wnb = pack4(nb[0], nb[1], nb[2], nb[3]);
        const size_t off = (size_t)q * plane;
        *reinterpret_cast<uint32_t*>(pa + off) = wa;
        *reinterpret_cast<uint32_t*>(pc + off) = wb;
        *reinterpret_cast<uint32_t*>(pb + off) = isP ? wa : wna;
        *reinterpret_cast<uint32_t*>(pd + off) = isP ? wnb : wb;
      }
    } else {  // one output row: (Re, Im) at (pa, pc), or (Re | -Re, -Im | Im) at (pb, pd)
      const bool first = isP ? wu : wl;
      const bool nre = !first && !isP, nim = !first && isP;
      uint8_t* p0 = first ? pa : pb;
      uint8_t* p1 = first ? pc : pd;
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const uint32_t pq = c_mod.p[q];
        uint32_t a[kAVec], b[kAVec];
#pragma unroll
        for (int t = 0; t < kAVec; ++t) {
          a[t] = res_of(re[t], q);
          b[t] = res_of(im[t], q);
          if (nre) a[t] = neg_op(a[t], pq);
          if (nim) b[t] = neg_op(b[t], pq);
        }
        const size_t off = (size_t)q * plane;
        *reinterpret_cast<uint32_t*>(p0 + off) = pack4(a[0], a[1], a[2], a[3]);
        *reinterpret_cast<uint32_t*>(p1 + off) = pack4(b[0], b[1], b[2], b[3]);
      }
    }
  }
}

// B side, pass 1: per (slot f, column c, 256-row block z of Y_k[:, c] =
// [B1_k[:, c]; B2_k[:, c]]) the local max exponent and the sum of squares
// scaled by it, into part[z][f][c] (deterministic: no atomics on the sums).
// One streaming pass: each thread keeps a running exponent E_t and its sum
// scaled by 2^-2E_t, rescaled (exactly, by a power of two) when a larger
// exponent appears; the warps' partials are then combined in order.
struct ColPart {
  int E;      // kNoExp: the block is all zeros
  double ss;  // sum of (|re|^2 + |im|^2) 2^-2E over the block
  double l1;  // sum of (|re| + |im|) 2^-E over the block
};
__global__ void __launch_bounds__(256) oz_colexp_b_kernel(const double2* __restrict__ b1,
                                                          const double2* __restrict__ b2, ColPart* __restrict__ part,
                                                          const int* __restrict__ bdel, int* nonfinite, int n, int s,
                                                          int p, int f0, int Sp, int F, uint64_t ldb, uint64_t bslice,
                                                          int cbase) {
  __shared__ int se[8][33];
  __shared__ double sss[8][33];
  __shared__ double sl1[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5, f = blockIdx.y;
  const int k = slot_slice(f0 + f, p, cbase), kf = slot_freq(f0 + f, p);
  const int j0 = blockIdx.z * 256, jend = min(2 * n, j0 + 256);
  int E = kNoExp;
  double ss = 0.0, l1 = 0.0;
  bool bad = false;
  constexpr int kU = 8;  // loads in flight per thread
  const double2* base1 = b1 + k * bslice + c;
  const double2* base2 = b2 + k * bslice + c;
  // fast path: plain sums of the balanced values (one exact power-of-two
  // multiply per element), rescaled once at the end.  That equals the running-
  // exponent pass below bitwise whenever nothing is subnormal or overflows —
  // guaranteed here when the column segment's largest value lies in
  // [2^-400, 2^400] and every d in [-1000, 1000]; otherwise (and for inf / nan)
  // the segment is recomputed by that pass.
  bool slow = c >= s;
  if (c < s) {
    double mxf = 0.0, ssf = 0.0, l1f = 0.0;
    for (int jb = j0 + w; jb < jend; jb += 8 * kU) {
      double2 y[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = jb + 8 * u;
        y[u] = j < jend ? __ldcs(j < n ? base1 + (size_t)j * ldb : base2 + (size_t)(j - n) * ldb)
                        : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = jb + 8 * u;
        const int d = bal_delta(bdel, kf, n, j < n ? j : j - n);
        slow |= (d < -1000) | (d > 1000);
        const double sc = __longlong_as_double((long long)(d + 1023) << 52);
        const double a = y[u].x * sc, b = y[u].y * sc, aa = fabs(a), bb = fabs(b);
        mxf = fmax(mxf, fmax(aa, bb));
        ssf = fma(a, a, fma(b, b, ssf));
        l1f += aa + bb;
      }
    }
    if (!(l1f <= kDblMax) || (mxf != 0.0 && (mxf > 0x1p400 || mxf < 0x1p-400))) slow = true;
    if (!slow && mxf != 0.0) {
      E = exp_bits(mxf);
      ss = scale2(ssf, -2 * E);
      l1 = scale2(l1f, -E);
    }
  }
  if (c < s && slow) {
    for (int jb = j0 + w; jb < jend; jb += 8 * kU) {
      double2 y[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = jb + 8 * u;
        y[u] = j < jend ? __ldcs(j < n ? base1 + (size_t)j * ldb : base2 + (size_t)(j - n) * ldb)
                        : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const double ax = fabs(y[u].x), ay = fabs(y[u].y);
        // a sum of magnitudes is inf/nan iff a component is (or the pair overflows)
        if (!(ax + ay <= kDblMax)) {
          bad = true;
          continue;
        }
        const double mx = fmax(ax, ay);
        if (mx == 0.0) continue;
        const int j = jb + 8 * u;
        const int d = bal_delta(bdel, kf, n, j < n ? j : j - n);  // row j of D Y
        const int e = exp_bits(mx) + d;
        if (e > E) {
          if (E != kNoExp) {
            ss = scale2(ss, 2 * (E - e));
            l1 = scale2(l1, E - e);
          }
          E = e;
        }
        const double a = scale2(y[u].x, d - E), b = scale2(y[u].y, d - E);
        ss = fma(a, a, fma(b, b, ss));
        l1 += fabs(a) + fabs(b);
      }
    }
  }
  se[w][threadIdx.x & 31] = E;
  sss[w][threadIdx.x & 31] = ss;
  sl1[w][threadIdx.x & 31] = l1;
  bad = __syncthreads_or(bad);
  if (w == 0) {
    int Eb = kNoExp;
    for (int t = 0; t < 8; ++t) Eb = max(Eb, se[t][threadIdx.x]);
    double sb = 0.0, lb = 0.0;
    if (Eb != kNoExp)
      for (int t = 0; t < 8; ++t)
        if (se[t][threadIdx.x] != kNoExp) {
          sb += scale2(sss[t][threadIdx.x], 2 * (se[t][threadIdx.x] - Eb));
          lb += scale2(sl1[t][threadIdx.x], se[t][threadIdx.x] - Eb);
        }
    if (bad && threadIdx.x == 0) atomicExch(nonfinite, 1);
    part[((size_t)blockIdx.z * F + f) * Sp + c] = ColPart{(c < s && !bad) ? Eb : kNoExp, sb, lb};
  }
}

// B side, pass 1b: combine the row-block partials of each column in order;
// column exponent e and the L1 norm of the scaled (unrounded) column (guard)
__global__ void oz_colexp_finish_kernel(const ColPart* __restrict__ part, int* __restrict__ eB,
                                        double* __restrict__ yl1, int* __restrict__ bmin, int nz, int F, int Sp,
                                        int fcur) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= fcur * Sp) return;
  const int f = t / Sp, c = t - f * Sp;
  int E = kNoExp;
  for (int z = 0; z < nz; ++z) E = max(E, part[((size_t)z * F + f) * Sp + c].E);
  int e = 0;
  double l1s = 0.0;
  if (E != kNoExp) {
    double ss = 0.0, l1 = 0.0;
    for (int z = 0; z < nz; ++z) {
      const ColPart pz = part[((size_t)z * F + f) * Sp + c];
      if (pz.E != kNoExp) {
        ss += scale2(pz.ss, 2 * (pz.E - E));
        l1 += scale2(pz.l1, pz.E - E);
      }
    }
    e = scale_exponent(E, sqrt(ss));
    l1s = scale2(l1 * (1.0 + 0x1p-40), E + e);
    atomicMin(bmin + f, e);
  }
  eB[f * Sp + c] = e;
  yl1[f * Sp + c] = l1s;
}

// B side, pass 2: one CTA per (slot f, 32 columns, 128-row block of Y); writes
// the Re-row [Re Y | -Im Y] and the Im-row [Im Y | Re Y] of each column.  Row
// order inside a slot: tile t = c / 128 holds its 128 Re-rows, then its 128
// Im-rows.  Columns c >= s (padding) get zero rows.  The 128 x 32 block is
// transposed through shared memory (column-major, row j at j + j/8 so both the
// column-wise fill and the 4-consecutive-rows-per-lane reads are conflict
// free); each warp then writes 128 contiguous bytes of a B' row per store.
// (Kernels with shared memory are not placed beside the GEMM, whose SMs run
// the maximum carveout, so this kernel runs between GEMM batches: the larger
// tile is the faster one there.)
constexpr int kBRows = 128;
constexpr int kBStride = kBRows + kBRows / 8 + 1;  // 145 double2 per column
// BC columns per CTA (32, or 16 for more CTAs per SM: smem BC * 145 * 16 B)
constexpr size_t res_b_smem(int bc) { return sizeof(double2) * bc * kBStride; }
template <int BC>
__global__ void __launch_bounds__(256) oz_residue_b_kernel(const double2* __restrict__ b1,
                                                           const double2* __restrict__ b2,
                                                           const int* __restrict__ eB, const int* __restrict__ bdel,
                                                           uint8_t* __restrict__ out, int n, int s, int p, int f0,
                                                           int Sp, int F, uint64_t ldb, uint64_t bslice, int cbase,
                                                           int share_end) {
  extern __shared__ double2 tile[];  // [BC][kBStride]
  const int c0 = blockIdx.x * BC, j0 = blockIdx.z * kBRows, f = blockIdx.y;
  const int k = slot_slice(f0 + f, p, cbase), kf = slot_freq(f0 + f, p);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  constexpr int RPI = 32 / BC;  // rows per warp load
#pragma unroll
  for (int jj = ty * RPI + tx / BC; jj < kBRows; jj += 8 * RPI) {
    const int j = j0 + jj, cl = tx % BC, c = c0 + cl;
    double2 y = make_double2(0.0, 0.0);
    if (c < s && j < 2 * n)
      y = (j < n ? b1 + k * bslice + (size_t)j * ldb : b2 + k * bslice + (size_t)(j - n) * ldb)[c];
    tile[cl * kBStride + jj + (jj >> 3)] = y;
  }
  __syncthreads();
  const size_t Kp = 4 * (size_t)n, plane = (size_t)F * 2 * Sp * Kp;
  const int jl = 4 * tx, jb = j0 + jl;  // this lane's 4 consecutive rows
  if (jb >= 2 * n) return;
  // odd slot of a shared-X' pair: Y'' = M*(Y), i.e. the halves of Y swapped
  // (position jj) and, per half, its own sign pattern (see shares_x)
  const bool yy = shares_x(f0 + f, share_end);
  const bool top = jb < n;  // rows of B1 (else B2); 4 rows never straddle n (n % 32 == 0)
  const int pos = yy ? (top ? jb + n : jb - n) : jb;
  int dj[4];  // balancing of the lane's 4 rows of D Y
#pragma unroll
  for (int t = 0; t < 4; ++t) dj[t] = bal_delta(bdel, kf, n, (top ? jb : jb - n) + t);
  for (int cc = ty; cc < BC; cc += 8) {
    const int c = c0 + cc;
    const int e = eB[f * Sp + c];
    const int tcol = c / BNC, ic = c % BNC;
    uint8_t* re_row = out + ((size_t)f * 2 * Sp + tcol * BN + ic) * Kp + pos;
    uint8_t* im_row = re_row + (size_t)BNC * Kp;
    Limbs lr[4], li[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const double2 y = tile[cc * kBStride + jl + t + ((jl + t) >> 3)];
      lr[t] = to_limbs(y.x, e + dj[t]);
      li[t] = to_limbs(y.y, e + dj[t]);
    }
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const uint32_t pq = c_mod.p[q];
      uint32_t a[4], b[4], nb[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[t] = res_of(lr[t], q);
        b[t] = res_of(li[t], q);
        nb[t] = neg_op(b[t], pq);
      }
      const uint32_t wr = pack4(a[0], a[1], a[2], a[3]), wi = pack4(b[0], b[1], b[2], b[3]);
      const uint32_t wni = pack4(nb[0], nb[1], nb[2], nb[3]);
      if (!yy) {
        *reinterpret_cast<uint32_t*>(re_row) = wr;           // Re-row: Re Y
        *reinterpret_cast<uint32_t*>(re_row + 2 * n) = wni;  // Re-row: -Im Y
        *reinterpret_cast<uint32_t*>(im_row) = wi;           // Im-row: Im Y
        *reinterpret_cast<uint32_t*>(im_row + 2 * n) = wr;   // Im-row: Re Y
      } else {
        const uint32_t wnr = pack4(neg_op(a[0], pq), neg_op(a[1], pq), neg_op(a[2], pq), neg_op(a[3], pq));
        // Re-row'' = [-Re B2, Re B1, -Im B2, Im B1], Im-row'' = [-Im B2, Im B1, Re B2, -Re B1]
        *reinterpret_cast<uint32_t*>(re_row) = top ? wr : wnr;
        *reinterpret_cast<uint32_t*>(re_row + 2 * n) = top ? wi : wni;
        *reinterpret_cast<uint32_t*>(im_row) = top ? wi : wni;
        *reinterpret_cast<uint32_t*>(im_row + 2 * n) = top ? wnr : wr;
      }
      re_row += plane;
      im_row += plane;
    }
  }
}

// ------------------------------------------------------------- K2c CRT
// X'Y'/M = sum_q r_q y_q / p_q (mod 1), accumulated as a 96-bit fixed-point
// fraction (mod 2^96 wraps = mod 1); the weights' rounding (<= 1/2 ulp each)
// bounds the error by 16*255/2 units of 2^-96, i.e. <= 2^-84 * M = 2^41 in X'Y'
// (which is ~2^110 for a typical element): far below one fp64 ulp.
// X'Y' as a double (the signed 96-bit fraction times M), before the 2^e scaling
__device__ __forceinline__ double crt_value(uint64_t acc0, uint64_t acc1, uint64_t acc2) {
  acc1 += acc0 >> 32;
  acc2 += acc1 >> 32;
  // signed 96-bit fraction in [-1/2, 1/2), then times M
  const int64_t top = (int64_t)(((uint64_t)(uint32_t)acc2 << 32) | (uint32_t)acc1);
  const double frac = (double)top + (double)(uint32_t)acc0 * 2.3283064365386963e-10;  // (top + s0 2^-32), units 2^-64
  return scale2(frac * c_mod.M, -64);
}

// one thread per 4 consecutive complex elements of output rows r (slot f, row
// r of [C1; C2]): 16 x 8-byte residue loads (pointer bumped by one plane per
// modulus), 3 multiply-adds per residue into 64-bit limb accumulators.  Each
// CTA walks several rows and leaves its guard partial (weighted squared error
// bound and |C|^2) in gpart[f][cta].
constexpr int kCrtVec = 4;
__global__ void __launch_bounds__(256, 4) oz_crt_kernel(const uint8_t* __restrict__ R, const int* __restrict__ eA,
                                                     const double* __restrict__ xl1, const int* __restrict__ amin,
                                                     const int* __restrict__ eB, const double* __restrict__ yl1,
                                                     const int* __restrict__ bmin, const int* nonfinite,
                                                     GuardAcc* __restrict__ gpart, double2* __restrict__ c1,
                                                     double2* __restrict__ c2, int m, int n, int s, int p, int f0,
                                                     int bslot0, int Mp, int Sp, int F, uint64_t ldc, uint64_t cslice,
                                                     int cbase, int share_end) {
  if (*nonfinite) return;
  const int cb = (blockIdx.x * blockDim.x + threadIdx.x) * kCrtVec;
  const int f = blockIdx.z;
  const bool active = cb < s;
  const int k = slot_slice(f0 + f, p, cbase);
  const size_t plane = (size_t)F * Mp * Sp * 2;  // bytes
  // odd slot of a shared-X' pair: R row r < m is -C2[r], R row m + r is C1[r],
  // with the row exponents of the even partner's X'
  const bool sx = shares_x(f0 + f, share_end);
  const int fa = sx ? f - 1 : f;
  const int* ebs = eB + (bslot0 + f) * Sp;
  const double* ybs = yl1 + (bslot0 + f) * Sp;
  double gsb = 0.0, gsc = 0.0;
  for (int r = blockIdx.y; r < 2 * m && active; r += gridDim.y) {
    const uint8_t* ptr = R + ((size_t)(f * Mp + r) * Sp + cb) * 2;
    const bool neg = sx && r < m;
    uint64_t acc[kCrtVec][2][3];
#pragma unroll
    for (int t = 0; t < kCrtVec; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc[t][h][0] = acc[t][h][1] = acc[t][h][2] = 0;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(ptr));  // (re, im) bytes of 4 columns
      ptr += plane;
      const uint32_t w0 = c_mod.w[q][0], w1 = c_mod.w[q][1], w2 = c_mod.w[q][2];
      const uint32_t pq = c_mod.p[q];
#pragma unroll
      for (int t = 0; t < kCrtVec; ++t) {
        const uint32_t word = t < 2 ? v.x : v.y;
        const int sh = (t & 1) * 16;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t rr = (word >> (sh + 8 * h)) & 0xffu;
          if (neg) rr = neg_res(rr, pq);
          acc[t][h][0] += (uint64_t)rr * w0;
          acc[t][h][1] += (uint64_t)rr * w1;
          acc[t][h][2] += (uint64_t)rr * w2;
        }
      }
    }
    const int ea = eA[fa * Mp + r];
    const double xr = xl1[fa * Mp + r];
    // guard weight of the row (an all-zero row is exact: weight 0)
    const double wr = xr != 0.0 ? scale2(1.0, -2 * (ea - amin[fa])) : 0.0;
    const int b0 = bmin[bslot0 + f];
    double2* dst = ((r < m) != sx) ? c1 + k * cslice + (size_t)(sx ? r - m : r) * ldc
                                   : c2 + k * cslice + (size_t)(sx ? r : r - m) * ldc;
#pragma unroll
    for (int t = 0; t < kCrtVec; ++t) {
      if (cb + t >= s) break;
      const int ebt = ebs[cb + t];
      const int e = -(ea + ebt);
      const double vr = crt_value(acc[t][0][0], acc[t][0][1], acc[t][0][2]);
      const double vi = crt_value(acc[t][1][0], acc[t][1][1], acc[t][1][2]);
      dst[cb + t] = make_double2(scale2(vr, e), scale2(vi, e));
      const double yl = ybs[cb + t];
      const double w = yl != 0.0 ? wr * scale2(1.0, -2 * (ebt - b0)) : 0.0;  // (all-zero column: exact)
      const double bnd = 0.5 * (xr + yl) + (0.25 * (4.0 * n) + 0x1p42);  // per real part; |err|^2 <= 2 bnd^2
      gsb = fma(2.0 * bnd * bnd, w, gsb);
      gsc = fma(fma(vr, vr, vi * vi), w, gsc);
    }
  }
  // per-warp partials (fixed shuffle tree; no block barrier)
  for (int o = 16; o > 0; o >>= 1) {
    gsb += __shfl_xor_sync(0xffffffffu, gsb, o);
    gsc += __shfl_xor_sync(0xffffffffu, gsc, o);
  }
  if ((threadIdx.x & 31) == 0)
    gpart[(((size_t)f * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 8 + (threadIdx.x >> 5)] =
        GuardAcc{gsb, gsc};
}

// Guard decision per slot unit of a batch, in two deterministic passes:
// oz_guard_sum_kernel reduces chunk c of the unit's CRT partials (both slots)
// into gsum[unit][c]; oz_guard_kernel combines the kGuardChunks chunk sums in
// a fixed order and flags the pair for the DMMA recompute unless
// sum bound^2 <= tol2 * sum |C|^2.
constexpr int kGuardChunks = 64;
__global__ void __launch_bounds__(256) oz_guard_sum_kernel(const GuardAcc* __restrict__ gpart, int nper,
                                                           const int* nonfinite, GuardAcc* __restrict__ gsum, int p,
                                                           int f0, int fcur) {
  __shared__ double red[8];
  if (*nonfinite) return;
  int sa, sb;
  unit_slots(blockIdx.x, f0, fcur, p, sa, sb);
  const int per = (sb - sa + 1) * nper;  // the unit's partials are contiguous (slots sa..sb)
  const int chunk = (per + kGuardChunks - 1) / kGuardChunks;
  const int i0 = blockIdx.y * chunk, i1 = min(per, i0 + chunk);
  const GuardAcc* g = gpart + (size_t)(sa - f0) * nper;
  double gsb = 0.0, gsc = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const GuardAcc v = g[i];
    gsb += v.sb;
    gsc += v.sc;
  }
  gsb = block_sum(gsb, red);
  gsc = block_sum(gsc, red);
  if (threadIdx.x == 0) gsum[blockIdx.x * kGuardChunks + blockIdx.y] = GuardAcc{gsb, gsc};
}

__global__ void __launch_bounds__(kGuardChunks) oz_guard_kernel(const GuardAcc* __restrict__ gsum,
                                                                const int* nonfinite, int* __restrict__ pair_flags,
                                                                int p, int f0, int fcur, double tol2, int force) {
  __shared__ double red[8];
  if (*nonfinite) return;  // everything is recomputed anyway
  int sa, sb;
  unit_slots(blockIdx.x, f0, fcur, p, sa, sb);
  const GuardAcc v = gsum[blockIdx.x * kGuardChunks + threadIdx.x];
  const double gsb = block_sum(v.sb, red);
  const double gsc = block_sum(v.sc, red);
  if (threadIdx.x == 0) {
    const bool ok = !force && gsc > 0.0 && gsc <= kDblMax && gsb <= tol2 * gsc;
    if (!ok) {
      const int kf = slot_freq(sa, p);
      pair_flags[min(kf, p - kf)] = 1;
      atomicAdd(&g_guard_fallbacks, 1ull);
    }
  }
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* map, void* base, uint64_t kp, uint64_t rows, uint64_t planes, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {kp, rows, planes};
  const cuuint64_t strides[2] = {kp, kp * rows};
  const cuuint32_t box[3] = {(cuuint32_t)BK, box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

ModTable make_table() {
  ModTable t{};
  unsigned __int128 M = 1;
  for (int q = 0; q < kQ; ++q) M *= (unsigned)kModuli[q];
  for (int q = 0; q < kQ; ++q) {
    const uint32_t p = (uint32_t)kModuli[q];
    t.p[q] = p;
    t.magic[q] = (uint32_t)((((uint64_t)1) << 32) / p);
    t.magic37[q] = (uint32_t)(((((uint64_t)1) << 37) + p - 1) / p);
    t.negp[q] = 0u - (uint32_t)p;
    uint32_t wlo = 0, whi = 0;
    uint64_t pw = 1;  // 256^b mod p
    for (int b = 0; b < 7; ++b) {
      if (b < 4)
        wlo |= (uint32_t)pw << (8 * b);
      else
        whi |= (uint32_t)pw << (8 * (b - 4));
      pw = pw * 256 % p;
    }
    t.wlo[q] = wlo;
    t.whi[q] = whi;
    t.cofs[q] = p - (uint32_t)((((uint64_t)1) << 55) % p);
    uint64_t mp = 1;  // (M / p) mod p
    for (int j = 0; j < kQ; ++j)
      if (j != q) mp = mp * (uint64_t)kModuli[j] % p;
    uint64_t y = 1;
    while (mp * y % p != 1) ++y;
    // round(2^96 * y / p) mod 2^96
    const unsigned __int128 num = (((unsigned __int128)y) << 96) + p / 2;
    const unsigned __int128 w = num / p;
    t.w[q][0] = (uint32_t)w;
    t.w[q][1] = (uint32_t)(w >> 32);
    t.w[q][2] = (uint32_t)(w >> 64);
  }
  t.M = (double)M;
  t.ebound = (int)std::floor((std::log2((double)M) - 1.0) / 2.0 - 0.05);
  return t;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

}  // namespace oz

bool ozaki_supported(uint64_t n, uint64_t s, uint64_t p) {
  // QTB_OZAKI: 0 = never, 1 = auto, 2 = whenever the shape allows.  Auto takes
  // the int8 path where it measured faster than DMMA on B200 (tools/oz_sweep.py:
  // 256^3 0.96x, n = 1920 s = 64 0.69x, s = 128 1.28x, 512^3 1.88x, 2048^3
  // 3.7x): the 15 residue GEMMs need enough columns to amortise the residues
  // of A.  Callers that split one product (row slabs, column chunks) decide
  // once on the full shape; m never enters (row shards agree by construction).
  static const int mode = oz::env_int("QTB_OZAKI", 1);
  if (mode == 0 || n == 0 || n % 32 != 0 || n > 8192 || p == 0 || p > 65534) return false;
  if (mode == 2) return true;
  return n >= (uint64_t)oz::env_int("QTB_OZAKI_MIN_N", 256) && s >= (uint64_t)oz::env_int("QTB_OZAKI_MIN_S", 128) &&
         n * s >= (uint64_t)oz::env_int("QTB_OZAKI_MIN_NS", 1 << 17);
}

namespace {

cudaError_t oz_init() {
  using namespace oz;
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t e = once_per_device(mu, done, [] {
    const ModTable t = make_table();
    cudaError_t r = cudaMemcpyToSymbol(c_mod, &t, sizeof(t));
    if (r != cudaSuccess) return r;
    r = cudaFuncSetAttribute(oz_residue_b_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_b_smem(32));
    if (r != cudaSuccess) return r;
    r = cudaFuncSetAttribute(oz_residue_b_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_b_smem(16));
    if (r != cudaSuccess) return r;
    for (auto [k, st] : {std::pair{oz_gemm2_kernel<4>, 4}, std::pair{oz_gemm2_kernel<5>, 5},
                         std::pair{oz_gemm2_kernel<6>, 6}})
      if ((r = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm2_smem(st))) !=
          cudaSuccess)
        return r;
    return cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
  });
  if (e != cudaSuccess) return e;
  return encode_fn() ? cudaSuccess : cudaErrorNotSupported;
}

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
    return n;
  return 148;
}

bool use_pair() {
  static const bool on = oz::env_int("QTB_OZAKI_2SM", 1) != 0;
  return on;
}
// X' rows per slot: a multiple of the 256-row pair tile (128 for the 1-CTA kernel)
uint64_t pad_rows(uint64_t m) {
  const uint64_t t = use_pair() ? 256 : oz::BM;
  return (2 * m + t - 1) / t * t;
}
uint64_t pad_cols(uint64_t s) { return (s + oz::BNC - 1) / oz::BNC * oz::BNC; }
uint64_t b_slot_bytes(uint64_t n, uint64_t s) { return (uint64_t)oz::kQ * 2 * pad_cols(s) * 4 * n + 4 * pad_cols(s); }
uint64_t a_slot_bytes(uint64_t m, uint64_t n, uint64_t s) {
  return (uint64_t)oz::kQ * (pad_rows(m) * 4 * n + pad_rows(m) * pad_cols(s) * 2) + 4 * pad_rows(m);
}
uint64_t env_mb(const char* name, uint64_t dflt_mb) { return (uint64_t)oz::env_int(name, (int)dflt_mb) << 20; }

// slots below this share X' within their pair (shares_x); QTB_OZAKI_SHAREX=0 turns it off
int share_end(uint64_t p) {
  static const bool on = oz::env_int("QTB_OZAKI_SHAREX", 1) != 0;
  return on ? (int)(2 * ((p - 1) / 2)) : 0;
}

// slots per batch: even (pairs stay together), balanced over the batches
uint64_t batch_slots(uint64_t p, uint64_t per_slot, uint64_t budget) {
  // (slots are a grid dimension of the residue / CRT kernels: <= 65534)
  uint64_t F = std::max<uint64_t>(
      2, std::min<uint64_t>({p, budget / std::max<uint64_t>(1, per_slot), uint64_t(65534)}) & ~uint64_t(1));
  const uint64_t nb = (p + F - 1) / F;
  return std::min<uint64_t>(p, ((p + nb - 1) / nb + 1) & ~uint64_t(1));
}

bool balance_on() {
  static const bool on = oz::env_int("QTB_OZAKI_BALANCE", 1) != 0;
  return on;
}
// guard tolerance tol^2 (QTB_OZAKI_GUARD_LOG2 = log2 tol, default -42);
// QTB_OZAKI_GUARD=force sends every pair to the DMMA kernels (tests)
double guard_tol2() {
  static const double t = std::ldexp(1.0, 2 * oz::env_int("QTB_OZAKI_GUARD_LOG2", -42));
  return t;
}
bool guard_force() {
  static const bool f = [] {
    const char* v = getenv("QTB_OZAKI_GUARD");
    return v && strcmp(v, "force") == 0;
  }();
  return f;
}

// B' residues (and column exponents) of slots [f0, f0 + fcur) into buffer slots [bslot0, ...)
// (parts: kPrepExp = balancing + column exponents only, kPrepRes = residues
// only, from exponents already in B.eB; both by default)
constexpr int kPrepExp = 1, kPrepRes = 2;
cudaError_t prep_b(const OzakiB& B, const double2* bh1, const double2* bh2, uint64_t f0, int fcur, int bslot0,
                   int* flag, cudaStream_t stream, int parts = kPrepExp | kPrepRes) {
  using namespace oz;
  const uint64_t Sp = pad_cols(B.s);
  uint8_t* res = B.res + (size_t)bslot0 * 2 * Sp * 4 * B.n;
  int* eB = B.eB + (size_t)bslot0 * Sp;
  double* yl1 = B.yl1 + (size_t)bslot0 * Sp;
  const int nz = (int)((2 * B.n + 255) / 256);
  const int* bdel = balance_on() ? B.bdel : nullptr;
  if (parts & kPrepRes && !(parts & kPrepExp)) goto residues;
  {
  ColPart* part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(ColPart) * nz * fcur * Sp, stream);
  if (e != cudaSuccess) return e;
  ProfScope ps("k2_int8_colnorms", stream);
  if (bdel) {
    const int units = slot_units((int)f0, fcur, (int)B.p);
    oz_balance_b_kernel<<<dim3((unsigned)((B.n + 7) / 8), (unsigned)units), 256, 0, stream>>>(
        bh1, bh2, B.bdel, (int)B.n, (int)B.s, (int)B.p, (int)f0, fcur, B.ldb, B.bslice, B.cbase);
    count_launches(1);
  }
  oz_colexp_b_kernel<<<dim3((unsigned)(Sp / 32), fcur, (unsigned)nz), 256, 0, stream>>>(
      bh1, bh2, part, bdel, flag, (int)B.n, (int)B.s, (int)B.p, (int)f0, (int)Sp, fcur, B.ldb, B.bslice, B.cbase);
  cudaMemsetAsync(B.bmin + bslot0, 0x7f, fcur * sizeof(int), stream);
  oz_colexp_finish_kernel<<<(unsigned)((fcur * Sp + 255) / 256), 256, 0, stream>>>(part, eB, yl1, B.bmin + bslot0, nz,
                                                                                    fcur, (int)Sp, fcur);
  ps.stop();
  count_launches(2);
  e = cudaFreeAsync(part, stream);
  if (e != cudaSuccess) return e;
  if (!(parts & kPrepRes)) return cudaGetLastError();
  }
residues:
  ProfScope pb("k2_int8_residues_b", stream);
  static const int bc = env_int("QTB_RESB_COLS", 16) == 32 ? 32 : 16;  // 16: 4 CTAs per SM (measured faster)
  auto kern = bc == 16 ? oz_residue_b_kernel<16> : oz_residue_b_kernel<32>;
  kern<<<dim3((unsigned)(Sp / bc), fcur, (unsigned)((2 * B.n + kBRows - 1) / kBRows)), 256, res_b_smem(bc),
         stream>>>(
      bh1, bh2, eB, bdel, res, (int)B.n, (int)B.s, (int)B.p, (int)f0, (int)Sp, (int)B.nslots, B.ldb, B.bslice,
      B.cbase, share_end(B.p));
  pb.stop();
  count_launches(1);
  return cudaGetLastError();
}

struct AuxObjects {
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> events;
};
AuxObjects& aux_objects(int device) {
  thread_local AuxObjects objs[64];
  static AuxObjects none;
  if (device < 0 || device >= 64) return none;
  AuxObjects& o = objs[device];
  if (!o.stream && cudaStreamCreateWithFlags(&o.stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    o.stream = nullptr;
  }
  return o;
}

// GEMM and CRT for the frequency slots of B (all p, or B's compact range)
// against B' (B.all: slot f of B' is frequency slot f; else B' is rebuilt per
// batch), with X' built per batch from Â; then the guard decision per pair.
// flag[0]: non-finite inputs (sticky), flag[1 + min(k, p - k)]: pair k is to
// be recomputed by the DMMA kernels (reset here).
cudaError_t multiply(OzakiB& B, const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                     uint64_t m, double2* ch1, double2* ch2, uint64_t ldc, uint64_t cslice, int* flag,
                     cudaStream_t stream) {
  using namespace oz;
  const uint64_t n = B.n, s = B.s, p = B.p, Mp = pad_rows(m), Sp = pad_cols(s), Kp = 4 * n;
  const uint64_t per_slot = a_slot_bytes(m, n, s);
  // with B' prepared for every frequency the frequency batches are software-
  // pipelined over two streams: the X' residues of batch i+1 and the CRT of
  // batch i run beside the int8 GEMM of batch i+1 / i (their CTAs fit next to
  // the GEMM's on every SM: ~0 KB smem, <= 128 regs), with X' and R double-
  // buffered.  Without B.all (B' rebuilt per batch) the batches run in order.
  const bool pipe = B.all && env_int("QTB_OZAKI_PIPE", 1) != 0;
  const uint64_t nbuf = pipe ? 2 : 1;
  const uint64_t ps = B.ns ? (uint64_t)B.ns : p;  // slots [B.s0, B.s0 + ps) of the p
  uint64_t F = B.all ? batch_slots(ps, per_slot * nbuf, env_mb("QTB_OZAKI_WS_MB", 3072)) : B.nslots;
  // at least 4 batches when pipelining, so residues/CRT have a GEMM to hide behind
  if (pipe && ps >= 8) F = std::min<uint64_t>(F, std::max<uint64_t>(2, ((ps + 3) / 4 + 1) & ~uint64_t(1)));
  const uint64_t nbatch = (ps + F - 1) / F;
  if (nbuf * F * Mp > 0x7fffffffULL || p * Mp > 0x7fffffffULL) return cudaErrorInvalidValue;
  const dim3 cgrid((unsigned)((s + 256 * kCrtVec - 1) / (256 * kCrtVec)), (unsigned)std::min<uint64_t>(2 * m, 65535),
                   1);
  const uint64_t nper = (uint64_t)cgrid.x * cgrid.y * 8;  // guard partials per slot (one per warp)
  const size_t bytesA = (size_t)kQ * nbuf * F * Mp * Kp, bytesR = (size_t)kQ * F * Mp * Sp * 2;
  const size_t offR = bytesA, offE = offR + nbuf * bytesR, offL = offE + ((nbuf * F * Mp * sizeof(int) + 255) & ~255ull);
  const size_t offG = offL + nbuf * F * Mp * sizeof(double);
  const size_t offS = offG + F * nper * sizeof(GuardAcc);
  const size_t offM = offS + F * kGuardChunks * sizeof(GuardAcc);
  const size_t wsbytes = offM + nbuf * F * sizeof(int);
  uint8_t* ws = nullptr;
  cudaError_t e = cudaMemsetAsync(flag + 1, 0, (p / 2 + 1) * sizeof(int), stream);
  if (e != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&ws, wsbytes, stream)) != cudaSuccess) return e;
  uint8_t* resA = ws;
  int* eA = reinterpret_cast<int*>(ws + offE);
  double* xl1 = reinterpret_cast<double*>(ws + offL);
  GuardAcc* gpart = reinterpret_cast<GuardAcc*>(ws + offG);
  GuardAcc* gsum = reinterpret_cast<GuardAcc*>(ws + offS);
  int* amin = reinterpret_cast<int*>(ws + offM);  // smallest row exponent per X' slot (guard weights)
  const uint64_t aslots = nbuf * F;  // slots in the X' buffer (its plane stride)
  const int* bdel = balance_on() ? B.bdel : nullptr;
  // rows [2m, Mp) of every X' slot are padding the residue kernel never writes
  if (Mp > 2 * m)
    e = cudaMemset2DAsync(resA + 2 * m * Kp, Mp * Kp, 0, (Mp - 2 * m) * Kp, (size_t)kQ * aslots, stream);
  CUtensorMap mapA, mapB;
  if (e == cudaSuccess && (!make_map(&mapA, resA, Kp, aslots * Mp, kQ, BM) ||
                           !make_map(&mapB, B.res, Kp, (uint64_t)B.nslots * 2 * Sp, kQ, use_pair() ? BN / 2 : BN)))
    e = cudaErrorInvalidValue;
  if (e == cudaSuccess && B.all && !B.ready && env_int("QTB_OZAKI_LAZYB", 1) == 0) {  // (experiment switch)
    if ((e = prep_b(B, B.bh1, B.bh2, (uint64_t)B.s0, (int)ps, 0, flag, stream)) == cudaSuccess) B.ready = true;
  }
  const bool lazyB = B.all && !B.ready;  // B' of each batch built beside the previous batch's GEMM
  // the balancing and column exponents of every slot first (a streaming read
  // of B̂ that would crawl beside the GEMM), the B' residues then batch by
  // batch; before the fork below, so the aux stream's batches see them
  if (e == cudaSuccess && lazyB) e = prep_b(B, B.bh1, B.bh2, (uint64_t)B.s0, (int)ps, 0, flag, stream, kPrepExp);
  // the second stream and the ordering events are per-thread, per-device
  // objects reused by every call (creating and destroying them per call cost
  // more than a mid-size product's batches); re-recording an event is safe:
  // a stream wait captures the event's state when it is enqueued
  int dev = 0;
  cudaGetDevice(&dev);
  AuxObjects& ao = aux_objects(dev);
  size_t nev = 0;
  auto mkev = [&]() {
    if (nev == ao.events.size()) {
      cudaEvent_t ev = nullptr;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return (cudaEvent_t) nullptr;
      ao.events.push_back(ev);
    }
    return ao.events[nev++];
  };
  cudaStream_t aux = stream;
  if (e == cudaSuccess && pipe && nbatch > 1 && ao.stream) {
    aux = ao.stream;
    cudaEvent_t fork = mkev();
    cudaEventRecord(fork, stream);
    cudaStreamWaitEvent(aux, fork, 0);
  }
  auto batch = [&](uint64_t i, uint64_t& f0, int& fcur) {
    f0 = B.s0 + i * F;
    fcur = (int)std::min<uint64_t>(F, B.s0 + ps - f0);
  };
  auto residues = [&](uint64_t i, cudaStream_t st) {
    uint64_t f0;
    int fcur;
    batch(i, f0, fcur);
    const uint64_t b = i % nbuf;
    ProfScope pr("k2_int8_residues", st);
    cudaMemsetAsync(amin + b * F, 0x7f, F * sizeof(int), st);
    oz_residue_a_kernel<<<dim3((unsigned)m, fcur), 256, 0, st>>>(
        ah1, ah2, resA + b * F * Mp * Kp, eA + b * F * Mp, xl1 + b * F * Mp, amin + b * F, bdel, flag, (int)m, (int)n,
        (int)p, (int)f0, (int)Mp, (int)aslots, B.cbase, share_end(p));
    pr.stop();
    count_launches(1);
    if (lazyB) {
      const cudaError_t eb = prep_b(B, B.bh1, B.bh2, f0, fcur, (int)(f0 - B.s0), flag, st, kPrepRes);
      if (eb != cudaSuccess && e == cudaSuccess) e = eb;
    }
  };
  auto crt = [&](uint64_t i, cudaStream_t st) {
    uint64_t f0;
    int fcur;
    batch(i, f0, fcur);
    const uint64_t b = i % nbuf;
    const int bslot0 = B.all ? (int)(f0 - B.s0) : 0;
    dim3 g = cgrid;
    g.z = (unsigned)fcur;
    ProfScope pc("k2_int8_crt", st);
    oz_crt_kernel<<<g, 256, 0, st>>>(ws + offR + b * bytesR, eA + b * F * Mp, xl1 + b * F * Mp, amin + b * F, B.eB,
                                     B.yl1, B.bmin, flag, gpart, ch1, ch2, (int)m, (int)n, (int)s, (int)p, (int)f0,
                                     bslot0, (int)Mp, (int)Sp, (int)F, ldc, cslice, B.cbase, share_end(p));
    const unsigned units = (unsigned)slot_units((int)f0, fcur, (int)p);
    oz_guard_sum_kernel<<<dim3(units, kGuardChunks), 256, 0, st>>>(gpart, (int)nper, flag, gsum, (int)p, (int)f0,
                                                                   fcur);
    oz_guard_kernel<<<units, kGuardChunks, 0, st>>>(gsum, flag, flag + 1, (int)p, (int)f0, fcur, guard_tol2(),
                                                    guard_force() ? 1 : 0);
    pc.stop();
    count_launches(3);
  };
  // batch 0's X' (and, lazily, its B' residues); without B.all its B' first
  if (e == cudaSuccess && !B.all) e = prep_b(B, bh1, bh2, B.s0, (int)std::min<uint64_t>(F, ps), 0, flag, stream);
  if (e == cudaSuccess) residues(0, stream);
  cudaEvent_t res_ready = nullptr, prev_gemm_done = nullptr;
  for (uint64_t i = 0; i < nbatch && e == cudaSuccess; ++i) {
    uint64_t f0;
    int fcur;
    batch(i, f0, fcur);
    const uint64_t b = i % nbuf;
    int bslot0 = (int)(f0 - B.s0);
    if (!B.all) {  // B' for this batch only (sequential schedule)
      bslot0 = 0;
      if (i > 0) {
        if ((e = prep_b(B, bh1, bh2, f0, fcur, 0, flag, stream)) != cudaSuccess) break;
        residues(i, stream);
      }
    }
    // X' of batch i (and, by stream order on aux, the CRT of batch i-2 that used R[b]) ready
    if (res_ready) cudaStreamWaitEvent(stream, res_ready, 0);
    ProfScope pg("k2_int8_gemm", stream);
    GemmParams gp{ws + offR + b * bytesR, kQ, (int)(Mp / BM), (int)Mp, (int)Sp, (int)(Kp / BK), (int)F, bslot0,
                  (int)(Sp / BNC), fcur, (int)(b * F), (int)f0, share_end(p)};
    if (use_pair()) {
      const uint64_t items = (uint64_t)fcur * kQ * (Mp / 256) * (Sp / BNC);
      const unsigned clusters = (unsigned)std::min<uint64_t>(items, (uint64_t)num_sms() / 2);
      // pipeline depth: fewer stages leave shared memory for the residue / CRT
      // CTAs of neighbouring batches that run beside the GEMM
      static const int stages = std::min(6, std::max(4, env_int("QTB_OZAKI_STAGES", 6)));
      if (stages == 4)
        oz_gemm2_kernel<4><<<2 * clusters, GEMM_THREADS, gemm2_smem(4), stream>>>(mapA, mapB, gp);
      else if (stages == 5)
        oz_gemm2_kernel<5><<<2 * clusters, GEMM_THREADS, gemm2_smem(5), stream>>>(mapA, mapB, gp);
      else
        oz_gemm2_kernel<6><<<2 * clusters, GEMM_THREADS, gemm2_smem(6), stream>>>(mapA, mapB, gp);
    } else {
      oz_gemm_kernel<<<dim3((unsigned)((Mp / BM) * (Sp / BNC)), fcur), GEMM_THREADS, GEMM_SMEM, stream>>>(mapA,
                                                                                                         mapB, gp);
    }
    pg.stop();
    count_launches(1);
    if (aux != stream) {
      cudaEvent_t gemm_done = mkev();
      cudaEventRecord(gemm_done, stream);
      // aux: X' residues of batch i+1 into the other buffer (free once GEMM i-1,
      // which precedes GEMM i on the main stream, is done), then the CRT of
      // batch i — which therefore also precedes residues(i+2) rewriting this
      // batch's row exponents / norms on the same stream
      if (i + 1 < nbatch) {
        if (prev_gemm_done) cudaStreamWaitEvent(aux, prev_gemm_done, 0);  // GEMM i-1 read this X' buffer
        residues(i + 1, aux);
      }
      res_ready = mkev();
      cudaEventRecord(res_ready, aux);
      cudaStreamWaitEvent(aux, gemm_done, 0);
      crt(i, aux);
      prev_gemm_done = gemm_done;
    } else {
      crt(i, stream);
      if (B.all && i + 1 < nbatch) residues(i + 1, stream);
    }
    e = cudaGetLastError();
  }
  if (aux != stream) {
    cudaEvent_t join = mkev();
    cudaEventRecord(join, aux);
    cudaStreamWaitEvent(stream, join, 0);
  }
  if (e == cudaSuccess && lazyB) B.ready = true;
  const cudaError_t fe = cudaFreeAsync(ws, stream);

  return e != cudaSuccess ? e : fe;
}

// B' storage: residues, column exponents, column norms (guard), balancing
cudaError_t alloc_b(OzakiB& B, cudaStream_t stream) {
  const uint64_t Sp = pad_cols(B.s);
  const size_t bytes = (size_t)oz::kQ * B.nslots * 2 * Sp * 4 * B.n;
  const size_t offE = bytes, offL = offE + (((size_t)B.nslots * Sp * sizeof(int) + 255) & ~size_t(255));
  const size_t offD = offL + (size_t)B.nslots * Sp * sizeof(double);
  const size_t offM = offD + B.p * B.n * sizeof(int);
  cudaError_t e = cudaMallocAsync(&B.res, offM + B.nslots * sizeof(int), stream);
  if (e != cudaSuccess) return e;
  B.eB = reinterpret_cast<int*>(B.res + offE);
  B.yl1 = reinterpret_cast<double*>(B.res + offL);
  B.bdel = reinterpret_cast<int*>(B.res + offD);
  B.bmin = reinterpret_cast<int*>(B.res + offM);
  return cudaSuccess;
}

}  // namespace

cudaError_t ozaki_prepare_b(const double2* bh1, const double2* bh2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                            uint64_t ldb, uint64_t bslice, int* flag, bool require_all, OzakiB* out,
                            cudaStream_t stream, bool lazy) {
  *out = OzakiB{};
  if (n % 32 != 0 || n > 8192 || p == 0) return cudaErrorInvalidValue;
  cudaError_t e = oz_init();
  if (e != cudaSuccess) return e;
  OzakiB B{};
  B.n = n;
  B.s = s;
  B.p = p;
  B.ldb = ldb;
  B.bslice = bslice;
  const uint64_t per_b = b_slot_bytes(n, s);
  // keep B' for every frequency when it fits (one residue pass over B̂, reused
  // by every A batch / row slab); otherwise B' is rebuilt per A batch
  B.s0 = 0;
  B.ns = (int)p;
  B.cbase = -1;
  B.all = require_all || per_b * p <= env_mb("QTB_OZAKI_B_MB", 24576);
  B.nslots = B.all ? (int)p : (int)batch_slots(p, a_slot_bytes(m, n, s) + per_b, env_mb("QTB_OZAKI_WS_MB", 3072));
  if ((uint64_t)B.nslots * 2 * pad_cols(s) > 0x7fffffffULL) return cudaErrorInvalidValue;
  if ((e = alloc_b(B, stream)) != cudaSuccess) return e;
  B.bh1 = bh1;
  B.bh2 = bh2;
  if (B.all && !lazy) e = prep_b(B, bh1, bh2, 0, (int)p, 0, flag, stream);
  B.ready = B.all && !lazy;
  if (e != cudaSuccess) {
    cudaFreeAsync(B.res, stream);
    return e;
  }
  *out = B;
  return cudaSuccess;
}

// Compact slot range: B̂ (ns, n, s) holds the frequency slots [s0, s0 + ns)
// in slot order (slice t = slot s0 + t), and so do the Â (ns, m, n) and Ĉ
// (ns, m, s) of every ozaki_multiply against the returned B'.  A pair occupies
// two adjacent slots (2j, 2j+1): neither end of the range may split one.  The
// frequency-parallel multi-GPU driver gives each rank such a range.
cudaError_t ozaki_prepare_b_slots(const double2* bh1, const double2* bh2, uint64_t n, uint64_t s, uint64_t p, int s0,
                                  int ns, int* flag, OzakiB* out, cudaStream_t stream) {
  *out = OzakiB{};
  // a boundary may not split a pair (an odd slot below 2 * npairs)
  const uint64_t pair_end = 2 * ((p - 1) / 2);
  auto splits = [&](uint64_t b) { return (b & 1) && b < pair_end; };
  if (n % 32 != 0 || n > 8192 || n == 0 || s == 0 || p == 0 || p > 65534 || s0 < 0 || ns <= 0 ||
      (uint64_t)s0 + ns > p || splits((uint64_t)s0) || splits((uint64_t)s0 + ns))
    return cudaErrorInvalidValue;
  cudaError_t e = oz_init();
  if (e != cudaSuccess) return e;
  OzakiB B{};
  B.n = n;
  B.s = s;
  B.p = p;
  B.ldb = s;
  B.bslice = n * s;
  B.s0 = s0;
  B.ns = ns;
  B.cbase = s0;
  B.all = true;
  B.nslots = ns;
  if ((uint64_t)ns * 2 * pad_cols(s) > 0x7fffffffULL) return cudaErrorInvalidValue;
  if ((e = alloc_b(B, stream)) != cudaSuccess) return e;
  B.bh1 = bh1;
  B.bh2 = bh2;
  if ((e = prep_b(B, bh1, bh2, (uint64_t)s0, ns, 0, flag, stream)) != cudaSuccess) {
    cudaFreeAsync(B.res, stream);
    return e;
  }
  B.ready = true;
  *out = B;
  return cudaSuccess;
}

cudaError_t ozaki_multiply(OzakiB& B, const double2* ah1, const double2* ah2, const double2* bh1, const double2* bh2,
                           uint64_t m, double2* ch1, double2* ch2, uint64_t ldc, uint64_t cslice, int* flag,
                           cudaStream_t stream) {
  if (m == 0 || B.s == 0) return cudaSuccess;
  return multiply(B, ah1, ah2, bh1, bh2, m, ch1, ch2, ldc, cslice, flag, stream);
}

cudaError_t ozaki_release(OzakiB& B, cudaStream_t stream) {
  cudaError_t e = B.res ? cudaFreeAsync(B.res, stream) : cudaSuccess;
  B = OzakiB{};
  return e;
}

cudaError_t launch_spectral_gemm_ozaki(const double2* ah1, const double2* ah2, const double2* bh1,
                                       const double2* bh2, double2* ch1, double2* ch2, uint64_t m, uint64_t n,
                                       uint64_t s, uint64_t p, uint64_t ldb, uint64_t ldc, uint64_t bslice,
                                       uint64_t cslice, int* flag, cudaStream_t stream) {
  if (m == 0 || s == 0 || p == 0) return cudaSuccess;
  OzakiB B;
  cudaError_t e = ozaki_prepare_b(bh1, bh2, m, n, s, p, ldb, bslice, flag, false, &B, stream, true);
  if (e != cudaSuccess) return e;
  e = ozaki_multiply(B, ah1, ah2, bh1, bh2, m, ch1, ch2, ldc, cslice, flag, stream);
  const cudaError_t fe = ozaki_release(B, stream);
  return e != cudaSuccess ? e : fe;
}

uint64_t int8_guard_fallbacks() {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, oz::g_guard_fallbacks, sizeof(v)) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return v;
}

}  // namespace qtb
