// qt_small.cu — the whole T-product in ONE launch for small products
// (tprod_fast, /root/reference/proj/src/tproduct.cpp:75-111; e.g. config 1,
// 32 x 32 x 32, p = 16): thread-block clusters exchanging through DSMEM.
//
// A small product is latency-bound: K1, K2 and K3 are three short kernels
// whose launch gaps and cold-cache round trips cost more than their work
// (DESIGN.md §7).  Here a cluster of Q = p/2 CTAs owns an 8 x 8 block of C
// and does all three stages without touching global memory in between:
//   1. forward tube FFTs (K1) of the block's A rows and B columns, spread
//      over the cluster's CTAs, one tube per thread in registers; every output
//      frequency is st.async'ed straight into the shared memory of the CTA
//      that owns that frequency, its bytes counted on that CTA's mbarrier;
//   2. each CTA waits for its own operand bytes only, runs the
//      paired-frequency product (K2) of its two frequency slices — a pair
//      (k, p - k), or the two self-paired frequencies 0 and p/2 — on the FP64
//      tensor pipe (DMMA m8n8k4) and st.async's each Ĉ value into the CTA that
//      inverts that tube (again counted on an mbarrier: a CTA leaves only
//      after every byte addressed to it has landed, and what it sends comes
//      from registers, so no CTA's shared memory is written after it exits);
//   3. inverse tube FFTs (K3) and the only global stores.
// One cluster barrier, at entry (every CTA running, its mbarriers
// initialised and its operands zeroed), split around the first tube loads.
// Every tube is transformed with the same butterflies and twiddles as
// qt_fft.cu, and every Ĉ element gets the same DMMA sequence (Gauss 3M, K-steps
// of 4 in order, zero padding to 16) as qt_gemm.cu's small tiles, so the
// result is bitwise the three-launch result (tests/test_gpu_small.py).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "qt_dmma_tile.cuh"
#include "qt_fft_reg.cuh"
#include "qt_internal.cuh"

namespace cg = cooperative_groups;

namespace qtb {
namespace {

constexpr int kRows = 8;       // C rows per cluster: one DMMA 8-row block
constexpr int kCols = 8;       // C columns per cluster: one 8-column DMMA block
constexpr int kThreads = 128;  // 4 warps: (side of the pair, C1 / C2 accumulators)
constexpr int kBK = 16;        // K tile of the operand layout (qt_gemm.cu SmallGaussCfg)
constexpr int kAPlane = kRows * kBK;              // 128 double2
constexpr int kBPlane = kBK * kCols;              // 128 double2
constexpr int kSlotTile = 2 * kAPlane + 2 * kBPlane;  // A1, A2, B1, B2 of one K tile of one frequency
constexpr int kCTubes = 2 * kRows * kCols;        // C tubes of a cluster (both CD planes)
constexpr int kMaxN = 64;

// phase timestamps for tools/microbench/small_trace.cu (compiled out here)
#ifdef QT_SMALL_TRACE
__device__ unsigned long long g_small_trace[4096 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SMALL_TRACE(k) \
  if (threadIdx.x == 0) g_small_trace[blockIdx.x * 8 + (k)] = gtimer()
#else
#define SMALL_TRACE(k)
#endif

// swizzled operand positions (the layouts of qt_dmma_tile.cuh's small tiles)
__device__ __forceinline__ int a_pos(int i, int c) { return i * kBK + (c ^ ((i & 1) << 2)); }
__device__ __forceinline__ int b_pos(int k, int j) { return k * kCols + (j ^ ((k & 3) << 1)); }

struct SmallArgs {
  const double2* a1;
  const double2* a2;
  const double2* b1;
  const double2* b2;
  double2* c1;
  double2* c2;
  const double2* tw;  // W_p table (twiddles_for)
  int m, n, s, nt, ncb;
  double isc;  // 1/p (the inverse jobs' scale, as qt_api.cu add_inverse computes it)
};

// y = F(x) for one tube in registers, as qt_fft.cu does it for single-pass p:
// p in {2, 4, 8} one radix-p stage; p = 16 the two-stage (8, 2) Stockham
// kernel (tube_fft2_kernel<8, 2>) with its stage-1 twiddles W_16^j.
template <int P>
__device__ __forceinline__ void tube_dft(double2 (&x)[P], const double2 (&tw)[8]) {
  if constexpr (P == 16) {
    double2 y[16];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double2 v[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = x[j + 2 * r];
      dft_reg<8>(v);
#pragma unroll
      for (int k = 0; k < 8; ++k) y[j * 8 + k] = v[k];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double2 v[2] = {y[j], y[j + 8]};
      if (j != 0) v[1] = cmul(v[1], tw[j]);
      dft_reg<2>(v);
      x[j] = v[0];
      x[j + 8] = v[1];
    }
  } else {
    dft_reg<P>(x);
  }
}

// split cluster barrier (not .aligned: threads of a warp may reach the wait
// at different points of the K1 loop); each thread arrives and waits once
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() { asm volatile("barrier.cluster.wait.acquire;" ::: "memory"); }

// mbarrier + st.async plumbing: a remote store lands in the destination CTA's
// shared memory and counts its bytes on that CTA's mbarrier, which the
// destination waits on — no cluster-wide barrier per exchange
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
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
// shared::cta address -> the same offset in cluster CTA `cta` (shared::cluster)
__device__ __forceinline__ uint32_t map_cta(uint32_t saddr, int cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(cta));
  return r;
}
__device__ __forceinline__ void st_async_f64x2(uint32_t dst, double x, double y, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
               "d"(x), "d"(y), "r"(mbar)
               : "memory");
}

// frequency f -> (CTA of the cluster that owns it, its slot there)
template <int P>
__device__ __forceinline__ void freq_owner(int f, int& cta, int& slot) {
  constexpr int Q = P / 2;
  if (f == 0 || 2 * f == P) {
    cta = Q - 1;
    slot = f == 0 ? 0 : 1;
  } else {
    cta = (f < P - f ? f : P - f) - 1;
    slot = 2 * f < P ? 0 : 1;
  }
}

template <int P>
__global__ void __launch_bounds__(kThreads, 1) small_tprod_kernel(SmallArgs A) {
  constexpr int Q = P / 2;               // CTAs per cluster, two frequencies each
  constexpr int TPC = kCTubes / Q;       // inverse tubes per CTA
  extern __shared__ double2 sm[];
  __shared__ __align__(8) uint64_t mb[2];  // [0]: K1 operands in, [1]: Ĉ tubes in
  const int rank = (int)cg::this_cluster().block_rank();
  const int cl = blockIdx.x / Q;
  const int row0 = (cl / A.ncb) * kRows, col0 = (cl % A.ncb) * kCols;
  const int m = A.m, n = A.n, s = A.s, nt = A.nt;
  const int vr = min(kRows, m - row0), vc = min(kCols, s - col0);  // valid rows / columns of the block
  const int tid = threadIdx.x;
  double2* ops = sm;                         // [2 slots][nt K tiles][kSlotTile]
  double2* rcv = sm + 2 * nt * kSlotTile;    // [TPC tubes][P frequencies]
  SMALL_TRACE(0);

  if (tid == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // padding (K beyond n, rows beyond m, columns beyond s) is +0, as the
  // zero-filled cp.async loads of the three-launch path.  The extent comes
  // from %dynamic_smem_size, not from the (cold) kernel parameters, so the
  // barrier arrive below does not wait for them.
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    for (uint32_t i = tid; i < dyn / 16; i += kThreads) sm[i] = make_double2(0.0, 0.0);
  }
  // every CTA of the cluster running, its barriers initialised and its
  // operands zeroed before any remote store: the cluster barrier's arrive is
  // here, its wait after this thread's loads and FFT
  cluster_arrive_release();
  SMALL_TRACE(1);
  if (tid == 0) {
    // bytes this CTA receives: both frequency slots of every valid A and B
    // tube of the block; every frequency of its valid inverse tubes
    int tubes = 0;
    for (int u = 0; u < TPC; ++u) {
      const int r = (rank * TPC + u) % (kRows * kCols);
      tubes += (r / kCols < vr && r % kCols < vc) ? 1 : 0;
    }
    mbar_expect_tx(&mb[0], (uint32_t)(2 * (2 * vr * n + 2 * n * vc) * 16));
    mbar_expect_tx(&mb[1], (uint32_t)(tubes * P * 16));
  }
  // stage-1 twiddles W_16^j, j < 8 (p = 16), in registers
  double2 tw[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) tw[j] = P == 16 ? __ldg(&A.tw[j]) : make_double2(0.0, 0.0);

  // ---- K1: forward transforms of the block's A rows and B columns, each
  // frequency stored into its owner CTA with st.async (completes on the
  // owner's mb[0])
  {
    bool waited = false;
    const int na = 2 * kRows * n, nall = na + 2 * n * kCols;
    const uint32_t ops_s = smem_u32(ops), mb0_s = smem_u32(&mb[0]);
    for (int u = rank * kThreads + tid; u < nall; u += Q * kThreads) {
      const bool isA = u < na;
      int pl, i, l, j;
      const double2* src;
      size_t base, stride;
      if (isA) {
        pl = u / (kRows * n);
        const int r = u - pl * kRows * n;
        i = r / n;
        l = r - i * n;
        j = 0;
        if (i >= vr) continue;
        src = pl ? A.a2 : A.a1;
        base = (size_t)(row0 + i) * n + l;
        stride = (size_t)m * n;
      } else {
        const int v = u - na;
        pl = v / (n * kCols);
        const int r = v - pl * n * kCols;
        l = r / kCols;
        j = r - l * kCols;
        i = 0;
        if (j >= vc) continue;
        src = pl ? A.b2 : A.b1;
        base = (size_t)l * s + col0 + j;
        stride = (size_t)n * s;
      }
      // qfft3_conj jobs: plane 1 ConjInForward (+1), plane 2 NegateForward (-1)
      double2 x[P];
#pragma unroll
      for (int r = 0; r < P; ++r) {
        x[r] = __ldg(src + base + r * stride);
        if (pl == 0) x[r].y = -x[r].y;
      }
      SMALL_TRACE(2);
      tube_dft<P>(x, tw);
      if (!waited) {
        cluster_wait_acquire();
        waited = true;
      }
      const double sc = pl == 0 ? 1.0 : -1.0;
      const int tile = l / kBK, kk = l - tile * kBK;
      const int off = isA ? pl * kAPlane + a_pos(i, kk) : 2 * kAPlane + pl * kBPlane + b_pos(kk, j);
#pragma unroll
      for (int f = 0; f < P; ++f) {
        int cta, slot;
        freq_owner<P>(f, cta, slot);
        const uint32_t dst = ops_s + (uint32_t)(((slot * nt + tile) * kSlotTile + off) * 16);
        st_async_f64x2(map_cta(dst, cta), x[f].x * sc, x[f].y * sc, map_cta(mb0_s, cta));
      }
    }
    if (!waited) cluster_wait_acquire();
  }
  SMALL_TRACE(3);
  mbar_wait(&mb[0], 0);  // this CTA's two frequency slices are complete
  SMALL_TRACE(4);

  // ---- K2: this CTA's two frequency slices.  Warp (side sd, half hf)
  // computes output hf (0: C1, 1: C2) at slot sd for the block's 8 rows x 8
  // columns.  A pair CTA holds (k, p - k): side 0 is frequency k with mirror
  // slot 1, side 1 is p - k with mirror slot 0; the self CTA holds 0 and p/2,
  // each its own mirror.  The DMMA sequence of every accumulator is
  // qt_gemm.cu's mma_stage_3m (side 0 = its sets 0-5, side 1 = sets 6-11, the
  // same formulas with k and p - k swapped; C1 = sets 0-2, C2 = sets 3-5).
  {
    const int warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3;
    const int sd = warp & 1, hf = warp >> 1;
    const bool self = rank == Q - 1;
    const int ms = self ? sd : 1 - sd;
    const int f = self ? (sd ? P / 2 : 0) : (sd ? P - rank - 1 : rank + 1);
    double S[3][2];
#pragma unroll
    for (int c = 0; c < 3; ++c) S[c][0] = S[c][1] = 0.0;
    const int ia0 = g * kBK;
    const int jb = g;
    for (int t = 0; t < nt; ++t) {
      const double2* T1 = ops + (sd * nt + t) * kSlotTile;  // A1, A2, B1, B2 of slot sd
      const double2* TM = ops + (ms * nt + t) * kSlotTile;  // A1, A2 of the mirror slot
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        const int kk = ks * 4 + q;
        const int ia = ia0 + (kk ^ ((g & 1) << 2));
        const int ib = kk * kCols + (jb ^ (q << 1));
        const double2 vb1 = T1[2 * kAPlane + ib], vb2 = T1[2 * kAPlane + kBPlane + ib];
        const double b1p = vb1.x + vb1.y, b2p = vb2.x + vb2.y;
        if (hf == 0) {  // C1 = A1 B1 - conj(A2m) B2: sets 0-2
          const double2 va1 = T1[ia], vm2 = TM[kAPlane + ia];
          const double a1p = va1.x + va1.y, m2m = vm2.x - vm2.y;
          dmma(S[0], va1.x, vb1.x);
          dmma(S[1], va1.y, vb1.y);
          dmma(S[2], a1p, b1p);
          dmma(S[0], vm2.x, dneg(vb2.x));
          dmma(S[1], vm2.y, vb2.y);
          dmma(S[2], m2m, dneg(b2p));
        } else {  // C2 = conj(A1m) B2 + A2 B1: sets 3-5
          const double2 va2 = T1[kAPlane + ia], vm1 = TM[ia];
          const double a2p = va2.x + va2.y, m1m = vm1.x - vm1.y;
          dmma(S[0], vm1.x, vb2.x);
          dmma(S[1], vm1.y, dneg(vb2.y));
          dmma(S[2], m1m, b2p);
          dmma(S[0], va2.x, vb1.x);
          dmma(S[1], va2.y, vb1.y);
          dmma(S[2], a2p, b1p);
        }
      }
    }
    if (g < vr) {
      const uint32_t rcv_s = smem_u32(rcv), mb1_s = smem_u32(&mb[1]);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jl = 2 * q + e;
        if (jl >= vc) continue;
        const double t1 = S[0][e], t2 = S[1][e], t3 = S[2][e];
        const int tau = (hf * kRows + g) * kCols + jl;
        const int own = tau / TPC;
        st_async_f64x2(map_cta(rcv_s + (uint32_t)((((tau % TPC) * P) + f) * 16), own), t1 - t2, t3 - t1 - t2,
                       map_cta(mb1_s, own));
      }
    }
  }
  SMALL_TRACE(5);
  mbar_wait(&mb[1], 0);  // every frequency of this CTA's inverse tubes is in
  SMALL_TRACE(6);

  // ---- K3: inverse transforms of this CTA's C tubes, straight to HBM
  for (int u = tid; u < TPC; u += kThreads) {
    const int tau = rank * TPC + u;
    const int pl = tau / (kRows * kCols);
    const int r = tau - pl * kRows * kCols;
    const int i = r / kCols, j = r - (r / kCols) * kCols;
    if (i >= vr || j >= vc) continue;
    // qifft3_conj jobs: InverseConjOut (conj in, +1/p), NegateInverse (conj in and out, -1/p)
    double2 x[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      x[k] = rcv[u * P + k];
      x[k].y = -x[k].y;
    }
    tube_dft<P>(x, tw);
    const double sc = pl == 0 ? A.isc : -A.isc;
    const double sci = pl == 0 ? sc : -sc;
    double2* dst = (pl ? A.c2 : A.c1) + (size_t)(row0 + i) * s + col0 + j;
    const size_t stride = (size_t)m * s;
#pragma unroll
    for (int k = 0; k < P; ++k) dst[k * stride] = make_double2(x[k].x * sc, x[k].y * sci);
  }
  SMALL_TRACE(7);
}

size_t small_smem(uint64_t n, uint64_t p) {
  const uint64_t nt = (n + kBK - 1) / kBK;
  return (2 * nt * kSlotTile + (uint64_t)kCTubes * 2) * sizeof(double2);  // TPC * P = 2 * kCTubes for every P
}

template <int P>
cudaError_t launch_p(const SmallArgs& a, unsigned nclusters, size_t smem, cudaStream_t st) {
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t e = once_per_device(mu, done, [] {
    return cudaFuncSetAttribute(small_tprod_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)small_smem(kMaxN, P));
  });
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * (P / 2));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P / 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, small_tprod_kernel<P>, a);
}

}  // namespace

// Shapes the one-launch kernel takes: p in {2, 4, 8, 16} (two frequencies per
// CTA, clusters of 1-8), the small DMMA tiles' region of the three-launch path
// (m, s <= 32, qt_gemm.cu) and n <= 64 (operands of both slots in shared
// memory), fp64 DMMA stage 2 with Gauss 3M and slice_reflect.  $QTB_SMALL=0
// turns it off (the three-launch path then runs; bitwise the same result).
bool small_fused_eligible(uint64_t m, uint64_t n, uint64_t s, uint64_t p) {
  static const bool on = [] {
    const char* v = getenv("QTB_SMALL");
    return !(v && *v == '0');
  }();
  if (!on || m == 0 || n == 0 || s == 0) return false;
  if (!(p == 2 || p == 4 || p == 8 || p == 16)) return false;
  if (m > 32 || s > 32 || n > (uint64_t)kMaxN) return false;
  return choose_gemm_algo(n, s, p) == kAlgoDmma && dmma_gauss() && !debug_noreflect();
}

cudaError_t launch_small_tprod(const double2* a1, const double2* a2, const double2* b1, const double2* b2,
                               double2* c1, double2* c2, uint64_t m, uint64_t n, uint64_t s, uint64_t p,
                               cudaStream_t stream, int device) {
  SmallArgs a;
  a.a1 = a1;
  a.a2 = a2;
  a.b1 = b1;
  a.b2 = b2;
  a.c1 = c1;
  a.c2 = c2;
  a.tw = twiddles_for(device, (int)p, stream);
  if (!a.tw) return cudaErrorMemoryAllocation;
  a.m = (int)m;
  a.n = (int)n;
  a.s = (int)s;
  a.nt = (int)((n + kBK - 1) / kBK);
  a.ncb = (int)((s + kCols - 1) / kCols);
  a.isc = 1.0 / (double)p;
  const unsigned nclusters = (unsigned)(((m + kRows - 1) / kRows) * a.ncb);
  const size_t smem = small_smem(n, p);
  ProfScope ps("small_fused", stream);
  cudaError_t e;
  if (p == 2) e = launch_p<2>(a, nclusters, smem, stream);
  else if (p == 4) e = launch_p<4>(a, nclusters, smem, stream);
  else if (p == 8) e = launch_p<8>(a, nclusters, smem, stream);
  else e = launch_p<16>(a, nclusters, smem, stream);
  ps.stop();
  count_launches(1);
  return e;
}

}  // namespace qtb
