// int8 tensor-core peak probe for B200 (sm_100a): tcgen05.mma.cta_group::1.kind::i8
// (u8 x u8 -> s32, M = 128, N = 256, K = 32 per instruction) issued back to
// back by one thread per SM from shared-memory operands (no TMA, no epilogue),
// accumulating into TMEM.  Measures the roofline denominator of the exact
// int8 stage 2 (csrc/qt_ozaki.cu): burst (best of short runs, clocks free to
// boost) and sustained (back-to-back launches for ~4 s, under the power cap).
// Operands are pseudo-random bytes (zeros would under-state the power draw).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int8_peak int8_peak.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__);                 \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr int BM = 128, BN = 256, BK = 128;  // one 128-byte swizzle row of K per stage
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK;
constexpr size_t SMEM = A_BYTES + B_BYTES + 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {  // K-major, 128B swizzle, SBO 1024
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// s32 accumulator, u8 x u8, K-major A and B, N = 256, M = 128
constexpr uint32_t kIdesc = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__global__ void __launch_bounds__(128, 1) i8_mma_loop(int iters, unsigned* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < (A_BYTES + B_BYTES) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)(i + 1) * 2654435761u ^ (blockIdx.x * 40503u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    reinterpret_cast<uint32_t*>(smem)[i] = h ^ (h >> 15);
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy (MMA reads)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + A_BYTES);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < BK / 32; ++kk) {
        const uint32_t acc = (it | kk) != 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(desc_sw128(a0 + kk * 32)), "l"(desc_sw128(b0 + kk * 32)), "r"(kIdesc), "r"(acc)
            : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@P1 bra DONE;\n\tbra WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(&bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (v == 0x12345679u) sink[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

int main(int argc, char** argv) {
  const double sustain_s = argc > 1 ? atof(argv[1]) : 4.0;
  int sms = 148, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  CK(cudaFuncSetAttribute(i8_mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  unsigned* sink;
  CK(cudaMalloc(&sink, 64));
  const double ops_per_iter = 2.0 * BM * BN * 32 * (BK / 32);  // multiply-add = 2 ops
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("SMs=%d clockRate=%d kHz\n", sms, clk);
  // burst: short launches (~2 ms), best of 7
  for (int iters : {2048, 8192}) {
    i8_mma_loop<<<sms, 128, SMEM>>>(iters, sink);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 7; ++r) {
      cudaEventRecord(e0);
      i8_mma_loop<<<sms, 128, SMEM>>>(iters, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double tops = sms * (double)iters * ops_per_iter / (best * 1e-3) / 1e12;
    printf("burst     iters=%6d  %8.3f ms  %8.1f TOPS  (%.0f int8 ops/clk/SM at the rated clock)\n", iters, best, tops,
           tops * 1e12 / sms / (clk * 1e3));
  }
  // sustained: back-to-back launches for sustain_s seconds
  const int iters = 65536;
  double total_ms = 0.0;
  long launches = 0;
  auto t0 = std::chrono::steady_clock::now();
  cudaEventRecord(e0);
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < sustain_s) {
    for (int k = 0; k < 4; ++k) i8_mma_loop<<<sms, 128, SMEM>>>(iters, sink);
    launches += 4;
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  total_ms = ms;
  const double tops = sms * (double)iters * ops_per_iter * launches / (total_ms * 1e-3) / 1e12;
  printf("sustained launches=%ld  %8.1f ms  %8.1f TOPS\n", launches, total_ms, tops);
  return 0;
}
