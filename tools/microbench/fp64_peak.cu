// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync f64) and DFMA throughput.
// Used to fill the P64 roofline denominator (MEASURED_PEAKS.json has no fp64 figure).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + i * 1e-9;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - i * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double x[NACC];
  double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
  for (int i = 0; i < NACC; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, int iters, double flops_per_warp_iter, const char* name, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(d, iters);  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double warps = (double)blocks * threads / 32;
  double tf = warps * iters * flops_per_warp_iter / (best * 1e-3) / 1e12;
  printf("%-28s blocks=%5d threads=%4d  %8.3f ms  %7.2f TFLOP/s\n", name, blocks, threads, best, tf);
  return tf;
}

int main() {
  double* d; CK(cudaMalloc(&d, 64));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs=%d\n", sms);
  const int it = 4096;
  for (int tpb : {128, 256, 512}) {
    for (int mult : {1, 2, 4}) {
      run(dmma_m8n8k4<8>, sms * mult, tpb, it, 8 * 512.0, "dmma m8n8k4 x8acc", d);
    }
  }
  run(dmma_m8n8k4<4>, sms * 2, 256, it, 4 * 512.0, "dmma m8n8k4 x4acc", d);
  run(dmma_m8n8k4<16>, sms * 2, 256, it, 16 * 512.0, "dmma m8n8k4 x16acc", d);
  run(dmma_m16n8k16<4>, sms * 2, 256, it / 4, 4 * 2 * 16 * 8 * 16.0, "dmma m16n8k16 x4acc", d);
  run(dmma_m16n8k16<8>, sms * 2, 256, it / 4, 8 * 2 * 16 * 8 * 16.0, "dmma m16n8k16 x8acc", d);
  for (int tpb : {256, 512, 1024})
    run(dfma_loop<16>, sms * 2, tpb, it, 16 * 32 * 2.0, "dfma x16", d);
  run(dfma_loop<8>, sms * 4, 256, it, 8 * 32 * 2.0, "dfma x8", d);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clockRate attr = %d kHz\n", clk);
  // sustained: the best burst shape back to back for ~4 s (clocks settle under the power cap)
  {
    const int blocks = sms * 4, threads = 256, iters = 65536;
    const double fl = (double)blocks * threads / 32 * iters * 8 * 512.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    long launches = 0;
    auto t0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0);
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 4.0) {
      for (int k = 0; k < 4; ++k) dmma_m8n8k4<8><<<blocks, threads>>>(d, iters);
      launches += 4;
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s sustained launches=%ld  %8.1f ms  %7.2f TFLOP/s\n", "dmma m8n8k4 x8acc", launches, ms,
           fl * launches / (ms * 1e-3) / 1e12);
  }
  return 0;
}
