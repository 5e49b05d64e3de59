// Phase timeline of the one-launch small-product kernel (csrc/qt_small.cu),
// config 1 (32^3, p = 16): %globaltimer stamps per CTA at kernel entry, after
// the cluster-barrier arrive, when the first tube's loads are back, before and
// after each cluster barrier and at exit; L2 flushed before every run (as
// bench.py does).  Build: see tools/microbench/README or the gpurun command in
// DESIGN.md (links the product library for its helpers).
#define QT_SMALL_TRACE 1
#include "../../paper_2212_14318_b200/csrc/qt_small.cu"

#include <algorithm>
#include <cstdio>
#include <vector>

int main() {
  using namespace qtb;
  const int m = 32, n = 32, s = 32, p = 16;
  const size_t an = (size_t)m * n * p, bn = (size_t)n * s * p, cn = (size_t)m * s * p;
  double2 *a1, *a2, *b1, *b2, *c1, *c2;
  cudaMalloc(&a1, an * 16); cudaMalloc(&a2, an * 16); cudaMalloc(&b1, bn * 16); cudaMalloc(&b2, bn * 16);
  cudaMalloc(&c1, cn * 16); cudaMalloc(&c2, cn * 16);
  cudaMemset(a1, 0, an * 16); cudaMemset(a2, 0, an * 16); cudaMemset(b1, 0, bn * 16); cudaMemset(b2, 0, bn * 16);
  float* flush = nullptr;
  cudaMalloc(&flush, 256u << 20);
  cudaStream_t st;
  cudaStreamCreate(&st);
  SmallArgs a;
  a.a1 = a1; a.a2 = a2; a.b1 = b1; a.b2 = b2; a.c1 = c1; a.c2 = c2;
  a.tw = twiddles_for(0, p, st);
  a.m = m; a.n = n; a.s = s; a.nt = 2; a.ncb = 4; a.isc = 1.0 / p;
  const unsigned ncl = 16;
  const int nblk = ncl * (p / 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[8] = {"entry", "arrive", "loads back", "K1 stores issued", "operands in (mb0)", "K2 done",
                          "C-hat in (mb1)", "exit"};
  std::vector<double> acc(8, 0.0), accmax(8, 0.0);
  double ev = 0;
  const int reps = 20;
  for (int r = 0; r < reps + 3; ++r) {
    cudaMemsetAsync(flush, r, 256u << 20, st);
    cudaEventRecord(e0, st);
    cudaError_t e = launch_p<16>(a, ncl, small_smem(n, p), st);
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<unsigned long long> t(nblk * 8);
    cudaMemcpyFromSymbol(t.data(), g_small_trace, t.size() * 8);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r < 3) continue;
    ev += ms * 1000.0;
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < nblk; ++b) t0 = std::min(t0, t[b * 8]);
    for (int k = 0; k < 8; ++k) {
      double mean = 0, mx = 0;
      for (int b = 0; b < nblk; ++b) {
        const double d = (double)(t[b * 8 + k] - t0) / 1000.0;
        mean += d / nblk;
        mx = std::max(mx, d);
      }
      acc[k] += mean / reps;
      accmax[k] += mx / reps;
    }
  }
  printf("event-timed kernel (after a 256 MB memset): %.2f us\n", ev / reps);
  for (int k = 0; k < 8; ++k) printf("%-18s mean %6.2f us  max %6.2f us (from the first CTA's entry)\n", names[k], acc[k], accmax[k]);
  return 0;
}
