// Launch-latency probe (sm_100a): what does a chain of dependent kernels cost
// after an L2 flush, with and without programmatic dependent launch (PDL), and
// from a CUDA graph?  Used to decide whether PDL pays for the small configs
// (1 and 3).  Each variant: flush (256 MB memset + read), then
// event -> chain -> event on one stream; median of 30 reps.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__);                   \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__global__ void empty_kernel(int pdl) {
  if (pdl) {
    pdl_trigger();
    pdl_wait();
  }
}

// copy n doubles2 (grid-stride), optionally PDL
__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n, int pdl) {
  if (pdl) {
    pdl_trigger();
    pdl_wait();
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = make_double2(in[i].x * 1.0000001, in[i].y);
}

__global__ void read_kernel(const float* __restrict__ in, size_t n, float* out) {
  float s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += in[i];
  if (s == 1234.5f) out[0] = s;
}

static cudaError_t launch(void (*k)(const double2*, double2*, size_t, int), int grid, int block, cudaStream_t st,
                          bool pdl, const double2* in, double2* out, size_t n) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, in, out, n, pdl ? 1 : 0);
}
static cudaError_t launch_empty(int grid, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, empty_kernel, pdl ? 1 : 0);
}

int main() {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  float* flush = nullptr;
  const size_t fl = 256ull << 20;
  CK(cudaMalloc(&flush, 2 * fl));
  float* sink = nullptr;
  CK(cudaMalloc(&sink, 64));
  const size_t small = 1 << 16;    // 1 MB of double2
  const size_t big = 4ull << 20;   // 64 MB of double2
  double2 *b0 = nullptr, *b1 = nullptr;
  CK(cudaMalloc(&b0, big * sizeof(double2)));
  CK(cudaMalloc(&b1, big * sizeof(double2)));
  CK(cudaMemset(b0, 0, big * sizeof(double2)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  auto do_flush = [&]() -> cudaError_t {
    cudaError_t e = cudaMemsetAsync(flush, 0, fl, st);
    if (e == cudaSuccess) read_kernel<<<148 * 8, 256, 0, st>>>(flush + fl / 4, fl / 4, sink);
    return e == cudaSuccess ? cudaGetLastError() : e;
  };

  struct Variant {
    const char* name;
    int nk;       // kernels in the chain
    int kind;     // 0 empty, 1 copy small, 2 copy big
    bool pdl;
    bool graph;
  };
  const Variant vs[] = {
      {"1 empty kernel", 1, 0, false, false},        {"3 empty kernels", 3, 0, false, false},
      {"3 empty kernels, PDL", 3, 0, true, false},   {"3 empty kernels, graph", 3, 0, false, true},
      {"3 empty kernels, graph+PDL", 3, 0, true, true},
      {"3 x copy 1 MB", 3, 1, false, false},         {"3 x copy 1 MB, PDL", 3, 1, true, false},
      {"3 x copy 1 MB, graph", 3, 1, false, true},   {"3 x copy 1 MB, graph+PDL", 3, 1, true, true},
      {"5 x copy 64 MB", 5, 2, false, false},        {"5 x copy 64 MB, PDL", 5, 2, true, false},    {"5 x copy 64 MB, graph", 5, 2, false, true},
      {"5 x copy 64 MB, graph+PDL", 5, 2, true, true},
  };
  for (const Variant& v : vs) {
    auto chain = [&]() -> cudaError_t {
      for (int k = 0; k < v.nk; ++k) {
        const bool pdl = v.pdl && k > 0;
        cudaError_t e;
        if (v.kind == 0) e = launch_empty(148, st, pdl);
        else if (v.kind == 1) e = launch(copy_kernel, 148, 256, st, pdl, (k & 1) ? b1 : b0, (k & 1) ? b0 : b1, small);
        else e = launch(copy_kernel, 148 * 8, 256, st, pdl, (k & 1) ? b1 : b0, (k & 1) ? b0 : b1, big);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    };
    cudaGraphExec_t ge = nullptr;
    if (v.graph) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      CK(chain());
      CK(cudaStreamEndCapture(st, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphDestroy(g));
    }
    std::vector<float> ts;
    for (int r = 0; r < 33; ++r) {
      CK(do_flush());
      CK(cudaEventRecord(e0, st));
      if (v.graph) CK(cudaGraphLaunch(ge, st));
      else CK(chain());
      CK(cudaEventRecord(e1, st));
      CK(cudaStreamSynchronize(st));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 3) ts.push_back(ms * 1000.f);
    }
    std::sort(ts.begin(), ts.end());
    printf("%-32s median %7.2f us  (min %7.2f, max %7.2f)\n", v.name, ts[ts.size() / 2], ts.front(), ts.back());
    if (ge) cudaGraphExecDestroy(ge);
  }
  return 0;
}
