// Launch-latency floor of dependent kernels on this GPU (measurement tool, not product code):
// a chain of N kernels, each reading its predecessor's output flag, run as (a) stream
// launches, (b) a captured graph, (c) a graph with programmatic dependent launch (PDL) edges,
// (d) PDL with an early trigger. Prints microseconds per kernel.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/launch_floor.cu -o build_var/launch_floor
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int MODE>  // 0: plain, 1: griddepcontrol.wait at start, 2: trigger at start then wait
__global__ void k_link(const double* in, double* out, int n) {
  if (MODE == 2) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (MODE >= 1) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] + 1.0;
}

struct Big { char pad[2304]; const double* in; double* out; int n; };
// the engine's gate/pair kernels take their descriptor (~2.3 KB) as a __grid_constant__ parameter
__global__ void k_big(const __grid_constant__ Big p) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  extern __shared__ double sm[];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p.n) p.out[i] = p.in[i] + 1.0 + (p.pad[i & 1023] ? sm[0] : 0.0);
}

// variants: big parameter block; dynamic shared memory alternating between two sizes
// (a different carve-out per launch); launches alternating between two captured streams
float run_var(int var, int N, int blocks, double* a, double* b, int n) {
  cudaStream_t s, s2;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<cudaEvent_t> evs(N);
  for (auto& ev : evs) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  Big p{};
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  if (var == 2) { CK(cudaEventRecord(evs[0], s)); CK(cudaStreamWaitEvent(s2, evs[0], 0)); }
  for (int i = 0; i < N; ++i) {
    p.in = (i & 1) ? b : a;
    p.out = (i & 1) ? a : b;
    p.n = n;
    cudaStream_t q = (var == 2 && (i & 1)) ? s2 : s;
    if (var == 2 && i > 0) CK(cudaStreamWaitEvent(q, evs[i - 1], 0));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = q;
    cfg.dynamicSmemBytes = var == 1 ? ((i & 1) ? 120 * 1024 : 1024) : (var == 3 ? 120 * 1024 : 0);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_big, p));
    if (var == 2) CK(cudaEventRecord(evs[i], q));
  }
  if (var == 2) CK(cudaStreamWaitEvent(s, evs[N - 1], 0));
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    CK(cudaEventRecord(e0, s));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (rep >= 2 && ms < best) best = ms;
  }
  return best * 1000.f / N;
}

template <int MODE>
void launch(cudaStream_t s, bool pdl, const double* in, double* out, int n, int blocks) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, k_link<MODE>, in, out, n));
}

template <int MODE>
float run(bool graph, bool pdl, int N, int blocks, double* a, double* b, int n) {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  auto chain = [&] {
    for (int i = 0; i < N; ++i) launch<MODE>(s, pdl, (i & 1) ? b : a, (i & 1) ? a : b, n, blocks);
  };
  if (graph) {
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    chain();
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
  }
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    CK(cudaEventRecord(e0, s));
    if (graph) CK(cudaGraphLaunch(ge, s));
    else chain();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (rep >= 2 && ms < best) best = ms;
  }
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return best * 1000.f / N;
}

int main() {
  const int N = 200;
  for (int blocks : {1, 148, 1184}) {
    const int n = blocks * 256;
    double *a, *b;
    CK(cudaMalloc(&a, n * sizeof(double)));
    CK(cudaMalloc(&b, n * sizeof(double)));
    CK(cudaMemset(a, 0, n * sizeof(double)));
    printf("blocks=%d  stream %.2f us  graph %.2f us  graph+pdl(wait) %.2f us  graph+pdl(early trigger) %.2f us  stream+pdl(wait) %.2f us\n",
           blocks, run<0>(false, false, N, blocks, a, b, n), run<0>(true, false, N, blocks, a, b, n),
           run<1>(true, true, N, blocks, a, b, n), run<2>(true, true, N, blocks, a, b, n),
           run<1>(false, true, N, blocks, a, b, n));
    printf("          graph+pdl, 2.3 KB parameter block %.2f us  + shared-memory size alternating 1 KB / 120 KB %.2f us  + all 120 KB %.2f us  + alternating between two streams (event edges) %.2f us\n",
           run_var(0, N, blocks, a, b, n), run_var(1, N, blocks, a, b, n), run_var(3, N, blocks, a, b, n), run_var(2, N, blocks, a, b, n));
    cudaFree(a);
    cudaFree(b);
  }
  return 0;
}
