// The whole-pass executor k_pass (kernels.cuh, QCG_PASS_TU) in its own translation unit.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#define QCG_PASS_TU 1
#include "kernels.cuh"

namespace qcg {

// Launched like every engine kernel: programmatic stream serialization (it waits on
// k_advance with griddepcontrol.wait).
void launch_pass(const PassArgs& a, unsigned grid, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kMegaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_pass, a);
  if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch (k_pass): ") + cudaGetErrorString(e));
}

const void* pass_kernel() { return reinterpret_cast<const void*>(&k_pass); }

}  // namespace qcg
