// host_err.h -- error and launch bookkeeping of the C ABI (defined in
// mclahe_gpu.cu) for the other host translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

namespace mg {
int host_fail(int code, const std::string& msg);          // sets mclahe_last_error
int host_cuda_fail(cudaError_t e, const char* where);     // CUDA / OOM codes
void host_count_launch();                                 // mclahe_launch_count
}  // namespace mg

#define MGH_CUDA(call)                                          \
  do {                                                          \
    cudaError_t e_ = (call);                                    \
    if (e_ != cudaSuccess) return mg::host_cuda_fail(e_, #call); \
  } while (0)

#define MGH_LAUNCHED()                                            \
  do {                                                            \
    mg::host_count_launch();                                      \
    cudaError_t e_ = cudaGetLastError();                          \
    if (e_ != cudaSuccess) return mg::host_cuda_fail(e_, __func__); \
  } while (0)
