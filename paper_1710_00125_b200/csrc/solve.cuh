// Device solve / reconstruction entry points (solve.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rcp {

size_t solve_workspace_bytes(int64_t n, int64_t nrhs);
cudaError_t solve_device(int64_t n, const int64_t* perm, const double* L, const double* dd, const double* doff,
                         const int8_t* pattern, int64_t nrhs, const double* b, double* x, void* ws, int* singular,
                         cudaStream_t st, int num_sms);
cudaError_t reconstruct_device(int64_t n, const double* L, const double* dd, const double* doff,
                               const int8_t* pattern, double* out, double* scratch, cudaStream_t st);

}  // namespace rcp
