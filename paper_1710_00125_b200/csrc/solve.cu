// Solve x = P^T L^-T D^-1 L^-1 P b against the device factorization
// (reference _substitute / block_diag_solve, solve.py:34-76), and L D L^T
// reconstruction (factor.py:663-665).
//
// L is the row-major unit lower factor.  The triangular solves are blocked by
// NB = 64 rows: one launch per block, in which every CTA solves the 64x64
// diagonal block redundantly (bitwise identical in all CTAs) and then applies the
// block's rank-64 update to its own slice of the remaining right-hand side, so no
// cross-CTA reduction or atomics are needed and the result is deterministic.
#include <algorithm>
#include "gemm_dmma.cuh"
#include "solve.cuh"

namespace rcp {

namespace {

constexpr int NB = 64;
constexpr int kSolveThreads = 256;

__global__ void gather_rows_kernel(int64_t n, int64_t nrhs, const int64_t* __restrict__ perm,
                                   const double* __restrict__ b, double* __restrict__ y) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t src = perm[i];
  for (int64_t c = 0; c < nrhs; ++c) y[i + c * n] = b[src + c * n];
}

__global__ void scatter_rows_kernel(int64_t n, int64_t nrhs, const int64_t* __restrict__ perm,
                                    const double* __restrict__ v, double* __restrict__ x) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t dst = perm[i];
  for (int64_t c = 0; c < nrhs; ++c) x[dst + c * n] = v[i + c * n];
}

// Forward block: solve rows [i0, i1) of L z = y (unit diagonal), then
// y[r] -= L[r, i0:i1] . z[i0:i1] for this CTA's rows r >= i1.
__global__ void __launch_bounds__(kSolveThreads) fwd_block_kernel(int64_t n, int64_t nrhs, int64_t i0,
                                                                  const double* __restrict__ L,
                                                                  double* __restrict__ y, double* __restrict__ zo) {
  __shared__ double Ld[NB][NB + 1];
  __shared__ double z[NB];
  const int64_t i1 = (n < i0 + NB ? n : i0 + NB);
  const int nb = (int)(i1 - i0);
  for (int f = threadIdx.x; f < nb * nb; f += blockDim.x) {
    int a = f / nb, c = f - a * nb;
    Ld[a][c] = (c < a) ? L[(i0 + a) * n + (i0 + c)] : 0.0;
  }
  __syncthreads();
  const int64_t rows = n - i1;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t rb = i1 + (int64_t)blockIdx.x * per, re = (n < rb + per ? n : rb + per);
  for (int64_t col = 0; col < nrhs; ++col) {
    double* yc = y + col * n;
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      for (int a = 0; a < nb; ++a) {
        double part = 0.0;
        for (int c = lane; c < a; c += 32) part = __fma_rn(Ld[a][c], z[c], part);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, off));
        if (lane == 0) z[a] = __dsub_rn(yc[i0 + a], part);
        __syncwarp();
      }
    }
    __syncthreads();
    if (blockIdx.x == 0) {
      for (int a = threadIdx.x; a < nb; a += blockDim.x) zo[col * n + i0 + a] = z[a];
    }
    // rank-nb update of this CTA's rows: one warp per row, lanes over the block columns
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int64_t r = rb + warp; r < re; r += nw) {
      const double* lr = L + r * n + i0;
      double part = 0.0;
      for (int c = lane; c < nb; c += 32) part = __fma_rn(lr[c], z[c], part);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, off));
      if (lane == 0) yc[r] = __dsub_rn(yc[r], part);
    }
    __syncthreads();
  }
}

// Backward block: solve rows [i0, i1) of L^T v = w, then w[c] -= sum_{r in block} L[r, c] v[r]
// for this CTA's columns c < i0.
__global__ void __launch_bounds__(kSolveThreads) bwd_block_kernel(int64_t n, int64_t nrhs, int64_t i0,
                                                                  const double* __restrict__ L,
                                                                  double* __restrict__ w, double* __restrict__ vo) {
  __shared__ double Ld[NB][NB + 1];
  __shared__ double v[NB];
  const int64_t i1 = (n < i0 + NB ? n : i0 + NB);
  const int nb = (int)(i1 - i0);
  for (int f = threadIdx.x; f < nb * nb; f += blockDim.x) {
    int a = f / nb, c = f - a * nb;
    Ld[a][c] = (c < a) ? L[(i0 + a) * n + (i0 + c)] : 0.0;
  }
  __syncthreads();
  const int64_t cols = i0;
  const int64_t per = (cols + gridDim.x - 1) / gridDim.x;
  const int64_t cb = (int64_t)blockIdx.x * per, ce = (cols < cb + per ? cols : cb + per);
  for (int64_t col = 0; col < nrhs; ++col) {
    double* wc = w + col * n;
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      for (int a = nb - 1; a >= 0; --a) {
        double part = 0.0;
        for (int bq = a + 1 + lane; bq < nb; bq += 32) part = __fma_rn(Ld[bq][a], v[bq], part);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, off));
        if (lane == 0) v[a] = __dsub_rn(wc[i0 + a], part);
        __syncwarp();
      }
    }
    __syncthreads();
    if (blockIdx.x == 0) {
      for (int a = threadIdx.x; a < nb; a += blockDim.x) vo[col * n + i0 + a] = v[a];
    }
    for (int64_t c = cb + threadIdx.x; c < ce; c += blockDim.x) {
      double part = 0.0;
      for (int a = 0; a < nb; ++a) part = __fma_rn(L[(i0 + a) * n + c], v[a], part);
      wc[c] = __dsub_rn(wc[c], part);
    }
    __syncthreads();
  }
}

// D w = z blockwise (solve.py:34-66): exact-zero blocks give zeros and set *singular.
__global__ void block_diag_kernel(int64_t n, int64_t nrhs, const double* __restrict__ dd,
                                  const double* __restrict__ doff, const int8_t* __restrict__ pattern,
                                  double* __restrict__ z, int* singular) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int8_t pt = pattern[i];
  if (pt == 2) return;  // second index of a 2x2 block, handled by its first index
  for (int64_t c = 0; c < nrhs; ++c) {
    double* zc = z + c * n;
    if (pt == 1 && i + 1 < n) {
      double d11 = dd[i], d21 = doff[i], d22 = dd[i + 1];
      double det = __dsub_rn(__dmul_rn(d11, d22), __dmul_rn(d21, d21));
      if (det == 0.0) {
        atomicOr(singular, 1);
        zc[i] = 0.0;
        zc[i + 1] = 0.0;
      } else {
        double z1 = zc[i], z2 = zc[i + 1];
        zc[i] = __ddiv_rn(__dsub_rn(__dmul_rn(d22, z1), __dmul_rn(d21, z2)), det);
        zc[i + 1] = __ddiv_rn(__dsub_rn(__dmul_rn(d11, z2), __dmul_rn(d21, z1)), det);
      }
    } else {
      double dv = dd[i];
      if (dv == 0.0) {
        atomicOr(singular, 1);
        zc[i] = 0.0;
      } else {
        zc[i] = __ddiv_rn(zc[i], dv);
      }
    }
  }
}

// LD = L * D (row-major), used by the reconstruction GEMM.
__global__ void scale_ld_kernel(int64_t n, const double* __restrict__ L, const double* __restrict__ dd,
                                const double* __restrict__ doff, const int8_t* __restrict__ pattern,
                                double* __restrict__ LD) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * n) return;
  int64_t i = idx / n, j = idx - i * n;
  const double* lr = L + i * n;
  double v;
  int8_t pj = pattern[j];
  if (pj == 1 && j + 1 < n) {
    v = lr[j] * dd[j] + lr[j + 1] * doff[j];
  } else if (pj == 2 && j > 0) {
    v = lr[j - 1] * doff[j - 1] + lr[j] * dd[j];
  } else {
    v = lr[j] * dd[j];
  }
  LD[idx] = v;
}

struct ReconEpi {
  static constexpr bool kHasInput = false;
  static constexpr bool kMirror = false;
  template <class Map>
  RCP_D bool prepare(Map&, int64_t&, OperandDesc&) { return true; }
  RCP_D double* cout_mirror(int64_t, int64_t) const { return nullptr; }
  double* out;
  int64_t n;
  RCP_D int map_row(int64_t) const { return 0; }
  RCP_D int map_col(int64_t) const { return 0; }
  RCP_D const double* dummy() const { return out; }
  RCP_D const double* cin(int64_t, int64_t, int, int) const { return nullptr; }
  // tile element (i, j) of L D L^T, stored row-major
  RCP_D double* cout(int64_t i, int64_t j) const { return (i < n && j < n) ? out + i * n + j : nullptr; }
};

}  // namespace

size_t solve_workspace_bytes(int64_t n, int64_t nrhs) { return 2 * (sizeof(double) * (size_t)n * (size_t)nrhs + 256); }

cudaError_t solve_device(int64_t n, const int64_t* perm, const double* L, const double* dd, const double* doff,
                         const int8_t* pattern, int64_t nrhs, const double* b, double* x, void* ws, int* singular,
                         cudaStream_t st, int num_sms) {
  double* y = reinterpret_cast<double*>(ws);
  double* z = y + (((size_t)n * nrhs + 31) / 32) * 32;
  const unsigned g1 = (unsigned)((n + 255) / 256);
  gather_rows_kernel<<<g1, 256, 0, st>>>(n, nrhs, perm, b, y);
  for (int64_t i0 = 0; i0 < n; i0 += NB) {
    int64_t rows = n - (n < i0 + NB ? n : i0 + NB);
    unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(num_sms * 2, (rows + 63) / 64));
    fwd_block_kernel<<<grid, kSolveThreads, 0, st>>>(n, nrhs, i0, L, y, z);
  }
  block_diag_kernel<<<g1, 256, 0, st>>>(n, nrhs, dd, doff, pattern, z, singular);
  const int64_t last = ((n - 1) / NB) * NB;
  for (int64_t i0 = last; i0 >= 0; i0 -= NB) {
    unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(num_sms * 2, (i0 + 255) / 256));
    bwd_block_kernel<<<grid, kSolveThreads, 0, st>>>(n, nrhs, i0, L, z, y);
  }
  scatter_rows_kernel<<<g1, 256, 0, st>>>(n, nrhs, perm, y, x);
  return cudaGetLastError();
}

cudaError_t reconstruct_device(int64_t n, const double* L, const double* dd, const double* doff,
                               const int8_t* pattern, double* out, double* scratch, cudaStream_t st) {
  const int64_t nn = n * n;
  scale_ld_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(n, L, dd, doff, pattern, scratch);
  const int64_t tm = (n + 63) / 64, tn = (n + 127) / 128;
  OperandDesc a{scratch, n, n, n};
  OperandDesc b{L, n, n, n};
  ReconEpi epi{out, n};
  RectMap map{tn, 64, 128};
  size_t smem = gemm_smem_bytes<64, 128, 3>();
  cudaError_t e = cudaFuncSetAttribute(dmma_gemm_kernel<64, 128, 3, 1, RectMap, ReconEpi>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dmma_gemm_kernel<64, 128, 3, 1, RectMap, ReconEpi><<<(unsigned)(tm * tn), kGemmThreads, smem, st>>>(a, b, n, map, epi);
  return cudaGetLastError();
}

}  // namespace rcp
