// Experiment diagnostics of the reference engine (not on the production path):
//   track_growth="full": a snapshot (max|S|, largest column norm of S) of every active Schur
//                        complement S = A[k:, k:] at the start of each step (factor.py:493-495,
//                        605-606; metrics.py:76-90 norm_1_inf / norm_1_2)
//   audit_sketch:        the sketch drift ||B[:, k:] - Omega[:, k:] S||_{1,2} after every panel
//                        (factor.py:497-504, 566-567), Omega kept in ORIGINAL column order and
//                        read through the current permutation (the reference swaps its columns,
//                        factor.py:346-347; a guard recompute overwrites Omega[:, k:], 402-403).
// Both force width-1 panels in the reference (factor.py:294-296); the host passes b = q = 1.
// The kernels read the panel outcome from the device-driven descriptor chain (panel.cuh), so
// they run inside the chain without host round trips; results are reduced with atomicMax on
// the bit patterns of non-negative doubles.
#include "misc.cuh"
#include "panel.cuh"
#include "rcp_common.cuh"

namespace rcp {

namespace {

constexpr int kDiagThreads = 256;

__device__ double block_reduce_max(double v, double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  __syncthreads();
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  double r = sm[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, sm[w]);
  return r;
}

__device__ double block_reduce_sum(double v, double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += sm[w];
  return r;
}

// One block per column j of the active block S = A[k0:, k0:] (column-major, ld n, both
// triangles valid): out[0] = max |S|, out[1] = max over columns of the scaled Euclidean norm
// (core.py:122-142).  k0 from the descriptor of the panel about to run (skipped unless it runs).
__global__ void snapshot_kernel(int64_t n, const double* __restrict__ A, const PanelDesc* __restrict__ d,
                                double* __restrict__ out) {
  __shared__ double sm[32];
  if (!d->run) return;
  const int64_t k0 = d->k0;
  const int64_t j = k0 + blockIdx.x;
  if (j >= n) return;
  const double* col = A + j * n;
  double mx = 0.0;
  for (int64_t i = k0 + threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, fabs(col[i]));
  mx = block_reduce_max(mx, sm);
  double ss = 0.0;
  if (mx > 0.0)
    for (int64_t i = k0 + threadIdx.x; i < n; i += blockDim.x) {
      const double x = fabs(col[i]) / mx;
      ss = __fma_rn(x, x, ss);
    }
  ss = block_reduce_sum(ss, sm);
  if (threadIdx.x == 0) {
    atomic_max_nonneg(out, mx);
    atomic_max_nonneg(out + 1, mx > 0.0 ? mx * sqrt(ss) : 0.0);
  }
}

// Drift after a committed panel with k = k_end < n: column j of E = B[:, k:] - Omega_cur S,
// Omega_cur[p, i] = omega_orig[p, perm[i]] (perm: original index per position, new order).
// One block per column; P accumulators in chunks of 8; the scaled norm of E[:, j] by thread 0.
__global__ void drift_kernel(int64_t n, int P, const double* __restrict__ A, const double* __restrict__ B,
                             const double* __restrict__ omega_orig, const int* __restrict__ perm,
                             const PanelDesc* __restrict__ d, double* __restrict__ out) {
  extern __shared__ double e[];  // P entries of E[:, j]
  __shared__ double sm[32];
  if (!d->ok) return;
  const int64_t k = d->k_end;
  if (k >= n) return;
  const int64_t j = k + blockIdx.x;
  if (j >= n) return;
  const double* col = A + j * n;
  for (int p0 = 0; p0 < P; p0 += 8) {
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) {
      const double a = col[i];
      const int64_t o = perm[i];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (p0 + q < P) acc[q] = __fma_rn(omega_orig[(int64_t)(p0 + q) * n + o], a, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double s = block_reduce_sum(acc[q], sm);
      if (threadIdx.x == 0 && p0 + q < P) e[p0 + q] = B[j * P + p0 + q] - s;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int p = 0; p < P; ++p) mx = fmax(mx, fabs(e[p]));
    double ss = 0.0;
    if (mx > 0.0)
      for (int p = 0; p < P; ++p) {
        const double x = fabs(e[p]) / mx;
        ss = __fma_rn(x, x, ss);
      }
    atomic_max_nonneg(out, mx > 0.0 ? mx * sqrt(ss) : 0.0);
  }
}

// Guard recompute at k0 (factor.py:400-403): omega_orig[:, perm[k0 + j]] = Omega'[:, j].
__global__ void omega_scatter_kernel(int64_t n, int P, int64_t k0, const double* __restrict__ om, int64_t m,
                                     const int* __restrict__ perm, double* __restrict__ omega_orig) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int64_t o = perm[k0 + j];
  for (int p = 0; p < P; ++p) omega_orig[(int64_t)p * n + o] = om[(int64_t)p * m + j];
}

}  // namespace

cudaError_t launch_snapshot(int64_t n, const double* A, const PanelDesc* d, double* out, cudaStream_t st) {
  snapshot_kernel<<<(unsigned)n, kDiagThreads, 0, st>>>(n, A, d, out);
  return cudaGetLastError();
}

cudaError_t launch_drift(int64_t n, int P, const double* A, const double* B, const double* omega_orig,
                         const int* perm, const PanelDesc* d, double* out, cudaStream_t st) {
  drift_kernel<<<(unsigned)n, kDiagThreads, sizeof(double) * (size_t)P, st>>>(n, P, A, B, omega_orig, perm, d, out);
  return cudaGetLastError();
}

cudaError_t launch_omega_scatter(int64_t n, int P, int64_t k0, const double* om, int64_t m, const int* perm,
                                 double* omega_orig, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  omega_scatter_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(n, P, k0, om, m, perm, omega_orig);
  return cudaGetLastError();
}

}  // namespace rcp
