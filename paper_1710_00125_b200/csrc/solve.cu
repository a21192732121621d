// Solve x = P^T L^-T D^-1 L^-1 P b against the device factorization
// (reference _substitute / block_diag_solve, solve.py:34-76), and L D L^T
// reconstruction (factor.py:663-665).
//
// L is the row-major unit lower factor.  The solve is HBM-bound (it reads L's lower
// triangle twice: n^2 * 8 bytes in total) with a sequential dependency along the
// diagonal, so each triangular sweep is ONE persistent launch:
//  * 64-row blocks are handed out by an atomic ticket in dependency order (forward:
//    0, 1, ...; backward: last first), so a CTA only ever waits for blocks already
//    owned by running CTAs -- no co-residency assumption, no deadlock.
//  * A block streams its off-diagonal L strip (rows i of L for the forward sweep,
//    the column strip below the block for the backward sweep) against the solution
//    blocks of earlier tickets as soon as each one is published (per-block
//    release/acquire flags, per-warp waits: no CTA barrier inside the stream loop).
//  * The diagonal block is applied as a product with its precomputed unit-lower
//    inverse (diag_inverse_kernel, all blocks in parallel), so the serial chain per
//    block is one flag hop plus a 64x64 matrix-vector product, not 64 dependent
//    substitution steps.
// Summation orders are fixed (per-lane partials over the strip, then a fixed shuffle
// tree), so the result is deterministic.
#include <algorithm>
#include "gemm_dmma.cuh"
#include "rcp_common.cuh"
#include "solve.cuh"

namespace rcp {

namespace {

constexpr int NB = 64;
constexpr int kSweepThreads = 256;  // 8 warps x 8 rows (forward) or 8 rows per strip block (backward)

RCP_D int ld_acquire_i(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
RCP_D void st_release_i(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

// Inverse of every 64x64 unit-lower diagonal block of L (rows beyond n: identity), stored
// row-major per block: Linv[blk][a][c], zero above the diagonal.  Thread c computes column c
// by forward substitution against e_c.
__global__ void __launch_bounds__(NB) diag_inverse_kernel(int64_t n, const double* __restrict__ L,
                                                            double* __restrict__ Linv) {
  __shared__ double X[NB][NB];  // column c belongs to thread c (conflict-free)
  const int64_t i0 = (int64_t)blockIdx.x * NB;
  const int nb = (int)(n - i0 < NB ? n - i0 : NB);
  const int c = threadIdx.x;
  for (int a = 0; a < NB; ++a) X[a][c] = 0.0;
  X[c][c] = 1.0;
  for (int a = c + 1; a < nb; ++a) {  // L_ii rows are read by all threads at once (broadcast)
    const double* la = L + (i0 + a) * n + i0;
    double s = 0.0;
    for (int j = c; j < a; ++j) s = __fma_rn(__ldg(la + j), X[j][c], s);
    X[a][c] = -s;
  }
  double* out = Linv + (int64_t)blockIdx.x * NB * NB;
  for (int a = 0; a < NB; ++a) out[a * NB + c] = X[a][c];
}

RCP_D double2 ld_pair(const double* p, bool aligned) {
  if (aligned) return __ldcs(reinterpret_cast<const double2*>(p));
  return make_double2(__ldcs(p), __ldcs(p + 1));
}

RCP_D double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// Forward sweep L z = P b (R right-hand sides; z column-major with ld ldz).  Block i:
// acc = y_i - sum_{j<i} L_ij z_j, z_i = Linv_ii acc.  The gather y = b[perm] is fused.
// Per warp: 8 rows of the block, lanes over 2 columns of each 64-wide strip block.  The L
// strip of block j is loaded BEFORE waiting for z_j's flag (L is read-only), so the wait for
// the last, just-published block overlaps its HBM latency; Linv_ii is staged in shared memory
// while the strip streams.
template <int R>
__global__ void __launch_bounds__(kSweepThreads) fwd_sweep_kernel(int64_t n, int64_t ldz, int nblk,
                                                                  const int64_t* __restrict__ perm,
                                                                  const double* __restrict__ L,
                                                                  const double* __restrict__ Linv,
                                                                  const double* __restrict__ b, double* __restrict__ z,
                                                                  int* flags, int* ticket) {
  __shared__ int s_blk;
  __shared__ double s_acc[R][NB];
  __shared__ double s_inv[NB][NB + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool al = (n & 1) == 0;  // rows of L are 16-byte aligned
  for (;;) {
    if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1);
    __syncthreads();
    const int i = s_blk;
    if (i >= nblk) return;
    const int64_t r0 = (int64_t)i * NB;
    for (int e = threadIdx.x; e < NB * NB; e += kSweepThreads) s_inv[e >> 6][e & 63] = Linv[(int64_t)i * NB * NB + e];
    double part[8][R];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int c = 0; c < R; ++c) part[q][c] = 0.0;
    int ready = 0;  // blocks j < ready are known to be published (lane 0 polls, the warp shares it)
    for (int j = 0; j < i; ++j) {
      const int64_t c0 = (int64_t)j * NB + 2 * lane;  // j < i: a full block
      double2 lv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t r = r0 + warp * 8 + q;
        lv[q] = (r < n) ? ld_pair(L + r * n + c0, al) : make_double2(0.0, 0.0);
      }
      if (j >= ready) {
        if (lane == 0) {
          while (ld_acquire_i(flags + j) == 0) {
          }
          int r = j + 1;
          while (r < i && ld_acquire_i(flags + r) != 0) ++r;
          ready = r;
        }
        ready = __shfl_sync(0xffffffffu, ready, 0);
        __syncwarp();
      }
      double2 zv[R];
#pragma unroll
      for (int c = 0; c < R; ++c) zv[c] = __ldcg(reinterpret_cast<const double2*>(z + c * ldz + c0));
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int c = 0; c < R; ++c) part[q][c] = __fma_rn(lv[q].y, zv[c].y, __fma_rn(lv[q].x, zv[c].x, part[q][c]));
    }
    // acc = y - sum (fixed shuffle tree), then z_i = Linv_ii acc
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int a = warp * 8 + q;
      const int64_t r = r0 + a;
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const double s = warp_sum(part[q][c]);
        if (lane == 0) s_acc[c][a] = (r < n) ? __dsub_rn(b[c * n + perm[r]], s) : 0.0;
      }
    }
    __syncthreads();
    {
      const int a = threadIdx.x >> 2, qtr = threadIdx.x & 3;  // 4 lanes per output row
      double d[R];
#pragma unroll
      for (int c = 0; c < R; ++c) d[c] = 0.0;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const double lv = s_inv[a][qtr * 16 + e];
#pragma unroll
        for (int c = 0; c < R; ++c) d[c] = __fma_rn(lv, s_acc[c][qtr * 16 + e], d[c]);
      }
#pragma unroll
      for (int c = 0; c < R; ++c) {
        d[c] = __dadd_rn(d[c], __shfl_xor_sync(0xffffffffu, d[c], 1));
        d[c] = __dadd_rn(d[c], __shfl_xor_sync(0xffffffffu, d[c], 2));
        if (qtr == 0 && r0 + a < n) z[c * ldz + r0 + a] = d[c];
      }
    }
    __syncthreads();  // every z_i store precedes the release (cumulativity through the barrier)
    if (threadIdx.x == 0) st_release_i(flags + i, 1);
  }
}

// Backward sweep L^T v = w (w = D^-1 z; v is a separate buffer).  Column block i:
// acc = w_i - sum_{j>i} L_ji^T v_j, v_i = Linv_ii^T acc; the scatter x[perm] = v is fused.
template <int R>
__global__ void __launch_bounds__(kSweepThreads) bwd_sweep_kernel(int64_t n, int64_t ldz, int nblk,
                                                                  const int64_t* __restrict__ perm,
                                                                  const double* __restrict__ L,
                                                                  const double* __restrict__ Linv,
                                                                  const double* __restrict__ w, double* __restrict__ v,
                                                                  double* __restrict__ x, int* flags, int* ticket) {
  __shared__ int s_blk;
  __shared__ double s_part[8][R][NB];
  __shared__ double s_acc[R][NB];
  __shared__ double s_inv[NB][NB + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool al = (n & 1) == 0;
  for (;;) {
    if (threadIdx.x == 0) s_blk = nblk - 1 - atomicAdd(ticket, 1);
    __syncthreads();
    const int i = s_blk;
    if (i < 0) return;
    const int64_t c0 = (int64_t)i * NB;
    const int ncol = (int)(n - c0 < NB ? n - c0 : NB);
    for (int e = threadIdx.x; e < NB * NB; e += kSweepThreads) s_inv[e >> 6][e & 63] = Linv[(int64_t)i * NB * NB + e];
    double part[2][R];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < R; ++c) part[e][c] = 0.0;
    int ready = nblk;  // blocks j >= ready are known to be published
    for (int j = nblk - 1; j > i; --j) {
      const int64_t rb = (int64_t)j * NB + warp * 8;
      double2 lv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t r = rb + q;
        const double* lp = L + r * n + c0 + 2 * lane;
        lv[q] = make_double2(0.0, 0.0);
        if (r < n) {
          if (2 * lane + 1 < ncol) {
            lv[q] = ld_pair(lp, al);
          } else if (2 * lane < ncol) {
            lv[q].x = __ldcs(lp);
          }
        }
      }
      if (j < ready) {
        if (lane == 0) {
          while (ld_acquire_i(flags + j) == 0) {
          }
          int r = j;
          while (r - 1 > i && ld_acquire_i(flags + r - 1) != 0) --r;
          ready = r;
        }
        ready = __shfl_sync(0xffffffffu, ready, 0);
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t r = rb + q;
        if (r < n) {
#pragma unroll
          for (int c = 0; c < R; ++c) {
            const double vr = __ldcg(v + c * ldz + r);
            part[0][c] = __fma_rn(lv[q].x, vr, part[0][c]);
            part[1][c] = __fma_rn(lv[q].y, vr, part[1][c]);
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < R; ++c) {
      s_part[warp][c][2 * lane] = part[0][c];
      s_part[warp][c][2 * lane + 1] = part[1][c];
    }
    __syncthreads();
    if (threadIdx.x < NB * R) {
      const int col = threadIdx.x % NB, c = threadIdx.x / NB;
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s = __dadd_rn(s, s_part[ww][c][col]);
      s_acc[c][col] = (col < ncol) ? __dsub_rn(w[c * ldz + c0 + col], s) : 0.0;
    }
    __syncthreads();
    {
      // v_i[col] = sum_a Linv[a][col] acc[a]: 4 lanes per output column, 16 rows each
      const int col = threadIdx.x >> 2, qtr = threadIdx.x & 3;
      double d[R];
#pragma unroll
      for (int c = 0; c < R; ++c) d[c] = 0.0;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int a = qtr * 16 + e;
        const double lv = s_inv[a][col];
#pragma unroll
        for (int c = 0; c < R; ++c) d[c] = __fma_rn(lv, s_acc[c][a], d[c]);
      }
#pragma unroll
      for (int c = 0; c < R; ++c) {
        d[c] = __dadd_rn(d[c], __shfl_xor_sync(0xffffffffu, d[c], 1));
        d[c] = __dadd_rn(d[c], __shfl_xor_sync(0xffffffffu, d[c], 2));
        if (qtr == 0 && col < ncol) {
          v[c * ldz + c0 + col] = d[c];
          x[c * n + perm[c0 + col]] = d[c];
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) st_release_i(flags + i, 1);
  }
}

// D w = z blockwise (solve.py:34-66): exact-zero blocks give zeros and set *singular.
__global__ void block_diag_kernel(int64_t n, int64_t ldz, int64_t nrhs, const double* __restrict__ dd,
                                  const double* __restrict__ doff, const int8_t* __restrict__ pattern,
                                  double* __restrict__ z, int* singular) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int8_t pt = pattern[i];
  if (pt == 2) return;  // second index of a 2x2 block, handled by its first index
  for (int64_t c = 0; c < nrhs; ++c) {
    double* zc = z + c * ldz;
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

// workspace: Linv (nblk x 64 x 64) | z (n x nrhs) | v (n x nrhs) | 2 x nblk flags + 2 tickets
static size_t rup(size_t x) { return (x + 255) / 256 * 256; }
size_t solve_workspace_bytes(int64_t n, int64_t nrhs) {
  const size_t nblk = (size_t)((n + NB - 1) / NB);
  return rup(nblk * NB * NB * 8) + 2 * rup(nblk * NB * (size_t)nrhs * 8) + rup((2 * nblk + 2) * 4);
}

template <int R>
static void launch_sweeps(int64_t n, int nblk, const int64_t* perm, const double* L, const double* Linv,
                          const double* dd, const double* doff, const int8_t* pattern, const double* b, double* x,
                          double* z, double* v, int* flags, int* singular, int grid_f, int grid_b, cudaStream_t st) {
  const int64_t ldz = (int64_t)nblk * NB;
  fwd_sweep_kernel<R><<<grid_f, kSweepThreads, 0, st>>>(n, ldz, nblk, perm, L, Linv, b, z, flags, flags + 2 * nblk);
  block_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, ldz, R, dd, doff, pattern, z, singular);
  bwd_sweep_kernel<R><<<grid_b, kSweepThreads, 0, st>>>(n, ldz, nblk, perm, L, Linv, z, v, x, flags + nblk,
                                                         flags + 2 * nblk + 1);
}

cudaError_t solve_device(int64_t n, const int64_t* perm, const double* L, const double* dd, const double* doff,
                         const int8_t* pattern, int64_t nrhs, const double* b, double* x, void* ws, int* singular,
                         cudaStream_t st, int num_sms) {
  const int nblk = (int)((n + NB - 1) / NB);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  double* Linv = reinterpret_cast<double*>(p);
  p += rup((size_t)nblk * NB * NB * 8);
  double* z = reinterpret_cast<double*>(p);
  const int64_t ldz = (int64_t)nblk * NB;
  p += rup((size_t)ldz * (size_t)nrhs * 8);
  double* v = reinterpret_cast<double*>(p);
  p += rup((size_t)ldz * (size_t)nrhs * 8);
  int* flags = reinterpret_cast<int*>(p);
  diag_inverse_kernel<<<nblk, NB, 0, st>>>(n, L, Linv);
  // x may alias b: the forward sweep reads b (gather) before the backward sweep writes x
  const int grid = std::max(1, std::min(nblk, 2 * num_sms));
  for (int64_t c0 = 0; c0 < nrhs; c0 += 3) {  // up to 3 right-hand sides per pair of sweeps (smem)
    const int64_t r = std::min<int64_t>(3, nrhs - c0);
    cudaError_t e = cudaMemsetAsync(flags, 0, (size_t)(2 * nblk + 2) * 4, st);
    if (e != cudaSuccess) return e;
    const double* bc = b + c0 * n;
    double* xc = x + c0 * n;
    double* zc = z + c0 * ldz;
    double* vc = v + c0 * ldz;
    if (r == 3)
      launch_sweeps<3>(n, nblk, perm, L, Linv, dd, doff, pattern, bc, xc, zc, vc, flags, singular, grid, grid, st);
    else if (r == 2)
      launch_sweeps<2>(n, nblk, perm, L, Linv, dd, doff, pattern, bc, xc, zc, vc, flags, singular, grid, grid, st);
    else
      launch_sweeps<1>(n, nblk, perm, L, Linv, dd, doff, pattern, bc, xc, zc, vc, flags, singular, grid, grid, st);
  }
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
