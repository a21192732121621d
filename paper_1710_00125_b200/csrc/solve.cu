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
#include <atomic>
#include "gemm_dmma.cuh"
#include "rcp_common.cuh"
#include "solve.cuh"

namespace rcp {

namespace {

constexpr int NB = 64;
// 8 warps x 8 rows of a 64-row block (measured: 128-thread CTAs, 4 per SM so that every C3 block row
// is resident from the start, were slower: 5.60 vs 4.56 ms -- the chain, not the tail, dominates)
constexpr int kSweepThreads = 256;
constexpr int kWarps = kSweepThreads / 32, kRPW = NB / kWarps;   // rows per warp
constexpr int kMvLanes = kSweepThreads / NB, kMvCols = NB / kMvLanes;  // matrix-vector split
// published strip blocks streamed per iteration (memory-level parallelism); measured at C3:
// R = 1: kU 4 -> 4.36 ms, kU 2 -> 4.82 ms; R = 3: kU 2 -> 8.37 ms, kU 4 -> 9.13 ms (registers)
// (strip_unroll: kU = 4 for one right-hand side, 2 for more)

RCP_D int ld_acquire_i(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
RCP_D void st_release_i(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

// Per 64-row block i of L (rows beyond n: identity / zero), all blocks in parallel:
//   Linv_i = inverse of the unit-lower diagonal block L_ii           (row-major [a][c])
//   M_i    = Linv_i L_{i,i-1}   (coupling of block i to the block before it, forward sweep)
//   N_i    = Linv_i^T L_{i+1,i}^T   (coupling to the block after it, backward sweep)
// With them the forward step is z_i = Linv_i (y_i - sum_{j<i-1} L_ij z_j) - M_i z_{i-1}: only the
// last product waits for the previous block, so the serial chain per block is one flag hop and a
// 64 x 64 matrix-vector product (same for the backward sweep with N_i).
constexpr int kPrepThreads = 256;
__global__ void __launch_bounds__(kPrepThreads) block_prep_kernel(int64_t n, int nblk, const double* __restrict__ L,
                                                                   double* __restrict__ Linv, double* __restrict__ M,
                                                                   double* __restrict__ N) {
  extern __shared__ double sp[];
  double(*X)[NB] = reinterpret_cast<double(*)[NB]>(sp);                // Linv_i, column c by thread c
  double(*B)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(sp + NB * NB);  // an off-diagonal L block
  const int i = blockIdx.x, tid = threadIdx.x;
  const int64_t i0 = (int64_t)i * NB;
  const int nb = (int)(n - i0 < NB ? n - i0 : NB);
  if (tid < NB) {
    const int c = tid;
    for (int a = 0; a < NB; ++a) X[a][c] = 0.0;
    X[c][c] = 1.0;
    for (int a = c + 1; a < nb; ++a) {  // L_ii rows are read by all threads at once (broadcast)
      const double* la = L + (i0 + a) * n + i0;
      double s = 0.0;
      for (int j = c; j < a; ++j) s = __fma_rn(__ldg(la + j), X[j][c], s);
      X[a][c] = -s;
    }
  }
  __syncthreads();
  for (int e = tid; e < NB * NB; e += kPrepThreads) Linv[(int64_t)i * NB * NB + e] = X[e >> 6][e & 63];
  // M_i = Linv_i L_{i,i-1}: B[e][c] = L[i0 + e][i0 - 64 + c]
  if (i > 0) {
    for (int e = tid; e < NB * NB; e += kPrepThreads) {
      const int r = e >> 6, c = e & 63;
      B[r][c] = (r < nb) ? L[(i0 + r) * n + i0 - NB + c] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < NB * NB; e += kPrepThreads) {
      const int a = e >> 6, c = e & 63;
      double s = 0.0;
      for (int k = 0; k < NB; ++k) s = __fma_rn(X[a][k], B[k][c], s);
      M[(int64_t)i * NB * NB + e] = s;
    }
    __syncthreads();
  }
  // N_i = Linv_i^T L_{i+1,i}^T: B[e'][a] = L[i0 + 64 + e'][i0 + a];  N[c][e'] = sum_a X[a][c] B[e'][a]
  if (i + 1 < nblk) {
    const int nb1 = (int)(n - i0 - NB < NB ? n - i0 - NB : NB);
    for (int e = tid; e < NB * NB; e += kPrepThreads) {
      const int r = e >> 6, a = e & 63;
      B[r][a] = (r < nb1) ? L[(i0 + NB + r) * n + i0 + a] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < NB * NB; e += kPrepThreads) {
      const int c = e >> 6, r = e & 63;
      double s = 0.0;
      for (int a = 0; a < NB; ++a) s = __fma_rn(X[a][c], B[r][a], s);
      N[(int64_t)i * NB * NB + e] = s;
    }
  }
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

// The block on the serial chain is also published as "LL" words (32 data bits + a 32-bit tag per
// 64-bit store, single-copy atomic): the next block polls the data itself, one L2 round trip instead
// of flag-then-data, and the producer needs no release fence for it.  tag = a per-call epoch.
typedef unsigned long long u64;
RCP_D void ll_put2(u64* p, unsigned tag, double x) {
  const u64 b = static_cast<u64>(__double_as_longlong(x));
  const u64 w0 = (static_cast<u64>(tag) << 32) | (b & 0xffffffffull), w1 = (static_cast<u64>(tag) << 32) | (b >> 32);
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
// Read N consecutive LL doubles (2 words each) once every word carries `tag`.
template <int N>
RCP_D void ll_get_n(const u64* p, unsigned tag, double (&out)[N]) {
  for (;;) {
    bool ok = true;
#pragma unroll
    for (int e = 0; e < N; ++e) {
      u64 w0, w1;
      asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p + 2 * e) : "memory");
      ok &= (static_cast<unsigned>(w0 >> 32) == tag) & (static_cast<unsigned>(w1 >> 32) == tag);
      out[e] = __longlong_as_double(static_cast<long long>((w1 << 32) | (w0 & 0xffffffffull)));
    }
    if (ok) return;
  }
}

// Forward sweep L z = P b (R right-hand sides; z column-major with ld ldz).  Block i:
//   pre = Linv_i (y_i - sum_{j<i-1} L_ij z_j)   (streamed as earlier blocks are published)
//   z_i = pre - M_i z_{i-1}                     (the one product on the serial chain)
// Warps take 8 rows of the block each, lanes 2 columns of each 64-wide strip block; the L strip of
// block j is loaded before waiting for z_j.  The gather y = b[perm] is fused.
template <int R>
__global__ void __launch_bounds__(kSweepThreads) fwd_sweep_kernel(int64_t n, int64_t ldz, int nblk,
                                                                  const int64_t* __restrict__ perm,
                                                                  const double* __restrict__ L,
                                                                  const double* __restrict__ Linv,
                                                                  const double* __restrict__ M,
                                                                  const double* __restrict__ b, double* __restrict__ z,
                                                                  u64* __restrict__ zll, unsigned tag, int* flags,
                                                                  int* ticket) {
  constexpr int kU = (R == 1) ? 4 : 2;  // see strip_unroll
  __shared__ int s_blk;
  __shared__ double s_acc[R][NB];
  __shared__ double s_cpl[NB][NB + 1];  // M_i, staged while the strip streams
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = threadIdx.x / kMvLanes, qtr = threadIdx.x % kMvLanes;  // matrix-vector: row a, kMvCols columns
  const bool al = (n & 1) == 0;
  for (;;) {
    if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1);
    __syncthreads();
    const int i = s_blk;
    if (i >= nblk) return;
    const int64_t r0 = (int64_t)i * NB;
    if (i > 0)  // M_i, needed after the wait (staged now, off the chain)
      for (int e = threadIdx.x; e < NB * NB; e += kSweepThreads) s_cpl[e >> 6][e & 63] = __ldg(M + (int64_t)i * NB * NB + e);
    double part[kRPW][R];
#pragma unroll
    for (int q = 0; q < kRPW; ++q)
#pragma unroll
      for (int c = 0; c < R; ++c) part[q][c] = 0.0;
    int ready = 0;  // blocks j < ready are known to be published
    for (int j = 0; j + 1 < i;) {
      if (j + kU <= i - 1 && j + kU <= ready) {  // kU published blocks: all their loads in flight at once
        double2 lv[kU][kRPW], zv[kU][R];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t c0 = (int64_t)(j + u) * NB + 2 * lane;
#pragma unroll
          for (int q = 0; q < kRPW; ++q) {
            const int64_t r = r0 + warp * kRPW + q;
            lv[u][q] = (r < n) ? ld_pair(L + r * n + c0, al) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int c = 0; c < R; ++c) zv[u][c] = __ldcg(reinterpret_cast<const double2*>(z + c * ldz + c0));
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int q = 0; q < kRPW; ++q)
#pragma unroll
            for (int c = 0; c < R; ++c)
              part[q][c] = __fma_rn(lv[u][q].y, zv[u][c].y, __fma_rn(lv[u][q].x, zv[u][c].x, part[q][c]));
        j += kU;
        continue;
      }
      const int64_t c0 = (int64_t)j * NB + 2 * lane;
      double2 lv[kRPW];
#pragma unroll
      for (int q = 0; q < kRPW; ++q) {
        const int64_t r = r0 + warp * kRPW + q;
        lv[q] = (r < n) ? ld_pair(L + r * n + c0, al) : make_double2(0.0, 0.0);
      }
      if (j >= ready) {
        if (lane == 0) {
          while (ld_acquire_i(flags + j) == 0) {
          }
          int rr = j + 1;
          while (rr + 1 < i && ld_acquire_i(flags + rr) != 0) ++rr;
          ready = rr;
        }
        ready = __shfl_sync(0xffffffffu, ready, 0);
        __syncwarp();
      }
      double2 zv[R];
#pragma unroll
      for (int c = 0; c < R; ++c) zv[c] = __ldcg(reinterpret_cast<const double2*>(z + c * ldz + c0));
#pragma unroll
      for (int q = 0; q < kRPW; ++q)
#pragma unroll
        for (int c = 0; c < R; ++c) part[q][c] = __fma_rn(lv[q].y, zv[c].y, __fma_rn(lv[q].x, zv[c].x, part[q][c]));
      ++j;
    }
#pragma unroll
    for (int q = 0; q < kRPW; ++q) {
      const int ar = warp * kRPW + q;
      const int64_t r = r0 + ar;
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const double sm = warp_sum(part[q][c]);
        if (lane == 0) s_acc[c][ar] = (r < n) ? __dsub_rn(b[c * n + perm[r]], sm) : 0.0;
      }
    }
    __syncthreads();
    double d[R];
    {
      const double* li = Linv + (int64_t)i * NB * NB + a * NB + qtr * kMvCols;
#pragma unroll
      for (int c = 0; c < R; ++c) d[c] = 0.0;
#pragma unroll
      for (int e = 0; e < kMvCols; ++e) {
        const double lv = __ldg(li + e);
#pragma unroll
        for (int c = 0; c < R; ++c) d[c] = __fma_rn(lv, s_acc[c][qtr * kMvCols + e], d[c]);
      }
    }
    if (i > 0) {  // the serial step: z_{i-1} straight from its LL words, subtract M_i z_{i-1}
#pragma unroll
      for (int c = 0; c < R; ++c) {
        double zz[kMvCols];
        ll_get_n<kMvCols>(zll + (((int64_t)(i - 1) * R + c) * NB + qtr * kMvCols) * 2, tag, zz);
        double m = 0.0;
#pragma unroll
        for (int e = 0; e < kMvCols; ++e) m = __fma_rn(s_cpl[a][qtr * kMvCols + e], zz[e], m);
        d[c] = __dsub_rn(d[c], m);
      }
    }
#pragma unroll
    for (int c = 0; c < R; ++c) {
#pragma unroll
      for (int off = 1; off < kMvLanes; off <<= 1) d[c] = __dadd_rn(d[c], __shfl_xor_sync(0xffffffffu, d[c], off));
      if (qtr == 0) {
        ll_put2(zll + (((int64_t)i * R + c) * NB + a) * 2, tag, d[c]);
        if (r0 + a < n) z[c * ldz + r0 + a] = d[c];
      }
    }
    __syncthreads();  // every z_i store precedes the release (cumulativity through the barrier)
    if (threadIdx.x == 0) st_release_i(flags + i, 1);
  }
}

// Backward sweep L^T v = w (w = D^-1 z; v a separate buffer).  Column block i (descending):
//   pre = Linv_i^T (w_i - sum_{j>i+1} L_ji^T v_j),  v_i = pre - N_i v_{i+1};  x[perm] = v fused.
template <int R>
__global__ void __launch_bounds__(kSweepThreads) bwd_sweep_kernel(int64_t n, int64_t ldz, int nblk,
                                                                  const int64_t* __restrict__ perm,
                                                                  const double* __restrict__ L,
                                                                  const double* __restrict__ Linv,
                                                                  const double* __restrict__ Nc,
                                                                  const double* __restrict__ w, double* __restrict__ v,
                                                                  double* __restrict__ x, u64* __restrict__ vll, unsigned tag,
                                                                  int* flags, int* ticket) {
  constexpr int kU = (R == 1) ? 4 : 2;  // see strip_unroll
  __shared__ int s_blk;
  __shared__ double s_part[kWarps][R][NB];
  __shared__ double s_acc[R][NB];
  __shared__ double s_cpl[NB][NB + 1];  // N_i, staged while the strip streams
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = threadIdx.x / kMvLanes, qtr = threadIdx.x % kMvLanes;  // output column col, kMvCols rows
  const bool al = (n & 1) == 0;
  for (;;) {
    if (threadIdx.x == 0) s_blk = nblk - 1 - atomicAdd(ticket, 1);
    __syncthreads();
    const int i = s_blk;
    if (i < 0) return;
    const int64_t c0 = (int64_t)i * NB;
    const int ncol = (int)(n - c0 < NB ? n - c0 : NB);
    if (i + 1 < nblk)
      for (int e = threadIdx.x; e < NB * NB; e += kSweepThreads) s_cpl[e >> 6][e & 63] = __ldg(Nc + (int64_t)i * NB * NB + e);
    double part[2][R];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < R; ++c) part[e][c] = 0.0;
    int ready = nblk;  // blocks j >= ready are known to be published
    for (int j = nblk - 1; j > i + 1;) {
      if (j - kU + 1 > i + 1 && j - kU + 1 >= ready) {  // blocks j-kU+1..j published: loads in flight together
        double2 lv[kU][kRPW];
        double vr[kU][kRPW][R];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t rb = (int64_t)(j - u) * NB + warp * kRPW;
#pragma unroll
          for (int q = 0; q < kRPW; ++q) {
            const int64_t r = rb + q;
            const double* lp = L + r * n + c0 + 2 * lane;
            lv[u][q] = make_double2(0.0, 0.0);
            if (r < n) {
              if (2 * lane + 1 < ncol) {
                lv[u][q] = ld_pair(lp, al);
              } else if (2 * lane < ncol) {
                lv[u][q].x = __ldcs(lp);
              }
            }
#pragma unroll
            for (int c = 0; c < R; ++c) vr[u][q][c] = (r < n) ? __ldcg(v + c * ldz + r) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int q = 0; q < kRPW; ++q)
#pragma unroll
            for (int c = 0; c < R; ++c) {
              part[0][c] = __fma_rn(lv[u][q].x, vr[u][q][c], part[0][c]);
              part[1][c] = __fma_rn(lv[u][q].y, vr[u][q][c], part[1][c]);
            }
        j -= kU;
        continue;
      }
      const int64_t rb = (int64_t)j * NB + warp * kRPW;
      double2 lv[kRPW];
#pragma unroll
      for (int q = 0; q < kRPW; ++q) {
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
          int rr = j;
          while (rr - 1 > i + 1 && ld_acquire_i(flags + rr - 1) != 0) --rr;
          ready = rr;
        }
        ready = __shfl_sync(0xffffffffu, ready, 0);
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < kRPW; ++q) {
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
      --j;
    }
#pragma unroll
    for (int c = 0; c < R; ++c) {
      s_part[warp][c][2 * lane] = part[0][c];
      s_part[warp][c][2 * lane + 1] = part[1][c];
    }
    __syncthreads();
    for (int f = threadIdx.x; f < NB * R; f += kSweepThreads) {
      const int cc = f % NB, c = f / NB;
      double sm = 0.0;
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) sm = __dadd_rn(sm, s_part[ww][c][cc]);
      s_acc[c][cc] = (cc < ncol) ? __dsub_rn(w[c * ldz + c0 + cc], sm) : 0.0;
    }
    __syncthreads();
    double d[R];
    {
      const double* li = Linv + (int64_t)i * NB * NB + col;
#pragma unroll
      for (int c = 0; c < R; ++c) d[c] = 0.0;
#pragma unroll
      for (int e = 0; e < kMvCols; ++e) {
        const int ar = qtr * kMvCols + e;
        const double lv = __ldg(li + ar * NB);
#pragma unroll
        for (int c = 0; c < R; ++c) d[c] = __fma_rn(lv, s_acc[c][ar], d[c]);
      }
    }
    if (i + 1 < nblk) {  // the serial step: v_{i+1} straight from its LL words, subtract N_i v_{i+1}
#pragma unroll
      for (int c = 0; c < R; ++c) {
        double vv[kMvCols];
        ll_get_n<kMvCols>(vll + (((int64_t)(i + 1) * R + c) * NB + qtr * kMvCols) * 2, tag, vv);
        double m = 0.0;
#pragma unroll
        for (int e = 0; e < kMvCols; ++e) m = __fma_rn(s_cpl[col][qtr * kMvCols + e], vv[e], m);
        d[c] = __dsub_rn(d[c], m);
      }
    }
#pragma unroll
    for (int c = 0; c < R; ++c) {
#pragma unroll
      for (int off = 1; off < kMvLanes; off <<= 1) d[c] = __dadd_rn(d[c], __shfl_xor_sync(0xffffffffu, d[c], off));
      if (qtr == 0) {
        ll_put2(vll + (((int64_t)i * R + c) * NB + col) * 2, tag, col < ncol ? d[c] : 0.0);
        if (col < ncol) {
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

// workspace: Linv, M, N (nblk x 64 x 64 each) | z, v (ldz x nrhs) | z, v LL words (nblk x 3 x 64 x 2) |
//            2 x nblk flags + 2 tickets
static size_t rup(size_t x) { return (x + 255) / 256 * 256; }
size_t solve_workspace_bytes(int64_t n, int64_t nrhs) {
  const size_t nblk = (size_t)((n + NB - 1) / NB);
  return 3 * rup(nblk * NB * NB * 8) + 2 * rup(nblk * NB * (size_t)nrhs * 8) + 2 * rup(nblk * 3 * NB * 16) +
         rup((2 * nblk + 2) * 4);
}

template <int R>
static void launch_sweeps(int64_t n, int nblk, const int64_t* perm, const double* L, const double* Linv,
                          const double* M, const double* N, const double* dd, const double* doff,
                          const int8_t* pattern, const double* b, double* x, double* z, double* v, u64* zll,
                          u64* vll, unsigned tag, int* flags, int* singular, int grid, cudaStream_t st) {
  const int64_t ldz = (int64_t)nblk * NB;
  fwd_sweep_kernel<R><<<grid, kSweepThreads, 0, st>>>(n, ldz, nblk, perm, L, Linv, M, b, z, zll, tag, flags,
                                                      flags + 2 * nblk);
  block_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, ldz, R, dd, doff, pattern, z, singular);
  bwd_sweep_kernel<R><<<grid, kSweepThreads, 0, st>>>(n, ldz, nblk, perm, L, Linv, N, z, v, x, vll, tag,
                                                      flags + nblk, flags + 2 * nblk + 1);
}

cudaError_t solve_device(int64_t n, const int64_t* perm, const double* L, const double* dd, const double* doff,
                         const int8_t* pattern, int64_t nrhs, const double* b, double* x, void* ws, int* singular,
                         cudaStream_t st, int num_sms) {
  const int nblk = (int)((n + NB - 1) / NB);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  const size_t blk_bytes = rup((size_t)nblk * NB * NB * 8);
  double* Linv = reinterpret_cast<double*>(p);
  double* M = reinterpret_cast<double*>(p + blk_bytes);
  double* N = reinterpret_cast<double*>(p + 2 * blk_bytes);
  p += 3 * blk_bytes;
  double* z = reinterpret_cast<double*>(p);
  const int64_t ldz = (int64_t)nblk * NB;
  p += rup((size_t)ldz * (size_t)nrhs * 8);
  double* v = reinterpret_cast<double*>(p);
  p += rup((size_t)ldz * (size_t)nrhs * 8);
  u64* zll = reinterpret_cast<u64*>(p);
  p += rup((size_t)nblk * 3 * NB * 16);
  u64* vll = reinterpret_cast<u64*>(p);
  p += rup((size_t)nblk * 3 * NB * 16);
  int* flags = reinterpret_cast<int*>(p);
  const size_t prep_smem = sizeof(double) * (NB * NB + NB * (NB + 1));
  static thread_local int prep_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != prep_dev) {
    cudaError_t e = cudaFuncSetAttribute(block_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prep_smem);
    if (e != cudaSuccess) return e;
    prep_dev = dev;
  }
  block_prep_kernel<<<nblk, kPrepThreads, prep_smem, st>>>(n, nblk, L, Linv, M, N);
  // x may alias b: the forward sweep reads b (gather) before the backward sweep writes x
  const int grid = std::max(1, std::min(nblk, 2 * num_sms));
  for (int64_t c0 = 0; c0 < nrhs; c0 += 3) {  // up to 3 right-hand sides per pair of sweeps
    const int64_t r = std::min<int64_t>(3, nrhs - c0);
    cudaError_t e = cudaMemsetAsync(flags, 0, (size_t)(2 * nblk + 2) * 4, st);
    if (e != cudaSuccess) return e;
    const double* bc = b + c0 * n;
    double* xc = x + c0 * n;
    double* zc = z + c0 * ldz;
    double* vc = v + c0 * ldz;
    // LL tag: a fresh epoch per pair of sweeps (the LL buffers are never cleared; a stale word from
    // an earlier call carries an older tag)
    static std::atomic<unsigned> epoch{0};
    const unsigned tag = epoch.fetch_add(1) + 1;
    if (r == 3)
      launch_sweeps<3>(n, nblk, perm, L, Linv, M, N, dd, doff, pattern, bc, xc, zc, vc, zll, vll, tag, flags, singular,
                       grid, st);
    else if (r == 2)
      launch_sweeps<2>(n, nblk, perm, L, Linv, M, N, dd, doff, pattern, bc, xc, zc, vc, zll, vll, tag, flags, singular,
                       grid, st);
    else
      launch_sweeps<1>(n, nblk, perm, L, Linv, M, N, dd, doff, pattern, bc, xc, zc, vc, zll, vll, tag, flags, singular,
                       grid, st);
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
