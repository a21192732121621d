// Trailing Schur update A22 <- A22 - L21 W21^T (factor.py:369-379 + core.py:115-119) as a
// dedicated FP64 DMMA kernel.
//
// Why a dedicated kernel: at K = t <= 129 the update is only ~10.7 flop/B (read C,
// write C and its mirror), close to the B200 FP64 ridge (~5.7 flop/B), so a tile's
// HBM epilogue costs about half of its MMA mainloop.  Two CTAs per SM (128 threads,
// 128 x 64 tile, <= 100 KB smem each) let one CTA's epilogue overlap the other's
// DMMA mainloop instead of serialising them.
//
// Tiles: row blocks of 128 (I), column blocks of 64 (J), only those touching the lower
// triangle (J <= 2I + 1).  The C-in gather (previous trailing block read through the
// panel permutation) is prefetched into L2 at tile start, fetched with cp.async into the
// freed operand ring after the mainloop, summed with the accumulators, and written back
// column-wise (lower part) and row-wise (mirror of the strictly-lower part), both
// coalesced.  Full symmetric storage keeps every column contiguous for the next panel.
#pragma once
#include "gemm_dmma.cuh"

namespace rcp {

constexpr int kSchurBM = 128, kSchurBN = 64, kSchurThreads = 128, kSchurStages = 3;

struct SchurSmem {
  union {
    struct {
      double a[kSchurStages][kSchurBM][kBK + kPad];
      double b[kSchurStages][kSchurBN][kBK + kPad];
    } op;
    double c[kSchurBN][kSchurBM + 1];  // epilogue C tile c[j][i], reuses the operand ring
  };
  int rowmap[kSchurBM];
  int colmap[kSchurBN];
};

// Operand stage loader: thread t copies 16-byte chunks (rows r0 + 16u, columns kk..kk+1) of
// a ROWS x kBK tile; the per-thread row base is computed once per launch.
template <int ROWS>
struct StageLoader {
  const double* base;  // row (row0 + tid/8) of the operand, column (tid%8)*2
  int64_t step;        // 16 rows
  int nvalid;          // rows r0 + 16u valid for u < nvalid
  int soff;            // smem column offset
  int srow;            // first smem row
  RCP_D void init(const double* op, int64_t ld, int64_t rows, int64_t row0) {
    srow = threadIdx.x / 8;
    soff = (threadIdx.x % 8) * 2;
    base = op + (row0 + srow) * ld + soff;
    step = 16 * ld;
    const int64_t left = rows - (row0 + srow);
    nvalid = left <= 0 ? 0 : (left + 15) / 16;
  }
  RCP_D void load(double (*dst)[kBK + kPad], int64_t k0) const {
    const double* src = base + k0;
#pragma unroll
    for (int u = 0; u < ROWS / 16; ++u) {
      const bool ok = u < nvalid;
      cp_async16(&dst[srow + 16 * u][soff], ok ? src + u * step : base, ok);
    }
  }
};

// Lneg, Wg: (rows x tpad) K-contiguous, zero padded in [t, tpad).  A_in / A_out: n x n
// column-major full symmetric.  phys[j]: physical row (panel-start order) of new logical k+j.
__global__ void __launch_bounds__(kSchurThreads, 2)
schur_update_kernel(const double* __restrict__ Lneg, const double* __restrict__ Wg, int tpad, int Kl,
                    const double* __restrict__ ain, double* __restrict__ aout, const int* __restrict__ phys,
                    int64_t n, int64_t k, int64_t mp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SchurSmem& sm = *reinterpret_cast<SchurSmem*>(smem_raw);
  // tile (I, J): I = floor((sqrt(4x+1)-1)/2), J = x - I(I+1)   (row block I has 2I+2 col blocks)
  const long long x = blockIdx.x;
  long long I = static_cast<long long>((sqrt(4.0 * (double)x + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) > x) --I;
  while ((I + 1) * (I + 2) <= x) ++I;
  const long long J = x - I * (I + 1);
  const int64_t m0 = I * kSchurBM, n0 = J * kSchurBN;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int wm0 = (warp >> 1) * 64, wn0 = (warp & 1) * 32;
  constexpr int MF = 8, NF = 4;

  for (int i = tid; i < kSchurBM; i += kSchurThreads) sm.rowmap[i] = (m0 + i < mp) ? phys[m0 + i] : 0;
  for (int j = tid; j < kSchurBN; j += kSchurThreads) sm.colmap[j] = (n0 + j < mp) ? phys[n0 + j] : 0;

  const int KT = Kl / kBK;
  StageLoader<kSchurBM> la;
  StageLoader<kSchurBN> lb;
  la.init(Lneg, tpad, mp, m0);
  lb.init(Wg, tpad, mp, n0);
#pragma unroll
  for (int s = 0; s < kSchurStages - 1; ++s) {
    if (s < KT) {
      la.load(sm.op.a[s], (int64_t)s * kBK);
      lb.load(sm.op.b[s], (int64_t)s * kBK);
    }
    cp_async_commit();
  }
  __syncthreads();  // row/col maps visible
  // L2 prefetch of the C-in gather (one 128-row column segment per tile column)
  for (int e = tid; e < kSchurBN * 8; e += kSchurThreads) {
    const int j = e >> 3, seg = e & 7;
    if (n0 + j < mp && m0 + seg * 16 < mp) {
      const double* pp = ain + (int64_t)sm.rowmap[seg * 16] + (int64_t)sm.colmap[j] * n;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pp));
    }
  }

  double acc[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<kSchurStages - 2>();
    __syncthreads();
    {
      const int nk = kt + kSchurStages - 1;
      if (nk < KT) {
        const int st = nk % kSchurStages;
        la.load(sm.op.a[st], (int64_t)nk * kBK);
        lb.load(sm.op.b[st], (int64_t)nk * kBK);
      }
      cp_async_commit();
    }
    const int st = kt % kSchurStages;
    // fragments double-buffered: the loads for k-step kk+4 are issued before the MMAs of kk
    double af[2][MF], bf[2][NF];
#pragma unroll
    for (int i = 0; i < MF; ++i) af[0][i] = sm.op.a[st][wm0 + 8 * i + g][q];
#pragma unroll
    for (int j = 0; j < NF; ++j) bf[0][j] = sm.op.b[st][wn0 + 8 * j + g][q];
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      const int cb = (kk / 4) & 1;
      if (kk + 4 < kBK) {
#pragma unroll
        for (int i = 0; i < MF; ++i) af[cb ^ 1][i] = sm.op.a[st][wm0 + 8 * i + g][kk + 4 + q];
#pragma unroll
        for (int j = 0; j < NF; ++j) bf[cb ^ 1][j] = sm.op.b[st][wn0 + 8 * j + g][kk + 4 + q];
      }
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cb][i], bf[cb][j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // operand ring free

  // ---- epilogue: C-in gather -> smem (cp.async, L2-prefetched), += acc, then store the
  //      lower part column-wise and its mirror row-wise, both coalesced from smem.
  // thread tid owns tile row i = tid for the gather and the column-wise store
  static_assert(kSchurThreads == kSchurBM, "one thread per tile row");
  const int64_t gi_row = m0 + tid;
  const bool row_ok = gi_row < mp;
  // j < jmax: element (gi_row, n0 + j) is in range and on/below the diagonal
  const int64_t jlim = (mp < gi_row + 1 ? mp : gi_row + 1) - n0;
  const int jmax = (int)(jlim < kSchurBN ? (jlim > 0 ? jlim : 0) : kSchurBN);
  {
    const double* src = ain + (int64_t)sm.rowmap[tid];
    for (int j = 0; j < kSchurBN; ++j) {
      const bool ok = row_ok && j < jmax;
      cp_async8(&sm.c[j][tid], ok ? src + (int64_t)sm.colmap[j] * n : ain, ok);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int li = wm0 + 8 * i + g, lj = wn0 + 8 * j + 2 * q;
      sm.c[lj][li] = __dadd_rn(sm.c[lj][li], acc[i][j][0]);
      sm.c[lj + 1][li] = __dadd_rn(sm.c[lj + 1][li], acc[i][j][1]);
    }
  __syncthreads();
  if (row_ok) {  // lower part: column j, rows m0..m0+127 (coalesced along the threads)
    double* dst = aout + (k + gi_row) + (k + n0) * n;
    for (int j = 0; j < jmax; ++j, dst += n) *dst = sm.c[j][tid];
  }
  if (m0 + kSchurBM - 1 > n0) {  // mirror of the strictly-lower part: row (k+n0+j), columns k+m0+i
    const int j = tid & 63, i0 = tid >> 6;
    const int64_t gj = n0 + j;
    if (gj < mp) {
      double* dst = aout + (k + gj) + (k + m0 + i0) * n;
      const int imax = (int)(mp - m0 < kSchurBM ? mp - m0 : kSchurBM);
      for (int i = i0; i < imax; i += 2, dst += 2 * n)
        if (m0 + i > gj) *dst = sm.c[j][i];
    }
  }
}

inline size_t schur_smem_bytes() { return sizeof(SchurSmem); }

}  // namespace rcp
