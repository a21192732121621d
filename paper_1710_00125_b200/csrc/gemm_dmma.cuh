// FP64 tensor-core GEMM core for the dense contractions of the RCP path:
//   - trailing Schur update   A22 <- A22 - L21 * W21^T   (lower tiles only, permuted gather-in)
//   - sketch                  B   <- Omega * A
//   - sketch correction       B2  <- B2 - Y * L21^T      (permuted gather-in)
//
// out[m][n] = cin[m][n] + sum_k Aop[m][k] * Bop[n][k]
// Both operands are K-contiguous row arrays (row r at base + r * ld), staged into
// shared memory by a cp.async ring (STAGES deep) and consumed by
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, the FP64 tensor pipe of sm_100a).
// The accumulators start at zero; the C-in tile (a gather through the panel
// permutation, supplied by the epilogue functor) is fetched with cp.async into a
// shared-memory tile together with the LAST operand stage, so its latency hides
// behind the remaining MMAs.  The epilogue adds the accumulators into that tile and
// writes it back column-wise (coalesced).
#pragma once
#include "rcp_common.cuh"

namespace rcp {

constexpr int kGemmThreads = 256;  // 8 warps: 2 (M) x 4 (N)
constexpr int kBK = 16;
constexpr int kPad = 4;            // operand smem row stride BK+4 doubles -> conflict-free fragment loads
constexpr int kCPad = 1;           // C tile column stride BM+1 doubles (conflict-free row and column reads)

struct OperandDesc {
  const double* ptr;
  int64_t ld;    // elements between consecutive rows
  int64_t rows;  // valid rows (others read as 0)
  int64_t k;     // valid K (others read as 0)
};

template <int BM, int BN, int STAGES>
struct GemmSmem {
  double a[STAGES][BM][kBK + kPad];
  double b[STAGES][BN][kBK + kPad];
  double c[BN][BM + kCPad];
  int rowmap[BM];  // epilogue index maps (e.g. physical rows of the permuted C-in)
  int colmap[BN];
};

template <int ROWS, int VEC>
RCP_D void load_tile(double (*dst)[kBK + kPad], const OperandDesc& op, int64_t row0, int64_t k0) {
  constexpr int kChunksPerRow = kBK / VEC;
  constexpr int kChunks = ROWS * kChunksPerRow;
#pragma unroll
  for (int c = threadIdx.x; c < kChunks; c += kGemmThreads) {
    int r = c / kChunksPerRow;
    int kk = (c % kChunksPerRow) * VEC;
    int64_t gr = row0 + r, gk = k0 + kk;
    bool ok = (gr < op.rows) && (gk + VEC <= op.k);
    const double* src = ok ? (op.ptr + gr * op.ld + gk) : op.ptr;
    if (VEC == 2) {
      cp_async16(&dst[r][kk], src, ok);
    } else {
      cp_async8(&dst[r][kk], src, ok);
    }
  }
}

// C-in gather: element (m0+i, n0+j) -> smem c[j][i]; threads run along i (coalesced).
template <int BM, int BN, class Epi>
RCP_D void load_cin(double (*c)[BM + kCPad], const int* rowmap, const int* colmap, const Epi& epi, int64_t m0,
                    int64_t n0) {
  for (int e = threadIdx.x; e < BM * BN; e += kGemmThreads) {
    const int j = e / BM, i = e - j * BM;
    const double* src = epi.cin(m0 + i, n0 + j, rowmap[i], colmap[j]);
    cp_async8(&c[j][i], src ? src : epi.dummy(), src != nullptr);
  }
}

// Generic tile-GEMM body.  TileMap: bool map(int bid, int64_t& m0, int64_t& n0).
// Epi: int map_row(m), int map_col(n) (staged once per tile), const double* cin(m, n, row, col)
//      (nullptr -> 0), double* cout(m, n) (nullptr -> skip), const double* dummy(),
//      static constexpr bool kHasInput.
template <int BM, int BN, int STAGES, int VEC, class TileMap, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
dmma_gemm_kernel(OperandDesc A, OperandDesc B, int64_t K, TileMap map, Epi epi) {
  constexpr int WM = BM / 2, WN = BN / 4;
  constexpr int MF = WM / 8, NF = WN / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<GemmSmem<BM, BN, STAGES>*>(smem_raw);
  if (!epi.prepare(map, K, B)) return;  // device-side dimensions (no-op for most epilogues)

  int64_t m0, n0;
  if (!map(blockIdx.x, m0, n0)) return;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int wm0 = (warp >> 2) * WM, wn0 = (warp & 3) * WN;

  double acc[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      acc[i][j][0] = 0.0;
      acc[i][j][1] = 0.0;
    }

  if (Epi::kHasInput) {
    for (int i = threadIdx.x; i < BM; i += kGemmThreads) sm.rowmap[i] = epi.map_row(m0 + i);
    for (int j = threadIdx.x; j < BN; j += kGemmThreads) sm.colmap[j] = epi.map_col(n0 + j);
    __syncthreads();
  }
  const int KT = static_cast<int>((K + kBK - 1) / kBK);
  // prologue: STAGES-1 operand stages; the C-in gather joins the group of the last stage
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      load_tile<BM, VEC>(sm.a[s], A, m0, (int64_t)s * kBK);
      load_tile<BN, VEC>(sm.b[s], B, n0, (int64_t)s * kBK);
    }
    if (Epi::kHasInput && s == STAGES - 2 && KT <= STAGES - 1) load_cin<BM, BN>(sm.c, sm.rowmap, sm.colmap, epi, m0, n0);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) {
        int st = nk % STAGES;
        load_tile<BM, VEC>(sm.a[st], A, m0, (int64_t)nk * kBK);
        load_tile<BN, VEC>(sm.b[st], B, n0, (int64_t)nk * kBK);
        if (Epi::kHasInput && nk == KT - 1) load_cin<BM, BN>(sm.c, sm.rowmap, sm.colmap, epi, m0, n0);
      }
      cp_async_commit();
    }
    const int st = kt % STAGES;
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      double af[MF], bf[NF];
#pragma unroll
      for (int i = 0; i < MF; ++i) af[i] = sm.a[st][wm0 + 8 * i + g][kk + q];
#pragma unroll
      for (int j = 0; j < NF; ++j) bf[j] = sm.b[st][wn0 + 8 * j + g][kk + q];
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  if (Epi::kHasInput && KT == 0) load_cin<BM, BN>(sm.c, sm.rowmap, sm.colmap, epi, m0, n0), cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // accumulate into the C tile (c[n][m]), then coalesced column-wise store
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int mi = wm0 + 8 * i + g;
      const int nj = wn0 + 8 * j + 2 * q;
      if (Epi::kHasInput) {
        sm.c[nj][mi] = __dadd_rn(sm.c[nj][mi], acc[i][j][0]);
        sm.c[nj + 1][mi] = __dadd_rn(sm.c[nj + 1][mi], acc[i][j][1]);
      } else {
        sm.c[nj][mi] = acc[i][j][0];
        sm.c[nj + 1][mi] = acc[i][j][1];
      }
    }
  __syncthreads();
  for (int e = threadIdx.x; e < BM * BN; e += kGemmThreads) {
    const int j = e / BM, i = e - j * BM;
    double* dst = epi.cout(m0 + i, n0 + j);
    if (dst) *dst = sm.c[j][i];
  }
  if (Epi::kMirror) {  // also store the transpose of the strictly-lower part (symmetric full storage)
    for (int e = threadIdx.x; e < BM * BN; e += kGemmThreads) {
      const int i = e / BN, j = e - i * BN;
      double* dst = epi.cout_mirror(m0 + i, n0 + j);
      if (dst) *dst = sm.c[j][i];
    }
  }
}

template <int BM, int BN, int STAGES>
constexpr size_t gemm_smem_bytes() {
  return sizeof(GemmSmem<BM, BN, STAGES>);
}

// ------------------------------------------------------------------ tile maps
struct RectMap {
  int64_t tiles_n;  // tiles along N
  int bm, bn;
  RCP_D bool operator()(int bid, int64_t& m0, int64_t& n0) const {
    int64_t tm = bid / tiles_n, tn = bid % tiles_n;
    m0 = tm * bm;
    n0 = tn * bn;
    return true;
  }
};

// Column-major tile enumeration (bid -> tm = bid % tiles_m, tn = bid / tiles_m); tiles with
// tn >= tiles_n (which an epilogue may lower on the device) are skipped.
struct ColMajorRectMap {
  int64_t tiles_n;
  int64_t tiles_m;
  int bm, bn;
  RCP_D bool operator()(int bid, int64_t& m0, int64_t& n0) const {
    const int64_t tm = bid % tiles_m, tn = bid / tiles_m;
    m0 = tm * bm;
    n0 = tn * bn;
    return tn < tiles_n;
  }
};

// Lower-triangular enumeration of square tiles (I >= J), bid -> (I, J).
struct LowerMap {
  int bt;  // tile size (BM == BN)
  RCP_D bool operator()(int bid, int64_t& m0, int64_t& n0) const {
    long long x = bid;
    long long I = static_cast<long long>((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);
    while (I * (I + 1) / 2 > x) --I;
    while ((I + 1) * (I + 2) / 2 <= x) ++I;
    long long J = x - I * (I + 1) / 2;
    m0 = I * bt;
    n0 = J * bt;
    return true;
  }
};

}  // namespace rcp
