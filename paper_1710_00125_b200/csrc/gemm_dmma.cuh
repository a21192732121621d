// FP64 tensor-core GEMM core for the dense contractions of the RCP path:
//   - trailing Schur update   A22 <- A22 - L21 * W21^T   (lower tiles only, permuted gather-in)
//   - sketch                  B   <- Omega * A
//   - sketch correction       B2  <- B2 - Y * L21^T      (permuted gather-in)
//
// acc[m][n] = init(m, n) + sum_k Aop[m][k] * Bop[n][k]
// Both operands are K-contiguous row arrays (row r at base + r * ld).  Tiles are staged
// into shared memory with a cp.async ring (STAGES deep) and consumed by
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, the FP64 tensor pipe of sm_100a).  Epilogue
// functors provide the accumulator initialisation (gather of the previous matrix) and
// the store, so the permutation and the symmetric "lower only" rule are fused into
// the GEMM instead of separate passes.
#pragma once
#include "rcp_common.cuh"

namespace rcp {

constexpr int kGemmThreads = 256;  // 8 warps: 2 (M) x 4 (N)
constexpr int kBK = 16;
constexpr int kPad = 4;            // smem row stride BK+4 doubles -> conflict-free fragment loads
constexpr int kStages = 3;

struct OperandDesc {
  const double* ptr;
  int64_t ld;    // elements between consecutive rows
  int64_t rows;  // valid rows (others read as 0)
  int64_t k;     // valid K (others read as 0)
};

template <int BM, int BN>
struct GemmSmem {
  double a[kStages][BM][kBK + kPad];
  double b[kStages][BN][kBK + kPad];
};

template <int ROWS, int VEC>
RCP_D void load_tile(double (*dst)[kBK + kPad], const OperandDesc& op, int64_t row0, int64_t k0) {
  // ROWS x kBK tile; VEC doubles per cp.async (1 -> 8 B, 2 -> 16 B).
  constexpr int kChunksPerRow = kBK / VEC;
  constexpr int kChunks = ROWS * kChunksPerRow;
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

// Generic tile-GEMM body.  TileMap: bool map(int bid, int64_t& m0, int64_t& n0).
// Epi: double init(m, n, valid) / void store(m, n, v) / bool need_init.
template <int BM, int BN, int VEC, class TileMap, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
dmma_gemm_kernel(OperandDesc A, OperandDesc B, int64_t K, TileMap map, Epi epi) {
  constexpr int WM = BM / 2, WN = BN / 4;
  constexpr int MF = WM / 8, NF = WN / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<GemmSmem<BM, BN>*>(smem_raw);

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
      if (Epi::kNeedInit) {
        int64_t m = m0 + wm0 + 8 * i + g;
        int64_t n = n0 + wn0 + 8 * j + 2 * q;
        acc[i][j][0] = epi.init(m, n);
        acc[i][j][1] = epi.init(m, n + 1);
      } else {
        acc[i][j][0] = 0.0;
        acc[i][j][1] = 0.0;
      }
    }

  const int KT = static_cast<int>((K + kBK - 1) / kBK);
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < KT) {
      load_tile<BM, VEC>(sm.a[s], A, m0, (int64_t)s * kBK);
      load_tile<BN, VEC>(sm.b[s], B, n0, (int64_t)s * kBK);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      int nk = kt + kStages - 1;
      if (nk < KT) {
        int st = nk % kStages;
        load_tile<BM, VEC>(sm.a[st], A, m0, (int64_t)nk * kBK);
        load_tile<BN, VEC>(sm.b[st], B, n0, (int64_t)nk * kBK);
      }
      cp_async_commit();
    }
    const int st = kt % kStages;
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
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      int64_t m = m0 + wm0 + 8 * i + g;
      int64_t n = n0 + wn0 + 8 * j + 2 * q;
      epi.store(m, n, acc[i][j][0]);
      epi.store(m, n + 1, acc[i][j][1]);
    }
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

// Lower-triangular enumeration of square tiles (I >= J), bid -> (I, J).
struct LowerMap {
  int bt;  // tile size (BM == BN)
  RCP_D bool operator()(int bid, int64_t& m0, int64_t& n0) const {
    // I = floor((sqrt(8 bid + 1) - 1) / 2), fixed up for rounding.
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
