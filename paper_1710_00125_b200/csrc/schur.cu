// FP64 DMMA GEMM instantiations: trailing Schur update (lower tiles, gather-fused),
// sketch projection and sketch correction.
#include "gemm_dmma.cuh"
#include "misc.cuh"

namespace rcp {

namespace {

// A22 <- A22 - L21 W21^T on the lower triangle, reading the previous matrix through the
// panel permutation (factor.py:369-379 + core.py:115-119: the stored value of (i, j),
// i > j, is the lower-computed one).
struct SchurEpi {
  static constexpr bool kNeedInit = true;
  const double* ain;
  double* aout;
  const int* phys;
  int64_t n, k, mp;
  RCP_D double init(int64_t i, int64_t j) const {
    if (i >= mp || j >= mp || i < j) return 0.0;
    return sym_lower(ain, n, phys[i], phys[j]);
  }
  RCP_D void store(int64_t i, int64_t j, double v) const {
    if (i < mp && j < mp && i >= j) aout[(k + i) + (k + j) * n] = v;
  }
};

struct SketchEpi {
  static constexpr bool kNeedInit = false;
  double* b;
  int64_t P, ncols, col0;
  RCP_D double init(int64_t, int64_t) const { return 0.0; }
  RCP_D void store(int64_t r, int64_t j, double v) const {
    if (r < P && j < ncols) b[r + (col0 + j) * P] = v;
  }
};

struct SketchCorrEpi {
  static constexpr bool kNeedInit = true;
  const double* bin;
  double* bout;
  const int* phys;
  int64_t P, mp, k;
  RCP_D double init(int64_t r, int64_t j) const {
    return (r < P && j < mp) ? bin[r + (int64_t)phys[j] * P] : 0.0;
  }
  RCP_D void store(int64_t r, int64_t j, double v) const {
    if (r < P && j < mp) bout[r + (k + j) * P] = v;
  }
};

template <int BM, int BN>
constexpr size_t smem_bytes() {
  return sizeof(GemmSmem<BM, BN>);
}

bool aligned16(const void* p, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 2 == 0);
}

}  // namespace

cudaError_t gemm_init_attributes() {
  cudaError_t e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<128, 128, 2, LowerMap, SchurEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<128, 128>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<64, 128, 2, RectMap, SketchEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<64, 128>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<64, 128, 1, RectMap, SketchEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<64, 128>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<64, 128, 2, RectMap, SketchCorrEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<64, 128>());
  return e;
}

cudaError_t launch_schur_update(int64_t n, int64_t k, int64_t mp, const double* Lneg, const double* Wg, int tpad,
                                int K, const double* A_in, const int* phys, double* A_out, cudaStream_t st) {
  if (mp <= 0 || K <= 0) return cudaSuccess;
  const int64_t nb = (mp + 127) / 128;
  const int64_t tiles = nb * (nb + 1) / 2;
  // operands are zero padded to tpad (a multiple of kBK) along K
  const int Kl = ((K + kBK - 1) / kBK) * kBK;
  OperandDesc a{Lneg, tpad, mp, tpad};
  OperandDesc b{Wg, tpad, mp, tpad};
  SchurEpi epi{A_in, A_out, phys, n, k, mp};
  dmma_gemm_kernel<128, 128, 2, LowerMap, SchurEpi>
      <<<(unsigned)tiles, kGemmThreads, smem_bytes<128, 128>(), st>>>(a, b, Kl, LowerMap{128}, epi);
  return cudaGetLastError();
}

cudaError_t launch_sketch_gemm(int P, int64_t m, const double* omega, int64_t ldo, const double* A, int64_t lda,
                               double* B, int64_t col0, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  const int64_t tm = (P + 63) / 64, tn = (m + 127) / 128;
  OperandDesc a{omega, ldo, P, m};
  OperandDesc b{A, lda, m, m};
  SketchEpi epi{B, P, m, col0};
  RectMap map{tn, 64, 128};
  if (aligned16(omega, ldo) && aligned16(A, lda) && (m % 2 == 0)) {
    dmma_gemm_kernel<64, 128, 2, RectMap, SketchEpi>
        <<<(unsigned)(tm * tn), kGemmThreads, smem_bytes<64, 128>(), st>>>(a, b, m, map, epi);
  } else {
    dmma_gemm_kernel<64, 128, 1, RectMap, SketchEpi>
        <<<(unsigned)(tm * tn), kGemmThreads, smem_bytes<64, 128>(), st>>>(a, b, m, map, epi);
  }
  return cudaGetLastError();
}

cudaError_t launch_sketch_correction(int P, int64_t mp, int64_t k, const double* Y, int tpad, int K,
                                     const double* Lneg, const double* B_in, const int* phys, double* B_out,
                                     cudaStream_t st) {
  if (mp <= 0 || K <= 0) return cudaSuccess;
  const int64_t tm = (P + 63) / 64, tn = (mp + 127) / 128;
  const int Kl = ((K + kBK - 1) / kBK) * kBK;
  OperandDesc a{Y, tpad, P, tpad};
  OperandDesc b{Lneg, tpad, mp, tpad};
  SketchCorrEpi epi{B_in, B_out, phys, P, mp, k};
  RectMap map{tn, 64, 128};
  dmma_gemm_kernel<64, 128, 2, RectMap, SketchCorrEpi>
      <<<(unsigned)(tm * tn), kGemmThreads, smem_bytes<64, 128>(), st>>>(a, b, Kl, map, epi);
  return cudaGetLastError();
}

}  // namespace rcp
