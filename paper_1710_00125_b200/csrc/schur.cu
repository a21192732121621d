// FP64 DMMA GEMM instantiations: trailing Schur update (lower tiles, gather-fused),
// sketch projection and sketch correction.
#include "gemm_dmma.cuh"
#include "misc.cuh"
#include "schur_ws.cuh"
#include "schur_ws2.cuh"
#include <cstdlib>
#include <algorithm>
#include <type_traits>

namespace rcp {

namespace {

struct SketchEpi {
  static constexpr bool kHasInput = false;
  static constexpr bool kMirror = false;
  template <class Map>
  RCP_D bool prepare(Map&, int64_t&, OperandDesc&) { return true; }
  RCP_D double* cout_mirror(int64_t, int64_t) const { return nullptr; }
  double* b;
  int64_t P, ncols, col0;
  RCP_D int map_row(int64_t) const { return 0; }
  RCP_D int map_col(int64_t) const { return 0; }
  RCP_D const double* dummy() const { return b; }
  RCP_D const double* cin(int64_t, int64_t, int, int) const { return nullptr; }
  RCP_D double* cout(int64_t r, int64_t j) const { return (r < P && j < ncols) ? b + r + (col0 + j) * P : nullptr; }
};

struct SketchCorrEpi {
  static constexpr bool kHasInput = true;
  static constexpr bool kMirror = false;
  // device-driven: mp / k / K / tile count from the committed panel descriptor
  const PanelDesc* d;
  int64_t n;
  template <class Map>
  RCP_D bool prepare(Map& map, int64_t& K, OperandDesc& B) {
    if (!d) return true;
    if (!d->ok || d->t <= 0 || d->k_end >= n) return false;
    k = d->k_end;
    mp = n - k;
    K = ((d->t + kBK - 1) / kBK) * kBK;
    B.rows = mp;
    map.tiles_n = (mp + map.bn - 1) / map.bn;
    return true;
  }
  RCP_D double* cout_mirror(int64_t, int64_t) const { return nullptr; }
  const double* bin;
  double* bout;
  const int* phys;
  int64_t P, mp, k;
  RCP_D int map_row(int64_t) const { return 0; }
  RCP_D int map_col(int64_t j) const { return j < mp ? phys[j] : -1; }
  RCP_D const double* dummy() const { return bin; }
  RCP_D const double* cin(int64_t r, int64_t j, int, int pj) const {
    return (r < P && j < mp) ? bin + r + (int64_t)pj * P : nullptr;
  }
  RCP_D double* cout(int64_t r, int64_t j) const { return (r < P && j < mp) ? bout + r + (k + j) * P : nullptr; }
};

constexpr int kRectStages = 3;

// Single-GPU trailing update kernel: 2 = schur_ws2_kernel (two MMA warps per sub-partition,
// default), 1 = schur_ws_kernel.  RCP_SCHUR_V=1 selects the first generation (A/B runs).
int schur_version() {
  static const int v = [] {
    const char* e = std::getenv("RCP_SCHUR_V");
    return (e && e[0] == '1') ? 1 : 2;
  }();
  return v;
}

// L2 cache-policy hints in schur_ws2_kernel: RCP_SCHUR_HINTS = 0 none, 1 (default) operand panels
// evict_last, 2 also C-in / C-out evict_first.
int schur_hints() {
  static const int v = [] {
    const char* e = std::getenv("RCP_SCHUR_HINTS");
    return (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 1;
  }();
  return v;
}
// TMA operand staging in schur_ws2_kernel (RCP_SCHUR_TMA=0: cp.async producer warps instead).
bool schur_tma_requested() {
  static const bool v = [] {
    const char* e = std::getenv("RCP_SCHUR_TMA");
    return !(e && e[0] == '0');
  }();
  return v;
}
using Ws2Kernel = decltype(&schur_ws2_kernel<0, false, false>);
template <bool kTma, bool kMulti>
Ws2Kernel ws2_pick(int h) {
  return h == 2 ? schur_ws2_kernel<2, kTma, kMulti> : (h == 1 ? schur_ws2_kernel<1, kTma, kMulti> : schur_ws2_kernel<0, kTma, kMulti>);
}
Ws2Kernel ws2_kernel(bool tma, bool multi) {
  const int h = schur_hints();
  if (multi) return tma ? ws2_pick<true, true>(h) : ws2_pick<false, true>(h);
  return tma ? ws2_pick<true, false>(h) : ws2_pick<false, false>(h);
}

// Tensor maps of the operand panels: a K-contiguous [rows][tpad] fp64 array viewed as
// {4, rows, tpad / 4} with box {4, 128, 4} (see tma_load_3d).  Encoded through the driver entry
// point (no link against libcuda) and cached per thread: the panels of one factorization keep
// their addresses.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
struct OperandMap {
  const void* ptr = nullptr;
  int64_t rows = 0;
  int tpad = 0;
  bool ok = false;
  CUtensorMap tm;
};
// Returns nullptr when the panel cannot be described (the caller then uses the cp.async kernel).
const CUtensorMap* operand_map(const double* ptr, int64_t rows, int tpad) {
  thread_local OperandMap cache[16];  // rank 0's three panels + the emulated workers' copies
  thread_local int next = 0;
  for (auto& c : cache)
    if (c.ptr == ptr && c.rows == rows && c.tpad == tpad) return c.ok ? &c.tm : nullptr;
  OperandMap& c = cache[next];
  next = (next + 1) % 16;
  c.ptr = ptr;
  c.rows = rows;
  c.tpad = tpad;
  c.ok = false;
  EncodeTiledFn enc = encode_tiled();
  if (enc && ptr && rows > 0 && tpad % 4 == 0 && reinterpret_cast<uintptr_t>(ptr) % 16 == 0) {
    const cuuint64_t dims[3] = {4, (cuuint64_t)rows, (cuuint64_t)(tpad / 4)};
    const cuuint64_t strides[2] = {(cuuint64_t)tpad * 8, 32};
    const cuuint32_t box[3] = {4, (cuuint32_t)ws::BM, (cuuint32_t)(ws2::KS / 4)};
    const cuuint32_t es[3] = {1, 1, 1};
    c.ok = enc(&c.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  return c.ok ? &c.tm : nullptr;
}

// One schur_ws2_kernel launch (TMA when the three operand maps exist, else cp.async).
cudaError_t launch_ws2(unsigned grid, cudaStream_t st, const double* Lneg, const double* Wg, int tpad, int Kl,
                       const double* A_in, double* A_out, const int* phys, int64_t n, int64_t k, int64_t mp,
                       const PanelDesc* d, const double* ysk, const double* bin, double* bout, int P,
                       unsigned long long* tstamp, int part = 0, int nparts = 1, const SchurDyn* dyn = nullptr) {
  const int64_t rows_pad = ((n + ws::BM - 1) / ws::BM) * ws::BM;  // layout.cuh: rows of Lneg / Wg
  const CUtensorMap* ta = nullptr;
  const CUtensorMap* tb = nullptr;
  const CUtensorMap* ty = nullptr;
  if (schur_tma_requested()) {
    ta = operand_map(Lneg, rows_pad, tpad);
    tb = operand_map(Wg, rows_pad, tpad);
    ty = ysk ? operand_map(ysk, P, tpad) : tb;
  }
  const bool tma = ta && tb && ty;
  static const CUtensorMap none{};
  ws2_kernel(tma, nparts > 1)<<<grid, ws2::kThreads, schur_ws2_smem_bytes(), st>>>(
      tma ? *ta : none, tma ? *tb : none, tma ? *ty : none, Lneg, Wg, tpad, Kl, A_in, A_out, phys, n, k, mp, d, ysk, bin,
      bout, P, tstamp, part, nparts, dyn);
  return cudaGetLastError();
}

bool aligned16(const void* p, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 2 == 0);
}

}  // namespace

cudaError_t gemm_init_attributes() {
  cudaError_t e;
  e = cudaFuncSetAttribute(schur_ws_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)schur_ws_smem_bytes());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(schur_ws_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)schur_ws_smem_bytes());
  if (e != cudaSuccess) return e;
  for (int h = 0; h < 3; ++h)
    for (Ws2Kernel f : {ws2_pick<false, false>(h), ws2_pick<true, false>(h), ws2_pick<false, true>(h),
                        ws2_pick<true, true>(h)}) {
      e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)schur_ws2_smem_bytes());
      if (e != cudaSuccess) return e;
    }
  e = cudaFuncSetAttribute(dmma_gemm_kernel<64, 128, kRectStages, 2, RectMap, SketchEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes<64, 128, kRectStages>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<64, 128, kRectStages, 1, RectMap, SketchEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes<64, 128, kRectStages>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<64, 128, kRectStages, 2, ColMajorRectMap, SketchCorrEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes<64, 128, kRectStages>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<48, 64, kRectStages, 2, ColMajorRectMap, SketchCorrEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes<48, 64, kRectStages>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<96, 64, kRectStages, 2, ColMajorRectMap, SketchCorrEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes<96, 64, kRectStages>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dmma_gemm_kernel<144, 64, kRectStages, 2, ColMajorRectMap, SketchCorrEpi>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes<144, 64, kRectStages>());
  return e;
}

cudaError_t launch_schur_update(int64_t n, int64_t k, int64_t mp, const double* Lneg, const double* Wg, int tpad,
                                int K, const double* A_in, const int* phys, double* A_out, cudaStream_t st,
                                const PanelDesc* d, int part, int nparts, const double* ysk, const double* bin,
                                double* bout, int P, unsigned long long* tstamp) {
  if (d) {  // persistent grid; the kernel reads the panel outcome
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // experiment knob: RCP_SCHUR_SMS runs the update on a partition of the SMs
    static const int sms_env = [] {
      const char* e = std::getenv("RCP_SCHUR_SMS");
      return e ? std::atoi(e) : 0;
    }();
    if (sms_env >= 1 && sms_env < sms) sms = sms_env;
    if (schur_version() == 2)  // nparts > 1: rank 0's share, no fused sketch tiles
      return launch_ws2((unsigned)sms, st, Lneg, Wg, tpad, 0, A_in, A_out, phys, n, 0, 0, d,
                        nparts > 1 ? nullptr : ysk, bin, bout, P, tstamp, part, nparts, nullptr);
    if (nparts > 1)
      schur_ws_kernel<true><<<(unsigned)sms, ws::kThreads, schur_ws_smem_bytes(), st>>>(
          Lneg, Wg, tpad, 0, A_in, A_out, phys, n, 0, 0, 0, d, part, nparts, nullptr, nullptr, nullptr, nullptr, 0,
          tstamp);
    else
      schur_ws_kernel<false><<<(unsigned)sms, ws::kThreads, schur_ws_smem_bytes(), st>>>(
          Lneg, Wg, tpad, 0, A_in, A_out, phys, n, 0, 0, 0, d, part, nparts, nullptr, ysk, bin, bout, P, tstamp);
    return cudaGetLastError();
  }
  if (mp <= 0 || K <= 0) return cudaSuccess;
  if (schur_version() == 2) {
    const int64_t nb2 = (mp + ws::BM - 1) / ws::BM;
    const long long supers = nb2 * (nb2 + 1) / 2;
    const int Kl2 = ((K + kBK - 1) / kBK) * kBK;
    int dev2 = 0, sms2 = 148;
    cudaGetDevice(&dev2);
    cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, dev2);
    return launch_ws2((unsigned)std::min<long long>(supers, sms2), st, Lneg, Wg, tpad, Kl2, A_in, A_out, phys, n, k, mp,
                      nullptr, nullptr, nullptr, nullptr, 0, nullptr);
  }
  const int64_t nbi = (mp + ws::BM - 1) / ws::BM;
  const long long tiles = nbi * (nbi + 1);  // row block I has 2I+2 column blocks of 64
  const int Kl = ((K + kBK - 1) / kBK) * kBK;  // operands are zero padded to tpad along K
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long grid = std::min<long long>(tiles, sms);
  schur_ws_kernel<false><<<(unsigned)grid, ws::kThreads, schur_ws_smem_bytes(), st>>>(Lneg, Wg, tpad, Kl, A_in, A_out, phys,
                                                                               n, k, mp, tiles, nullptr, 0, 1, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_schur_update_dyn(int64_t n, const double* Lneg, const double* Wg, int tpad, const int* phys,
                                    const SchurDyn* dyn, int part, int nparts, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (schur_version() == 2)
    return launch_ws2((unsigned)sms, st, Lneg, Wg, tpad, 0, nullptr, nullptr, phys, n, 0, 0, nullptr, nullptr, nullptr,
                      nullptr, 0, nullptr, part, nparts, dyn);
  schur_ws_kernel<true><<<(unsigned)sms, ws::kThreads, schur_ws_smem_bytes(), st>>>(
        Lneg, Wg, tpad, 0, nullptr, nullptr, phys, n, 0, 0, 0, nullptr, part, nparts, dyn);
  return cudaGetLastError();
}

cudaError_t launch_sketch_gemm(int P, int64_t m, const double* omega, int64_t ldo, const double* A, int64_t lda,
                               double* B, int64_t col0, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  OperandDesc a{omega, ldo, P, m};
  OperandDesc b{A, lda, m, m};
  SketchEpi epi{B, P, m, col0};
  if (P <= 144 && aligned16(omega, ldo) && aligned16(A, lda) && (m % 2 == 0)) {
    // one tile row over all P sketch rows (48 / 96 / 144), 64-column tiles: no padded MMA rows
    auto one_row = [&](auto bm_tag) -> cudaError_t {
      constexpr int BM = decltype(bm_tag)::value;
      const int64_t tn = (m + 63) / 64;
      RectMap map{tn, BM, 64};
      cudaError_t e = cudaFuncSetAttribute(dmma_gemm_kernel<BM, 64, kRectStages, 2, RectMap, SketchEpi>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)gemm_smem_bytes<BM, 64, kRectStages>());
      if (e != cudaSuccess) return e;
      dmma_gemm_kernel<BM, 64, kRectStages, 2, RectMap, SketchEpi>
          <<<(unsigned)tn, kGemmThreads, gemm_smem_bytes<BM, 64, kRectStages>(), st>>>(a, b, m, map, epi);
      return cudaGetLastError();
    };
    if (P <= 48) return one_row(std::integral_constant<int, 48>{});
    if (P <= 96) return one_row(std::integral_constant<int, 96>{});
    return one_row(std::integral_constant<int, 144>{});
  }
  const int64_t tm = (P + 63) / 64, tn = (m + 127) / 128;
  RectMap map{tn, 64, 128};
  const size_t smem = gemm_smem_bytes<64, 128, kRectStages>();
  if (aligned16(omega, ldo) && aligned16(A, lda) && (m % 2 == 0)) {
    dmma_gemm_kernel<64, 128, kRectStages, 2, RectMap, SketchEpi>
        <<<(unsigned)(tm * tn), kGemmThreads, smem, st>>>(a, b, m, map, epi);
  } else {
    dmma_gemm_kernel<64, 128, kRectStages, 1, RectMap, SketchEpi>
        <<<(unsigned)(tm * tn), kGemmThreads, smem, st>>>(a, b, m, map, epi);
  }
  return cudaGetLastError();
}

cudaError_t launch_sketch_correction(int P, int64_t mp, int64_t k, const double* Y, int tpad, int K,
                                     const double* Lneg, const double* B_in, const int* phys, double* B_out,
                                     cudaStream_t st, const PanelDesc* d, int64_t n) {
  // with d: mp / k / K are upper bounds for the grid; the kernel reads the actual values
  if (mp <= 0 || K <= 0) return cudaSuccess;
  const int Kl = ((K + kBK - 1) / kBK) * kBK;
  OperandDesc a{Y, tpad, P, tpad};
  OperandDesc b{Lneg, tpad, mp, tpad};
  SketchCorrEpi epi{d, n, B_in, B_out, phys, P, mp, k};
  // one tile row covering all P sketch rows when P <= 144 (no padded MMA rows beyond a multiple
  // of 48); 64-wide column tiles.  SketchCorrEpi::prepare rescales tiles_n for N = 64 below.
  auto one_row = [&](auto bm_tag) -> cudaError_t {
    constexpr int BM = decltype(bm_tag)::value;
    const int64_t tn = (mp + 63) / 64;
    ColMajorRectMap map{tn, 1, BM, 64};
    dmma_gemm_kernel<BM, 64, kRectStages, 2, ColMajorRectMap, SketchCorrEpi>
        <<<(unsigned)tn, kGemmThreads, gemm_smem_bytes<BM, 64, kRectStages>(), st>>>(a, b, Kl, map, epi);
    return cudaGetLastError();
  };
  if (P <= 48) return one_row(std::integral_constant<int, 48>{});
  if (P <= 96) return one_row(std::integral_constant<int, 96>{});
  if (P <= 144) return one_row(std::integral_constant<int, 144>{});
  const int64_t tm = (P + 63) / 64, tn = (mp + 127) / 128;
  ColMajorRectMap map{tn, tm, 64, 128};
  dmma_gemm_kernel<64, 128, kRectStages, 2, ColMajorRectMap, SketchCorrEpi>
      <<<(unsigned)(tm * tn), kGemmThreads, gemm_smem_bytes<64, 128, kRectStages>(), st>>>(a, b, Kl, map, epi);
  return cudaGetLastError();
}

}  // namespace rcp

extern "C" int64_t rcp_schur_tile_plan(int64_t mp, int32_t P, int32_t part, int32_t nparts, int32_t grid,
                                       int64_t* m0, int64_t* n0, int8_t* sketch, int64_t cap) {
  using namespace rcp;
  if (mp < 1 || P < 0 || nparts < 1 || part < 0 || part >= nparts || grid < 1) return -1;
  const long long nbi = (mp + ws::BM - 1) / ws::BM;
  const long long tiles_tri = nbi * (nbi + 1);
  const int nbp = P > 0 ? (P + ws::BN - 1) / ws::BN : 0;
  const long long tiles = tiles_tri + nbi * nbp;
  int64_t cnt = 0;
  auto emit = [&](int64_t a, int64_t b, bool sk) {
    if (cnt < cap) {
      if (m0) m0[cnt] = a;
      if (n0) n0[cnt] = b;
      if (sketch) sketch[cnt] = sk ? 1 : 0;
    }
    ++cnt;
  };
  if (schur_version() == 2) {  // schur_ws2_kernel: supertiles = two 128x64 tiles each
    const int nbp2 = P > 0 ? (P + ws2::SN - 1) / ws2::SN : 0;
    const long long s_tri = nbi * (nbi + 1) / 2, s_all = s_tri + nbi * nbp2;
    for (int cta = 0; cta < grid; ++cta) {
      long long x0, xs;
      ws2::super_sequence(nparts > 1, part, nparts, cta, grid, x0, xs);
      for (long long x = x0; x < s_all; x += xs) {
        int64_t a, b;
        const bool sk = ws2::super_at(x, s_tri, nbp2, a, b);
        for (int h = 0; h < 2; ++h)  // halves beyond the last sketch row are loaded as zeros and never stored
          if (!sk || b + h * ws::BN < P) emit(a, b + h * ws::BN, sk);
      }
    }
    return cnt;
  }
  for (int cta = 0; cta < grid; ++cta) {
    long long x0, xs;
    ws::tile_sequence(nparts > 1, part, nparts, cta, grid, x0, xs);
    for (long long x = x0; x < tiles; x += xs) {
      int64_t a, b;
      const bool sk = ws::tile_at(x, tiles_tri, nbp, a, b);
      emit(a, b, sk);
    }
  }
  return cnt;
}

