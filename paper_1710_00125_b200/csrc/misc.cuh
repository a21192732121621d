// Launchers of the bandwidth-bound helper kernels (misc.cu) and GEMMs (schur.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rcp {

struct PanelDesc;
struct SchurDyn;

cudaError_t launch_validate_copy(const double* a, int64_t lda, int64_t n, double* out, int* flags, double* amax,
                                 cudaStream_t st, int half = 0);
cudaError_t launch_tstamp_init(unsigned long long* ts, int64_t count, cudaStream_t st);
cudaError_t launch_sketch_norm_max(const double* B, int P, int64_t ncols, double* out, cudaStream_t st);
cudaError_t launch_gather(int64_t n, int k0, int k_end, int t, int tpad, int64_t rows_pad, const int* phys_of_log,
                          const double* Lbuf, const double* W, const int* perm_cur, int* perm_next, int* snap,
                          int* phys, double* Lneg, double* Wg, double* L11, cudaStream_t st,
                          const PanelDesc* d = nullptr, double* lorig = nullptr);
cudaError_t launch_finalize_rows(int64_t n, int64_t ra, int64_t rb, int64_t kp, int t, const int64_t* perm,
                                 const double* lorig, const double* L11T, double* L, double* maxmult,
                                 int max_rows, cudaStream_t st, const PanelDesc* d = nullptr);
cudaError_t launch_ysolve(int64_t n, int P, int k0, int t, int tpad, const int* phys_of_log, const double* Bin,
                          const double* L11, double* Y, cudaStream_t st, const PanelDesc* d = nullptr);
cudaError_t launch_assemble_panel(int64_t n, int k0, int k_end, const int* snap, int* pos_of_orig,
                                  const int64_t* perm, const double* Lbuf, double* L, double* maxmult,
                                  cudaStream_t st);
cudaError_t launch_unit_diag(int64_t n, double* L, cudaStream_t st);
cudaError_t launch_dmax(int64_t n, const double* dd, const double* doff, double* out, cudaStream_t st);
cudaError_t launch_deficient_fill(int64_t n, int64_t k0, const int* perm_cur, int64_t* perm_out, double* dd,
                                  double* doff, int8_t* pattern, cudaStream_t st);
cudaError_t launch_mirror_lower(int64_t n, int64_t k, double* A, cudaStream_t st);
cudaError_t launch_iota(int64_t n, int* p, cudaStream_t st);

// ---- experiment diagnostics (diag.cu): track_growth="full" snapshots and the audit_sketch drift
cudaError_t launch_snapshot(int64_t n, const double* A, const PanelDesc* d, double* out, cudaStream_t st);
cudaError_t launch_drift(int64_t n, int P, const double* A, const double* B, const double* omega_orig,
                         const int* perm, const PanelDesc* d, double* out, cudaStream_t st);
cudaError_t launch_omega_scatter(int64_t n, int P, int64_t k0, const double* om, int64_t m, const int* perm,
                                 double* omega_orig, cudaStream_t st);

// ---- FP64 tensor-core GEMMs (schur.cu)
// A_out[k+i, k+j] = A_in(phys[i], phys[j]) - sum_s L[i,s] W[j,s]   for i >= j (lower tiles)
cudaError_t launch_schur_update(int64_t n, int64_t k, int64_t mp, const double* Lneg, const double* Wg, int tpad,
                                int K, const double* A_in, const int* phys, double* A_out, cudaStream_t st,
                                const PanelDesc* d = nullptr, int part = 0, int nparts = 1,
                                const double* ysk = nullptr, const double* bin = nullptr, double* bout = nullptr,
                                int P = 0, unsigned long long* tstamp = nullptr);
// multi-GPU worker: buffers / panel outcome resolved on the device (dist.cuh)
cudaError_t launch_schur_update_dyn(int64_t n, const double* Lneg, const double* Wg, int tpad, const int* phys,
                                    const SchurDyn* dyn, int part, int nparts, cudaStream_t st);
// B[:, col0 + j] = sum_i Omega[r, i] * A[i, j]   (Omega row-major P x m, A col-major ld lda, full columns)
cudaError_t launch_sketch_gemm(int P, int64_t m, const double* omega, int64_t ldo, const double* A, int64_t lda,
                               double* B, int64_t col0, cudaStream_t st);
// B_out[:, k+j] = B_in[:, phys[j]] - Y * L[j,:]^T  (Y row-major P x tpad; Lneg = -L rows)
cudaError_t launch_sketch_correction(int P, int64_t mp, int64_t k, const double* Y, int tpad, int K,
                                     const double* Lneg, const double* B_in, const int* phys, double* B_out,
                                     cudaStream_t st, const PanelDesc* d = nullptr, int64_t n = 0);
cudaError_t gemm_init_attributes();

}  // namespace rcp
