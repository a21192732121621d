/*
 * rcp_b200.h — C ABI of the B200-native RCP block-LDL^T factor/solve.
 *
 * Drop-in boundary for the reference package `randldl` (pure Python; paths
 * below are relative to /root/reference/pkg/src/randldl/).  The reference has
 * no FFI; its public Python API is the boundary, and each entry point here
 * replaces one of those calls (see INTEGRATION.md for the ctypes binding a
 * maintainer adds to `randldl`):
 *
 *   rcp_factor          <- randldl.factor / factor_robust   (factor.py:637-660)
 *                          with strategy="rcp", q = b (panel QRCP preselect) or
 *                          q = 1 (per-step sketch pivot + per-step sketch downdate)
 *   rcp_solve           <- randldl.solve / solve_many        (solve.py:79-107)
 *   rcp_reconstruct     <- randldl.reconstruct               (factor.py:663-665)
 *   rcp_workspace_bytes    workspace query (no reference counterpart)
 *   rcp_factor_dist     <- randldl.factor on several GPUs of one node (config C3,
 *                          "1/2/4/8 GPU"): rank 0 owns the matrix and the panels,
 *                          the trailing update is dealt over all GPUs (rcp_schur_worker
 *                          on the other ranks) through NVLink peer memory
 *   rcp_factor_batched  <- a loop of randldl.factor over independent small
 *                          matrices sharing one FactorConfig (BASELINE config C5;
 *                          q = b, n <= 256): one CTA per matrix, no host round trip
 *   rcp_solve_batched   <- a loop of randldl.solve over those factorizations
 *
 * Conventions
 *  - All matrix pointers are DEVICE pointers to fp64 data.  The input matrix
 *    is dense, symmetric, n x n with leading dimension lda (row- and
 *    column-major coincide for a symmetric matrix).  It is never modified
 *    (factor.py:285 copies A).
 *  - Omega (the initial Gaussian sketch, p x n, row-major as numpy draws it,
 *    sketch.py:83-84) is supplied by the caller so both sides see identical
 *    bits.  Guard recomputes (factor.py:392-410) call `draw` to obtain the
 *    next p x m normals from the same advancing stream; a NULL `draw` turns a
 *    recompute into RCP_ERR_NEED_NORMALS.
 *  - Outputs: perm (int64[n]), L (fp64 n x n ROW-major, unit lower, final
 *    pivot order — the reference's dense L), d_diag/d_off (fp64[n]: the 1x1
 *    entries and the 2x2 blocks [[d_diag[k], d_off[k]], [d_off[k],
 *    d_diag[k+1]]] where pattern[k] == 1), pattern (int8[n], factor.py:94-97).
 *  - Every call is reentrant: caller-provided workspace, one CUDA stream,
 *    no global state.  Calls block until the result is on the device
 *    (the host drives one panel at a time).
 */
#ifndef RCP_B200_H
#define RCP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (0 = ok).  Python maps them to the reference's exceptions. */
enum {
  RCP_OK = 0,
  RCP_ERR_INVALID_ARG = 1,      /* bad config / sizes -> ValueError (factor.py:137-149)          */
  RCP_ERR_NOT_SYMMETRIC = 2,    /* -> ValueError "must be symmetric" (core.py:48-53)             */
  RCP_ERR_NONFINITE_INPUT = 3,  /* -> ValueError "contains NaN or Inf" (factor.py:280-281)        */
  RCP_ERR_NUMERICAL = 4,        /* -> NumericalError; kind/step in rcp_stats (factor.py:455-466) */
  RCP_ERR_NEED_NORMALS = 5,     /* guard recompute needed but no `draw` callback                  */
  RCP_ERR_CUDA = 6,             /* CUDA runtime failure; message in rcp_stats                     */
  RCP_ERR_WORKSPACE = 7,        /* workspace smaller than rcp_workspace_bytes()                   */
  RCP_ERR_UNSUPPORTED = 8       /* configuration beyond the on-chip panel capacity (message says) */
};

/* NumericalError kinds (factor.py:214, 222, 456, 464-466). */
enum {
  RCP_NUM_NONE = 0,
  RCP_NUM_ZERO_1X1 = 1,        /* "zero 1x1 pivot under a nonzero column"             */
  RCP_NUM_SINGULAR_2X2 = 2,    /* "singular 2x2 pivot block"                          */
  RCP_NUM_NONFINITE = 3,       /* "non-finite pivot data at step {k}"                 */
  RCP_NUM_DET_BOUND = 4        /* "2x2 block at step {k} violates its determinant bound" */
};

/* Pivoting strategy (reference Strategy, factor.py:104-113; pivot.py). */
enum {
  RCP_STRATEGY_RCP = 0,   /* randomized complete pivoting: sketch + SBKP rule (the BASELINE path) */
  RCP_STRATEGY_BKPP = 1,  /* Bunch-Kaufman partial pivoting (pivot.py:146-171), no sketch         */
  RCP_STRATEGY_BBK = 2    /* rook / bounded Bunch-Kaufman (pivot.py:189-218), no sketch           */
};

/* Mirror of the engine-relevant FactorConfig fields (factor.py:116-135).  Zero-initialised
 * trailing fields select the defaults (strategy rcp). */
typedef struct rcp_config {
  int32_t p;          /* sketch rows (reference FactorConfig.p)                */
  int32_t b;          /* panel width                                            */
  int32_t q;          /* 1 or b                                                 */
  int32_t robust_r;   /* recompute budget exponent; 0 disables the guard        */
  int32_t strategy;   /* RCP_STRATEGY_*                                         */
} rcp_config;

/* Mirror of GrowthStats' engine-produced fields (metrics.py:47-65, factor.py:514-527)
 * plus the run's structure. */
typedef struct rcp_stats {
  double rho_cheap;          /* max|D| / max|A|                                  */
  double max_multiplier;     /* max |tril(L, -1)|                                 */
  double amax;               /* max|A|                                            */
  double dmax;               /* max|D|                                            */
  int64_t recompute_count;   /* guard recomputes                                  */
  int64_t n_panels;
  int64_t n_steps;           /* pivot decisions taken                             */
  int64_t n_2x2;
  int64_t deficient_from;    /* first PAT_DEFICIENT index, -1 if none             */
  int32_t num_kind;          /* RCP_NUM_* when status == RCP_ERR_NUMERICAL        */
  int32_t num_step;          /* step k of the numerical error                     */
  double t_factor_ms;        /* device time of the factorization (CUDA events)    */
  double t_schur_ms;         /* device time inside the trailing Schur updates     */
  double t_panel_ms;         /* device time inside the panel kernels              */
  double schur_flops;        /* algorithmic flops of the trailing updates: sum t*m*(m+1) */
  int64_t n_launches;        /* kernels launched by this call                     */
  int64_t mults, adds, divs, comps; /* the reference's OpCounters (metrics.py:28-43), exact */
  double panel_prof_ms[16];  /* CTA-0 cycle profile of the panel kernels (ms at the max SM clock):
                                0 qrcp, 1 qrcp-exchange, 2 sbkp-gemv, 3 sbkp-exchange, 4 sbkp-eliminate,
                                5 next-pivot, 6 qrcp-reflect, 7 total, 8 sbkp-local-argmax,
                                9 qrcp-local-argmax, 10 qrcp-householder */
  char message[160];
} rcp_stats;

/* Fill host `out` (row-major rows x cols) with the next standard normals of the
 * factorization's generator (numpy Generator(Philox(seed)).standard_normal).
 * Return 0 on success. */
typedef int (*rcp_draw_fn)(void* ctx, int64_t rows, int64_t cols, double* out);

/* Bytes of device workspace rcp_factor needs for this (n, cfg). */
size_t rcp_workspace_bytes(int64_t n, const rcp_config* cfg);

/* Factor A[perm][:, perm] = L D L^T (randldl.factor, factor.py:637-647) with the strategy in
 * cfg->strategy.  omega (p x n, device, row-major: the first draw of the factorization's
 * generator) is required for RCP_STRATEGY_RCP and ignored (may be NULL) for bkpp / bbk.
 * Optional per-step trace (device, may be NULL): trace_kind[k] in {0 skip, 1 1x1,
 * 2 1x1-swap, 3 2x2} at each decision position k, trace_r[k] = partner r or -1. */
int rcp_factor(const rcp_config* cfg, int64_t n, const double* a, int64_t lda,
               const double* omega, rcp_draw_fn draw, void* draw_ctx,
               void* workspace, size_t workspace_bytes,
               int64_t* perm, double* L, double* d_diag, double* d_off, int8_t* pattern,
               int8_t* trace_kind, int32_t* trace_r,
               rcp_stats* stats, void* cuda_stream);

/* rcp_factor with L also delivered to L_host (pinned host memory, dense row-major n x n): block
 * rows of L's lower trapezoid are copied while later panels still run, the strictly-upper part is
 * zeroed on host threads; returns once L_host is complete.  The device outputs are as rcp_factor's.
 * Serves randldl.factor's host result (factor.py:637-647: L is returned dense). */
int rcp_factor_host_l(const rcp_config* cfg, int64_t n, const double* a, int64_t lda,
                      const double* omega, rcp_draw_fn draw, void* draw_ctx,
                      void* workspace, size_t workspace_bytes,
                      int64_t* perm, double* L, double* d_diag, double* d_off, int8_t* pattern,
                      int8_t* trace_kind, int32_t* trace_r,
                      rcp_stats* stats, double* L_host, void* cuda_stream);

/* rcp_factor from a HOST matrix (row-major n x n, ld lda; pinned for full PCIe speed): only its
 * lower trapezoid is copied to the device (the kernel mirrors it) while host threads check the
 * exact symmetry of the whole matrix (core.py:48-53; reported first, as the reference does).
 * omega may be NULL for RCP_STRATEGY_RCP: Omega is then the first draw of `draw`, taken while
 * the copies run.  L_host (optional, pinned, dense n x n) receives L as in rcp_factor_host_l.
 * Serves randldl.factor(a) on a host array (factor.py:637-647). */
int rcp_factor_host(const rcp_config* cfg, int64_t n, const double* a_host, int64_t lda,
                    const double* omega, rcp_draw_fn draw, void* draw_ctx,
                    void* workspace, size_t workspace_bytes,
                    int64_t* perm, double* L, double* d_diag, double* d_off, int8_t* pattern,
                    int8_t* trace_kind, int32_t* trace_r,
                    rcp_stats* stats, double* L_host, void* cuda_stream);

/* Experiment diagnostics of the reference engine (FactorConfig.track_growth="full" and
 * audit_sketch, factor.py:294-296, 493-504, 566-567, 605-606).  The reference forces width-1
 * panels for them; pass cfg->b = cfg->q = 1.  All buffers are device memory. */
typedef struct rcp_diag {
  int32_t track_full;     /* 1: one snapshot per step: (max|S|, largest column norm of S) of the
                             active Schur complement S = A[k:, k:] at the step start            */
  int32_t audit;          /* 1: sketch drift ||B[:, k:] - Omega[:, k:] S||_{1,2} after each panel
                             with k < n (unnormalised; the caller divides by ||A||_{1,2})       */
  double* snapshots;      /* [cap][2], zeroed by the call                                       */
  double* drift;          /* [cap], zeroed by the call                                          */
  double* omega_orig;     /* audit scratch, p x n                                               */
  int64_t cap;            /* >= n + 1                                                            */
  int64_t n_snapshots;    /* out */
  int64_t n_drift;        /* out */
} rcp_diag;
/* rcp_factor plus the diagnostics above (replaces randldl.factor with track_growth="full" or
 * audit_sketch=True, factor.py:637-647). */
int rcp_factor_diag(const rcp_config* cfg, int64_t n, const double* a, int64_t lda,
                    const double* omega, rcp_draw_fn draw, void* draw_ctx,
                    void* workspace, size_t workspace_bytes,
                    int64_t* perm, double* L, double* d_diag, double* d_off, int8_t* pattern,
                    int8_t* trace_kind, int32_t* trace_r, rcp_stats* stats, rcp_diag* diag,
                    void* cuda_stream);
/* x = P^T L^-T D^-1 L^-1 P b for nrhs right-hand sides (solve.py:69-92).
 * b and x are device, column-major n x nrhs (ld = n); may alias.  *singular is
 * set to 1 if an exact-zero block was met (solve.py:47-58). */
int rcp_solve(int64_t n, const int64_t* perm, const double* L, const double* d_diag,
              const double* d_off, const int8_t* pattern, int64_t nrhs,
              const double* b, double* x, void* workspace, size_t workspace_bytes,
              int32_t* singular, void* cuda_stream);

/* Workspace bytes for rcp_solve. */
size_t rcp_solve_workspace_bytes(int64_t n, int64_t nrhs);

/* out (n x n row-major) = L D L^T (factor.py:663-665). */
int rcp_reconstruct(int64_t n, const double* L, const double* d_diag, const double* d_off,
                    const int8_t* pattern, double* out, void* cuda_stream);

/* ---- several GPUs of one node (C3) --------------------------------------------------------
 * Rank 0 calls rcp_factor_dist(world = N); ranks 1..N-1 call rcp_schur_worker with rank 0's
 * workspace mapped into their address space (rcp_ipc_export / rcp_ipc_import of a workspace
 * obtained from rcp_device_alloc).  Before the workers attach, rank 0 calls rcp_dist_prepare.
 * Every panel's trailing Schur update (the O(n^3) part) is split tile-round-robin over the N
 * devices; C-in tiles are read from and results written to rank 0's matrix over NVLink, the
 * panel operands are copied once per panel.  emulate = 1 runs the N-1 worker parts on this
 * device instead (same kernels, same results; used by the tests); worker_ws then holds
 * N-1 slots of rcp_worker_workspace_bytes. */
int rcp_factor_dist(const rcp_config* cfg, int64_t n, const double* a, int64_t lda,
                    const double* omega, rcp_draw_fn draw, void* draw_ctx,
                    void* workspace, size_t workspace_bytes,
                    int64_t* perm, double* L, double* d_diag, double* d_off, int8_t* pattern,
                    int8_t* trace_kind, int32_t* trace_r, rcp_stats* stats,
                    int world, int emulate, void* worker_ws, size_t worker_ws_bytes, void* cuda_stream);
size_t rcp_worker_workspace_bytes(int64_t n, const rcp_config* cfg);
int rcp_dist_prepare(int64_t n, const rcp_config* cfg, void* workspace, void* cuda_stream);
int rcp_schur_worker(const rcp_config* cfg, int64_t n, int rank, int world, void* rank0_workspace,
                     void* worker_ws, size_t worker_ws_bytes, void* cuda_stream);
/* Host-side plan of one panel's trailing update: the tiles (m0 = first trailing row, n0 = first
 * column or, for a sketch tile, first sketch row; sketch = 1 for the fused sketch-correction tiles,
 * which exist only when P > 0 on a single device) that device `part` of `nparts` processes, in the
 * order its `grid` CTAs take them (CTA 0's tiles, then CTA 1's, ...).  Computed with the same
 * functions the kernel uses (schur_ws2.cuh super_sequence / super_at: a CTA takes 128x128 supertiles,
 * reported as their two 128x64 tiles; with RCP_SCHUR_V=1 schur_ws.cuh tile_sequence / tile_at); lets
 * the distributed host logic and its tests check the dealing without a GPU.  Returns the tile count
 * (entries beyond cap are not written), -1 on bad arguments. */
int64_t rcp_schur_tile_plan(int64_t mp, int32_t P, int32_t part, int32_t nparts, int32_t grid,
                            int64_t* m0, int64_t* n0, int8_t* sketch, int64_t cap);
/* Dense host copy of a device unit-lower L (row-major n x n): the lower trapezoid is copied,
 * the strictly upper part is written as zeros on the host; synchronises cuda_stream.
 * Replaces the dense L transfer of the reference's result (factor.py:637-647 returns L dense). */
int rcp_lower_to_host(int64_t n, const double* dL, double* hL, void* cuda_stream);
int rcp_device_alloc(size_t bytes, void** ptr);
int rcp_device_free(void* ptr);
/* handle_out: 64 bytes (cudaIpcMemHandle_t); base must come from rcp_device_alloc. */
int rcp_ipc_export(const void* base, void* handle_out);
int rcp_ipc_import(const void* handle, void** ptr);
int rcp_ipc_close(void* ptr);

/* ---- batched small matrices (C5) -------------------------------------------------------- */

/* Per-matrix outcome of rcp_factor_batched (status uses the RCP_* codes above). */
typedef struct rcp_batch_stats {
  int32_t status;            /* RCP_OK / NOT_SYMMETRIC / NONFINITE_INPUT / NUMERICAL / NEED_NORMALS */
  int32_t num_kind;          /* RCP_NUM_* when status == RCP_ERR_NUMERICAL                      */
  int32_t num_step;          /* step k of the numerical error                                    */
  int32_t recompute_count;   /* guard recomputes                                                 */
  int32_t deficient_from;    /* first PAT_DEFICIENT index, -1 if none                            */
  int32_t n_2x2;
  int32_t n_steps;
  int32_t n_panels;
  double rho_cheap, max_multiplier, amax, dmax;
  int64_t mults, adds, divs, comps;  /* OpCounters (metrics.py:28-43)                           */
} rcp_batch_stats;

/* Device workspace bytes for rcp_factor_batched (independent of `count`: the kernel is
 * persistent, one slot per resident CTA). */
size_t rcp_batched_workspace_bytes(int64_t n, const rcp_config* cfg);

/* Factor `count` independent symmetric n x n matrices (n <= 256, q == b <= 32, p <= 64):
 * matrix i is a + i * a_stride (leading dimension lda).  `normals` (device, length
 * normals_len >= p * n) is the factorization's normal stream
 * Generator(Philox(seed)).standard_normal(normals_len): its first p * n values are Omega
 * (row-major, sketch.py:83-84) and each guard recompute of a matrix consumes the next p * m
 * values (sketch.py:63-84) — every matrix starts the stream afresh, exactly as separate
 * randldl.factor calls with one cfg.seed do.  A matrix that would need more normals than
 * supplied gets status RCP_ERR_NEED_NORMALS (re-run it with rcp_factor).
 * Outputs are per matrix, contiguous: perm[count][n], L[count][n][n] (row-major),
 * d_diag/d_off[count][n], pattern[count][n], mstats[count] (all device).
 * Returns RCP_OK when the launch succeeded; per-matrix outcomes are in mstats. */
int rcp_factor_batched(const rcp_config* cfg, int64_t count, int64_t n, const double* a,
                       int64_t lda, int64_t a_stride, const double* normals, int64_t normals_len,
                       void* workspace, size_t workspace_bytes, int64_t* perm, double* L,
                       double* d_diag, double* d_off, int8_t* pattern, rcp_batch_stats* mstats,
                       void* cuda_stream);

/* x[i] = solve(factorization i, b[i]) for `count` factorizations from rcp_factor_batched
 * (solve.py:34-76); b and x are [count][n] (may alias); singular[i] set as in rcp_solve. */
int rcp_solve_batched(int64_t count, int64_t n, const int64_t* perm, const double* L,
                      const double* d_diag, const double* d_off, const int8_t* pattern,
                      const double* b, double* x, int32_t* singular, void* cuda_stream);

/* Library identification: "rcp_b200 <version> sm_100a". */
const char* rcp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RCP_B200_H */
