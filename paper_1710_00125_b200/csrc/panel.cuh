// Panel-kernel parameter/state structs shared by panel.cu and the host driver.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rcp {

// Device-resident state that persists across panel launches.
struct PanelState {
  long long seq;       // monotonically increasing exchange sequence number
  long long err;       // (step << 8) | kind of the first numerical error, LLONG_MAX if none
  int k_end;           // logical index after the panel
  int t_end;           // columns eliminated by the panel
  int status;          // 0 ok, 1 guard trip (recompute needed), 2 guard stop (deficient tail)
  int n_steps;         // decisions taken (cumulative)
  int n_2x2;           // 2x2 blocks (cumulative)
  int end_reason;      // why the panel ended early: 0 none, 1 2x2 defer, 2 q=1 guard defer
  long long cnt[4];    // step op counters (mults, adds, divs, comps), cumulative
  // SM-cycle profile of CTA 0 (cumulative), see kProfNames in capi.cu
  long long cyc[16];
};

constexpr int kXWords = 16;  // 11 used, padded to 128 B per record
constexpr int kQWords = 8;  // norm(2) pos col coef(2) skip, padded

// One CTA's contribution to a pivot-search exchange (SBKP step).
struct XRec {
  double key;   // |c| of the CTA's best candidate row, -1 if none
  double val;   // signed c at that row
  double diag;  // current Schur-complement diagonal at that row
  double akk;   // pivot diagonal (valid if has_akk)
  int lidx;     // logical (panel-relative) index of the candidate
  int phys;     // physical (panel-relative) row of the candidate
  int has_akk;
  int err;
  double pad[2];  // 64-byte records
};

// One CTA's contribution to a QRCP exchange.
struct QRec {
  double norm;  // residual norm of the best local column, -1 if none
  int pos;      // its current position (panel-relative)
  int col;      // its panel-start column (panel-relative)
};

struct PanelParams {
  int64_t n;
  int k0, width, P, qn;
  int guard_mode;      // 0 none, 1 trip check, 2 stop check (after a recompute)
  double guard_limit;  // thr * beta
  double alpha;
  int G, R, Rs, Ls, Wn;
  int qmode;           // QRCP: 1 = register mode (one column per thread), 0 = generic
  int q1;              // 1: q = 1 mode (per-step sketch pivot + per-step sketch downdate)
  double* Bout;        // q = 1: updated sketch written in the new logical order
  const double* A;     // trailing matrix at panel start, col-major ld n, lower triangle valid
  const double* B;     // sketch, P x n col-major (ld P), panel-start order
  double* qscr;        // spill for sketch columns that do not fit in smem
  double* Lbuf;        // n x n col-major; column c holds rows in its panel's start order
  double* W;           // n x (b+2) col-major, unscaled panel columns (L * D)
  int* log_of_phys;    // out: logical index of each physical row (absolute)
  int* phys_of_log;    // out: physical row of each logical index (absolute)
  const int* perm_cur; // original index of each physical row at panel start
  int64_t* perm_out;
  double* d_diag;
  double* d_off;
  int8_t* pattern;
  int8_t* trace_kind;
  int32_t* trace_r;
  // Exchange buffers in LL format (NCCL-style): every 64-bit word carries 32 data bits and
  // the 32-bit exchange tag, so a reader validates data and arrival with one load.
  unsigned long long* xll;   // SBKP records  [2][G][kXWords]
  unsigned long long* qll;   // QRCP records  [2][G][kQWords]
  unsigned long long* qcll;  // QRCP candidate columns [2][G][2P]
  unsigned long long* sdll;  // SBKP decision broadcast by the reducer CTA [2][kXWords]
  unsigned long long* qdll;  // QRCP decision header [2][8]
  PanelState* st;
};

cudaError_t panel_init_attributes(int max_dyn_smem);
cudaError_t launch_panel(const PanelParams& prm, int G, size_t smem, cudaStream_t st);
int panel_static_smem_bytes();

}  // namespace rcp
