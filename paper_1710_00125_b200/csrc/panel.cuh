// Panel-kernel parameter/state structs shared by panel.cu and the host driver.
#pragma once
#include <climits>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace rcp {

#define RCP_PG __host__ __device__ inline

#ifndef RCP_PANEL_ROWS_MIN
#define RCP_PANEL_ROWS_MIN 128
#endif
// Fewest rows per CTA before the panel uses fewer CTAs.  One row / sketch column per thread costs the same
// wall time for 32 or 128 rows per CTA, while every exchange gets cheaper with fewer CTAs (fewer records
// for the reducer, less arrival skew): 128 vs 32 measured -5 % panel time at C2 / C4, -1.5 % at C3
// (profiles/r02_panel_experiments.txt); results are bit-identical for any value.
constexpr int kPanelRowsMin = RCP_PANEL_ROWS_MIN;
constexpr int kPanelMaxCTAs = 160;  // == kMaxSMs (exchange buffers are sized for it)
constexpr int kPanelRegRows = 32;   // QRCP register mode: sketch rows [0, 32) in registers

// Device-driven host loop: the host enqueues panels back to back without reading their
// outcome.  Panel p reads desc[p & 1]; its commit kernel finalises that descriptor (ok,
// k_end, t) for the gather / Schur / sketch kernels of the same panel and writes the next
// panel's descriptor desc[(p + 1) & 1].  A panel whose descriptor has run == 0 (finished,
// guard event or error upstream) and every kernel reading ok == 0 is a no-op.
struct PanelDesc {
  int k0;      // first logical column of the panel
  int run;     // 1: the panel must run
  int pidx;    // panel index
  int ok;      // set by the commit kernel: the panel completed normally
  int k_end;   // outcome (valid when ok)
  int t;
  long long snap_off;  // offset of the panel's start-order snapshot
};

// Per-panel record for the final assembly and the statistics.
struct PanelLog {
  int k0, k_end, m0, qn;
  long long snap_off;
};

// Launch geometry of one panel (shared by the host and the kernel).
struct PanelGeom {
  int m0, width, G, R, Wn, qn, qmode, Rs, Ls;
};

RCP_PG int pg_min(int a, int b) { return a < b ? a : b; }
RCP_PG int pg_max(int a, int b) { return a > b ? a : b; }

RCP_PG PanelGeom panel_geometry(int64_t n, int k0, int b, int q, int P, int num_sms, int smem_budget) {
  PanelGeom g{};
  g.m0 = (int)(n - k0);
  if (g.m0 <= 0) return g;
  g.width = pg_min(b, g.m0);
  int G = pg_min(num_sms, pg_max(1, (g.m0 + kPanelRowsMin - 1) / kPanelRowsMin));
  if (G > kPanelMaxCTAs) G = kPanelMaxCTAs;
  const int R = (g.m0 + G - 1) / G;
  g.G = (g.m0 + R - 1) / R;
  g.R = R;
  g.Wn = g.width + 2;
  g.qn = (q > 1 && g.m0 > 1) ? pg_min(pg_min(q, g.width), pg_min(g.m0, P)) : 0;
  auto a16 = [](long long x) { return (x + 15) & ~15LL; };
  const long long fixed = a16(4LL * g.Wn) + a16(4LL * R) + 2 * a16(8LL * P) + 4 * a16(8LL * g.Wn);
  const long long avail = (long long)smem_budget - fixed;
  g.qmode = 0;
  g.Rs = 0;
  if (g.qn > 0) {
    const int ps_reg = P - pg_min(P, kPanelRegRows);
    const long long need_reg = 8LL * ps_reg * R + 64;
    if (R <= 256 && need_reg <= avail) {
      g.qmode = 1;
      g.Rs = R;
    } else {
      long long rs = (avail - 12LL * R - 64) / (8LL * P);
      if (rs > R) rs = R;
      if (rs < 0) rs = 0;
      g.Rs = (int)rs;
    }
  }
  const bool q1 = (q == 1);
  long long ls = q1 ? (avail - 24LL * R - 8LL * P * R - 8LL * P - 128) / (8LL * R) : (avail - 24LL * R - 64) / (8LL * R);
  if (ls > g.Wn) ls = g.Wn;
  if (ls < 0) ls = 0;
  g.Ls = (int)ls;
  return g;
}

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
  int stop_pidx;       // first panel that ended with a guard event / error (-1: none)
  int panels_done;     // panels committed
  long long cnt[4];    // step op counters (mults, adds, divs, comps), cumulative
  // SM-cycle profile of CTA 0 (cumulative), see kProfNames in capi.cu
  long long cyc[16];
};

constexpr int kXWords = 16;  // 11 used, padded to 128 B per record
constexpr int kQWords = 8;  // norm(2) pos col coef(2) skip, padded
constexpr int kMWords = 16;  // one 128-byte decision mailbox line per CTA
// LL words of one CTA's candidate-column buffer: 2 per sketch row + coef (2) + skip (1), padded
RCP_PG size_t qcol_stride(int P) { return 2 * (size_t)P + 4; }

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
  unsigned long long* qcll;  // QRCP candidate columns [2][G][qcol_stride(P)]
  // Decisions are pushed by the reducer CTA into one private mailbox line per CTA, so each CTA
  // polls its own line (no hot line polled by the whole grid).
  unsigned long long* sdll;  // SBKP decision mailboxes [2][G][kMWords]
  unsigned long long* qdll;  // QRCP / q = 1 decision mailboxes [2][G][kMWords]
  PanelState* st;
  // device-driven geometry (desc != nullptr): k0 from the descriptor, the rest recomputed
  const PanelDesc* desc;
  int b, q, num_sms, smem_budget;
  int strategy;  // RCP_STRATEGY_*: decision rule of the pivot steps
  double* bkscr;  // bbk: per-CTA global scratch (third column + W-row buffer), G * (R + Wn) doubles
  unsigned long long* tstamp;  // [panel][4] timestamps (panel start/end, Schur start/end), or null
};

cudaError_t panel_init_attributes(int max_dyn_smem);
cudaError_t launch_panel(const PanelParams& prm, int G, size_t smem, cudaStream_t st);
cudaError_t launch_panel_commit(PanelDesc* din, PanelDesc* dout, PanelLog* plog, PanelState* st, int64_t n, int b,
                                int q, int P, long long snap_cap, cudaStream_t stream);
int panel_static_smem_bytes();

}  // namespace rcp
