// Persistent cooperative panel kernel: the sequential critical path of RCP.
//
// One launch factors one panel (reference _run_panel minus the trailing flush,
// factor.py:540-568):
//   1. guard check + partial QRCP on the (p x m) sketch           (factor.py:570-600, sketch.py:135-169)
//   2. up to b SBKP decisions with symmetric swaps + elimination  (factor.py:602-634, 414-489)
//
// Layout: the grid's G CTAs own contiguous slices of R physical rows (= sketch
// columns) of the active block [k0, n).  Symmetric swaps are NOT applied to the
// matrix: the panel works on the panel-start ("physical") order and tracks the
// permutation (replicated window `win` for the pivot positions, `lpos` for owned
// rows).  The permutation is applied later by the gather-fused trailing update.
//
// Every pivot search / QRCP step is ONE all-to-all exchange: each CTA publishes its
// local best candidate (plus the data the decision needs) behind a release flag;
// every CTA polls all G flags, loads all G records and reduces them identically, so
// all CTAs take the same decision without a second barrier.  Values a CTA needs from
// rows it does not own (the next pivot's W-row entries of the columns produced in
// this step) are recomputed redundantly with the same bitwise-deterministic dot
// routine the owner used.
#include <cfloat>
#include <climits>
#include "panel.cuh"
#include "rcp_common.cuh"

namespace rcp {

namespace {

constexpr int kPanelThreads = 256;
constexpr int kWarps = kPanelThreads / 32;
constexpr int kRegRows = 32;  // QRCP register mode: 32 sketch rows of each column live in registers
#ifndef RCP_QRCP_REG_TAIL
#define RCP_QRCP_REG_TAIL 0
#endif
// Which rows: head (0, default) = rows [0, 32); tail (1) = the last 32 rows, which stay live through
// every QRCP step (rows [0, j) are finished after step j), cutting the shared-memory row passes of
// a 128-step panel at P = 144 from 9776 to 6328.  Measured at C3: panel 407.3 ms (tail) vs 404.8 ms
// (head), identical results -- the reflect pass is bound by its per-thread dependent chain, not by
// shared-memory bandwidth, and the tail mode runs the 32 predicated register rows in all steps.
constexpr bool kRegTail = RCP_QRCP_REG_TAIL != 0;
constexpr long long kWatchdogCycles = 8000000000LL;

struct BlockBest {
  double key;
  long long idx;
  int slot;
};

RCP_D void argmax_step(double& key, long long& idx, int& slot, int off) {
  double k2 = __shfl_down_sync(0xffffffffu, key, off);
  long long i2 = __shfl_down_sync(0xffffffffu, idx, off);
  int s2 = __shfl_down_sync(0xffffffffu, slot, off);
  if (better(k2, i2, key, idx)) {
    key = k2;
    idx = i2;
    slot = s2;
  }
}

// Block-wide argmax (numpy first-index semantics), broadcast to all threads; one barrier:
// warps reduce by shuffles, then every thread reduces the kWarps warp results itself (`better`
// is a strict total order, so every thread gets the same answer).  `parity` alternates between
// consecutive calls (the per-warp slots are double-buffered).
__device__ BlockBest block_argmax(double key, long long idx, int slot, int parity) {
  __shared__ double sk[2][kWarps];
  __shared__ long long si[2][kWarps];
  __shared__ int ss[2][kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) argmax_step(key, idx, slot, off);
  if (lane == 0) {
    sk[parity][warp] = key;
    si[parity][warp] = idx;
    ss[parity][warp] = slot;
  }
  __syncthreads();
  double wk[kWarps];
  long long wi[kWarps];
  int wsl[kWarps];
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    wk[w] = sk[parity][w];
    wi[w] = si[parity][w];
    wsl[w] = ss[parity][w];
  }
  BlockBest r{wk[0], wi[0], wsl[0]};
#pragma unroll
  for (int w = 1; w < kWarps; ++w)
    if (better(wk[w], wi[w], r.key, r.idx)) r = BlockBest{wk[w], wi[w], wsl[w]};
  return r;
}

// Deterministic sum of squares over vals[lo, hi) by warp 0 (lane-strided partials + fixed
// tree): every CTA obtains the same bits.  Result valid in lane 0.
__device__ double warp0_sum_sq(const double* vals, int lo, int hi) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int r = lo + lane; r < hi; r += 32) acc = __fma_rn(vals[r], vals[r], acc);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, off));
  return acc;
}

// ---- LL exchange words: 32 data bits + 32-bit tag per 64-bit store (single-copy atomic),
// so a reader validates arrival and data with the same load and no fences are needed.
typedef unsigned long long u64;
RCP_D void ll_put(u64* p, unsigned tag, unsigned data) {
  const u64 v = (static_cast<u64>(tag) << 32) | data;
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
RCP_D u64 ll_get(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
RCP_D void ll_put_d(u64* p, unsigned tag, double x) {
  const u64 b = static_cast<u64>(__double_as_longlong(x));
  ll_put(p, tag, static_cast<unsigned>(b));
  ll_put(p + 1, tag, static_cast<unsigned>(b >> 32));
}
RCP_D double ll_d(unsigned lo, unsigned hi) {
  return __longlong_as_double(static_cast<long long>((static_cast<u64>(hi) << 32) | lo));
}
// Spin until all NW words carry `tag`; false if the watchdog fired (a lost peer).
template <int NW>
RCP_D bool ll_read(const u64* p, unsigned tag, unsigned (&out)[NW]) {
  const long long t0 = clock64();
  while (true) {
    bool ok = true;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const u64 v = ll_get(p + w);
      out[w] = static_cast<unsigned>(v);
      ok &= static_cast<unsigned>(v >> 32) == tag;
    }
    if (ok) return true;
    if (clock64() - t0 > kWatchdogCycles) return false;
  }
}

// Euclidean norm from a fused (sum of squares, max |x|) pass; falls back to the
// reference's scaled formulation (core.py:122-142) when the plain sum could over/underflow.
template <class Get>
RCP_D double safe_norm(double sumsq, double amax, Get get, int lo, int hi) {
  if (amax == 0.0) return 0.0;
  if (amax > 1e-140 && amax < 1e140) return sqrt(sumsq);
  double ss = 0.0;
  for (int r = lo; r < hi; ++r) {
    double x = fabs(get(r)) / amax;
    ss = __fma_rn(x, x, ss);
  }
  return amax * sqrt(ss);
}

RCP_D long long prof_now() { return clock64(); }


}  // namespace

// STRAT: RCP_STRATEGY_* as a template argument, so the rcp kernel carries no bkpp / bbk code.
template <int STRAT>
__global__ void __launch_bounds__(kPanelThreads, 1) panel_kernel(PanelParams pin) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int cta = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  PanelParams p = pin;
  if (p.desc) {  // device-driven: this panel's k0 comes from the descriptor chain
    const int run = p.desc->run;
    if (!run) return;
    const PanelGeom g = panel_geometry(p.n, p.desc->k0, p.b, p.q, p.P, p.num_sms, p.smem_budget);
    p.k0 = p.desc->k0;
    p.width = g.width;
    p.G = g.G;
    p.R = g.R;
    p.Wn = g.Wn;
    p.qn = g.qn;
    p.qmode = g.qmode;
    p.Rs = g.Rs;
    p.Ls = g.Ls;
    if (!(g.qn > 0 || p.q1)) p.guard_mode = 0;
    if (cta >= g.G) return;
  }
  unsigned long long* const ts_panel = (p.tstamp && p.desc) ? p.tstamp + 4 * (size_t)p.desc->pidx : nullptr;
  stamp_start(ts_panel);
  const int64_t n = p.n;
  const int k0 = p.k0, P = p.P, R = p.R, G = p.G, Wn = p.Wn;
  const size_t QS = qcol_stride(P);  // LL words per candidate-column buffer
#ifndef RCP_REDUCER_LAST
#define RCP_REDUCER_LAST 1
#endif
  // Reducer CTA of every exchange.  The last CTA owns the fewest rows (m - (G-1) R), so it tends
  // to publish its record first and starts reducing earliest.
  const int kRed = RCP_REDUCER_LAST ? G - 1 : 0;
  const int m0 = static_cast<int>(n - k0);
  const int r0 = cta * R;
  const int rcnt = max(0, min(R, m0 - r0));
#ifndef RCP_PANEL_PROF
#define RCP_PANEL_PROF 0  // build with -DRCP_PANEL_PROF=1 for the per-phase cycle profile
#endif
#ifndef RCP_PROF_CTA
#define RCP_PROF_CTA 0  // CTA whose phases the profile build times
#endif
  const bool prof = RCP_PANEL_PROF && (cta == RCP_PROF_CTA && tid == 0);
  const long long c_kernel0 = prof ? prof_now() : 0;
  long long c_mark = 0;
#define PROF_BEGIN() \
  if (prof) c_mark = prof_now()
#define PROF_END(slot) \
  if (prof) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->cyc[slot]), (unsigned long long)(prof_now() - c_mark))

  // ---- shared memory carve-up
  unsigned char* sp = smem_raw;
  auto carve = [&](size_t bytes) {
    unsigned char* q = sp;
    sp += (bytes + 15) & ~size_t(15);
    return q;
  };
  int* win = reinterpret_cast<int*>(carve(sizeof(int) * Wn));
  int* lpos = reinterpret_cast<int*>(carve(sizeof(int) * R));
  double* vvec = reinterpret_cast<double*>(carve(sizeof(double) * P));
  double* vvec2 = reinterpret_cast<double*>(carve(sizeof(double) * P));  // QRCP: previous reflector
  double* wrow = reinterpret_cast<double*>(carve(sizeof(double) * Wn));
  double* wrrow = reinterpret_cast<double*>(carve(sizeof(double) * Wn));
  double* lnext = reinterpret_cast<double*>(carve(sizeof(double) * Wn));
  double* wnext = reinterpret_cast<double*>(carve(sizeof(double) * Wn));
  unsigned char* region = sp;  // QRCP and SBKP phases reuse the rest

  __shared__ int s_abort, s_gerr, s_lerr, s_skip, s_wcol;
  __shared__ double s_coef, s_gakk, s_akk;
  __shared__ XRec s_win;
  __shared__ unsigned s_qhdr[8], s_dhdr[12];
  __shared__ int s_wpos, s_qflags, s_hascand, s_wcta, s_gs1, s_gs2;
  __shared__ double s_bkarr, s_bkcp;  // bkpp / bbk: a_rr of the partner column, c_p(imax)
  __shared__ int s_bkhas, s_bkjph;

  for (int x = tid; x < Wn; x += nthr) win[x] = x;
  for (int i = tid; i < rcnt; i += nthr) lpos[i] = r0 + i;
  if (tid == 0) {
    s_abort = 0;
    s_lerr = 0;
  }
  long long seq = p.st->seq;
  int par = 0;  // block_argmax result buffer parity
  __syncthreads();

  // =====================================================================
  // Phase 1: guard + partial QRCP on the sketch (q = b mode).
  // =====================================================================
  const long long c_q0 = prof ? prof_now() : 0;
  if (p.qn > 0) {
    // Register mode: one column per thread, rows [0, 32) in registers, the rest in smem.
    // Generic mode: columns spread over threads; smem with a global spill.
    const bool regmode = p.qmode == 1;
    const int PRr = regmode ? min(P, kRegRows) : 0;
    const int Ps = P - PRr;
    const int RR0 = kRegTail ? P - PRr : 0;  // first register row (register rows [RR0, RR0 + PRr))
    const int S0 = kRegTail ? 0 : PRr;       // first shared-memory row (rows [S0, S0 + Ps))
    const int S1 = S0 + Ps;
    const int Rs = regmode ? R : p.Rs;  // columns whose rows >= PRr live in smem
    const int Rg = R - Rs;
    double* Bs = reinterpret_cast<double*>(region);  // [Ps][Rs] row-major
    double* qnorm = Bs + (size_t)Ps * Rs;             // generic mode only
    int* qsel = reinterpret_cast<int*>(qnorm + R);
    double* qg = p.qscr + (size_t)cta * Ps * (Rg > 0 ? Rg : 0);
    auto bsm = [&](int r, int c) -> double& {  // shared-memory row r in [S0, S1) of column c
      return c < Rs ? Bs[(r - S0) * Rs + c] : qg[(size_t)(r - S0) * Rg + (c - Rs)];
    };
    double rg[kRegRows];
    const bool own = regmode && tid < rcnt;
    bool mysel = !own;
    double myn = -1.0, myn2 = 0.0, myn2x = 0.0;
    bool exact_only = false;
    int mypos = own ? r0 + tid : INT_MAX;
    // Register mode defers each reflector's update of the smem rows to the next step's pass
    // (x <- x - v_prev * w_prev, then the dot with v): one smem pass per step instead of two, with
    // bit-identical values.  Reflectors alternate between vvec / vvec2.
    double wpend = 0.0;  // w of the pending (previous) reflector for the own column
    bool pend = false;   // rows >= j of Bs still need the previous reflector

    // ---- load
    if (own) {
      const double* src = p.B + (size_t)(k0 + r0 + tid) * P;
#pragma unroll
      for (int r = 0; r < kRegRows; ++r) rg[r] = (r < PRr) ? src[RR0 + r] : 0.0;
    }
    {  // sketch rows >= PRr of the owned columns: 8 independent loads in flight per thread
      const int tot = Ps * rcnt;
      int f = tid;
      for (; f + 7 * nthr < tot; f += 8 * nthr) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = f + u * nthr, c = e / Ps, r = e - c * Ps;
          v[u] = __ldcg(p.B + (size_t)(k0 + r0 + c) * P + S0 + r);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = f + u * nthr, c = e / Ps, r = e - c * Ps;
          bsm(S0 + r, c) = v[u];
        }
      }
      for (; f < tot; f += nthr) {
        const int c = f / Ps, r = f - c * Ps;
        bsm(S0 + r, c) = p.B[(size_t)(k0 + r0 + c) * P + S0 + r];
      }
    }
    if (!regmode)
      for (int c = tid; c < rcnt; c += nthr) qsel[c] = 0;
    __syncthreads();
    // exact residual norm of the own column over rows [lo, P): sets myn, myn2, myn2x, exact_only
    auto exact_norm = [&](int lo) {
      double ss0 = 0.0, ss1 = 0.0, am = 0.0;
#pragma unroll
      for (int r = 0; r < kRegRows; ++r) {
        if (RR0 + r >= lo && r < PRr) {
          am = fmax(am, fabs(rg[r]));
          if (r & 1) ss1 = __fma_rn(rg[r], rg[r], ss1); else ss0 = __fma_rn(rg[r], rg[r], ss0);
        }
      }
      for (int r = max(lo, S0); r < S1; ++r) {
        const double x = Bs[(r - S0) * Rs + tid];
        am = fmax(am, fabs(x));
        if (r & 1) ss1 = __fma_rn(x, x, ss1); else ss0 = __fma_rn(x, x, ss0);
      }
      const double ss = __dadd_rn(ss0, ss1);
      if (am == 0.0) {
        myn = 0.0;
        myn2 = 0.0;
      } else if (am > 1e-140 && am < 1e140) {
        myn2 = ss;
        myn = sqrt(ss);
      } else {
        double s2 = 0.0;
#pragma unroll
        for (int r = 0; r < kRegRows; ++r)
          if (RR0 + r >= lo && r < PRr) {
            const double x = fabs(rg[r]) / am;
            s2 = __fma_rn(x, x, s2);
          }
        for (int r = max(lo, S0); r < S1; ++r) {
          const double x = fabs(Bs[(r - S0) * Rs + tid]) / am;
          s2 = __fma_rn(x, x, s2);
        }
        myn = am * sqrt(s2);
        myn2 = myn * myn;
        exact_only = true;  // out of the safe range for squared downdates
      }
      myn2x = myn2;
    };
    // Householder reflector (vc over rows [jj, P), coef, skip) applied to the own column, then the
    // residual-norm downdate (|r|^2 -= y^2, recomputed exactly whenever cancellation could cost
    // more than ~1e-10 relative accuracy: LAPACK xLAQP2 policy).  Register mode: the pending
    // reflector (vp, wpend) of the previous step is applied to the smem rows while forming this
    // step's dot, and this step's reflector becomes the pending one -- one smem pass per step,
    // values bit-identical to applying each reflector eagerly.
    auto reflect_fused = [&](const double* vc, const double* vp, int jj, double coef, int skip) {
      double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
      const bool regs_live = jj < RR0 + PRr;  // uniform: false once every register row is finished
      const double* vcr = vc + RR0;           // reflector entries of the register rows
      if (!skip && regs_live) {
#pragma unroll
        for (int r = 0; r < kRegRows; r += 4) {
          if (RR0 + r >= jj && r < PRr) d0 = __fma_rn(vcr[r], rg[r], d0);
          if (RR0 + r + 1 >= jj && r + 1 < PRr) d1 = __fma_rn(vcr[r + 1], rg[r + 1], d1);
          if (RR0 + r + 2 >= jj && r + 2 < PRr) d2 = __fma_rn(vcr[r + 2], rg[r + 2], d2);
          if (RR0 + r + 3 >= jj && r + 3 < PRr) d3 = __fma_rn(vcr[r + 3], rg[r + 3], d3);
        }
      }
      const int rs = max(jj, S0);
      double xjj = 0.0;  // x at row jj (smem rows) after the pending update
      {
        int r = rs;
        double* bw = Bs + (size_t)(r - S0) * Rs + tid;
        if (pend) {
          const double wp = wpend;
          for (; r + 4 <= S1; r += 4, bw += 4 * Rs) {
            double x0 = bw[0], x1 = bw[Rs], x2 = bw[2 * Rs], x3 = bw[3 * Rs];
            x0 = __fma_rn(-vp[r], wp, x0);
            x1 = __fma_rn(-vp[r + 1], wp, x1);
            x2 = __fma_rn(-vp[r + 2], wp, x2);
            x3 = __fma_rn(-vp[r + 3], wp, x3);
            bw[0] = x0;
            bw[Rs] = x1;
            bw[2 * Rs] = x2;
            bw[3 * Rs] = x3;
            if (r == jj) xjj = x0;
            if (!skip) {
              d0 = __fma_rn(vc[r], x0, d0);
              d1 = __fma_rn(vc[r + 1], x1, d1);
              d2 = __fma_rn(vc[r + 2], x2, d2);
              d3 = __fma_rn(vc[r + 3], x3, d3);
            }
          }
          for (; r < S1; ++r, bw += Rs) {
            const double x = __fma_rn(-vp[r], wp, *bw);
            *bw = x;
            if (r == jj) xjj = x;
            if (!skip) d0 = __fma_rn(vc[r], x, d0);
          }
        } else {
          for (; r + 4 <= S1; r += 4, bw += 4 * Rs) {
            const double x0 = bw[0], x1 = bw[Rs], x2 = bw[2 * Rs], x3 = bw[3 * Rs];
            if (r == jj) xjj = x0;
            if (!skip) {
              d0 = __fma_rn(vc[r], x0, d0);
              d1 = __fma_rn(vc[r + 1], x1, d1);
              d2 = __fma_rn(vc[r + 2], x2, d2);
              d3 = __fma_rn(vc[r + 3], x3, d3);
            }
          }
          for (; r < S1; ++r, bw += Rs) {
            const double x = *bw;
            if (r == jj) xjj = x;
            if (!skip) d0 = __fma_rn(vc[r], x, d0);
          }
        }
      }
      double wv = 0.0;
      if (!skip) {
        wv = __dmul_rn(coef, __dadd_rn(__dadd_rn(d0, d1), __dadd_rn(d2, d3)));
        if (regs_live) {
#pragma unroll
          for (int r2 = 0; r2 < kRegRows; ++r2)
            if (RR0 + r2 >= jj && r2 < PRr) rg[r2] = __fma_rn(-vcr[r2], wv, rg[r2]);
        }
      }
      double yj;
      if (jj >= RR0 && jj < RR0 + PRr) {
        yj = 0.0;
#pragma unroll
        for (int r2 = 0; r2 < kRegRows; ++r2)
          if (RR0 + r2 == jj) yj = rg[r2];
      } else {
        yj = skip ? xjj : __fma_rn(-vc[jj], wv, xjj);
      }
      wpend = wv;
      const double n2 = __fma_rn(-yj, yj, myn2);
      if (exact_only || !(n2 > 1e-6 * myn2x) || !(n2 > 1e-280)) {
        // the exact recompute needs the current values: apply this step's reflector now
        if (!skip) {
          double* bw = Bs + (size_t)(rs - S0) * Rs + tid;
          for (int r = rs; r < S1; ++r, bw += Rs) *bw = __fma_rn(-vc[r], wv, *bw);
          wpend = 0.0;  // already applied; x - v * 0 leaves the values unchanged next step
        }
        exact_norm(jj + 1);
      } else {
        myn2 = n2;
        myn = sqrt(n2);
      }
    };
    if (own) exact_norm(0);

    if (!regmode) {
      for (int c = tid; c < rcnt; c += nthr) {
        double ss = 0.0, am = 0.0;
        for (int r = 0; r < P; ++r) {
          double x = bsm(r, c);
          am = fmax(am, fabs(x));
          ss = __fma_rn(x, x, ss);
        }
        qnorm[c] = safe_norm(ss, am, [&](int r) { return bsm(r, c); }, 0, P);
      }
    }
    __syncthreads();

    for (int j = 0; j < p.qn; ++j) {
      double* const vcur = (regmode && (j & 1)) ? vvec2 : vvec;  // this step's reflector
      const double* const vprv = (regmode && (j & 1)) ? vvec : vvec2;  // the pending one (regmode)
      // ---- local candidate: largest residual norm, ties to the lowest position
      PROF_BEGIN();
      double bk = -1.0;
      long long bi = LLONG_MAX;
      int bs = -1;
      if (regmode) {
        if (own && !mysel) {
          bk = myn;
          bi = mypos;
          bs = tid;
        }
      } else {
        for (int c = tid; c < rcnt; c += nthr) {
          if (qsel[c]) continue;
          double v = qnorm[c];
          long long ix = lpos[c];
          if (better(v, ix, bk, bi)) {
            bk = v;
            bi = ix;
            bs = c;
          }
        }
      }
      BlockBest lb = block_argmax(bk, bi, bs, par);
      par ^= 1;
      const long long nseq = seq + 1;
      const int pb = static_cast<int>(nseq & 1);
      const unsigned tag = static_cast<unsigned>(nseq);
      // ---- speculative Householder vector of this CTA's candidate (sketch.py:159-168):
      //      only the global winner's v is used, so every CTA prepares its own and the
      //      reducer broadcasts just a small header.
      if (tid == 0) {  // the record goes out first; the reflector is built while it travels
        u64* q = p.qll + ((size_t)pb * G + cta) * kQWords;
        const bool has = lb.slot >= 0;
        ll_put_d(q, tag, has ? lb.key : -1.0);
        ll_put(q + 2, tag, has ? static_cast<unsigned>(lb.idx) : 0x7fffffffu);
        ll_put(q + 3, tag, has ? static_cast<unsigned>(r0 + lb.slot) : 0xffffffffu);
      }
      seq = nseq;
      __syncthreads();  // records out before anyone polls (measured: avoids a delayed store)
      PROF_END(9);
      {
        // Speculative reflector of this CTA's candidate (sketch.py:159-168), built by the warp holding
        // the column (warp 0 in generic mode) while the exchange is in flight; only the winner's is read.
        const int lane = tid & 31;
        const int hwarp = lb.slot < 0 ? -1 : (regmode ? (lb.slot >> 5) : 0);
        if ((tid >> 5) == hwarp) {
          if (regmode && j < RR0 + PRr && lane == (lb.slot & 31)) {
#pragma unroll
            for (int r = 0; r < kRegRows; ++r)
              if (RR0 + r >= j && r < PRr) vcur[RR0 + r] = rg[r];
          }
          const double wc = __shfl_sync(0xffffffffu, wpend, lb.slot & 31);  // candidate's pending w
          for (int r = max(j, S0) + lane; r < S1; r += 32) {
            if (regmode) {
              const double x = Bs[(r - S0) * Rs + lb.slot];
              vcur[r] = pend ? __fma_rn(-vprv[r], wc, x) : x;
            } else {
              vcur[r] = bsm(r, lb.slot);
            }
          }
          __syncwarp();
          const double xn = __shfl_sync(0xffffffffu, sqrt(warp0_sum_sq(vcur, j, P)), 0);
          double coef = 0.0;
          unsigned skip = 1;
          if (xn != 0.0) {
            if (lane == 0) {
              const double x0 = vcur[j];
              vcur[j] = __dadd_rn(x0, copysign(xn, x0 != 0.0 ? x0 : 1.0));
            }
            __syncwarp();
            const double vn2 = __shfl_sync(0xffffffffu, warp0_sum_sq(vcur, j, P), 0);
            skip = (vn2 == 0.0) ? 1u : 0u;
            coef = (vn2 == 0.0) ? 0.0 : 2.0 / vn2;
          }
          u64* dst = p.qcll + ((size_t)pb * G + cta) * QS;
          for (int r = j + lane; r < P; r += 32) ll_put_d(dst + 2 * r, tag, vcur[r]);
          if (lane == 0) {
            ll_put_d(dst + 2 * P, tag, coef);
            ll_put(dst + 2 * P + 2, tag, skip);
          }
        }
      }
      PROF_BEGIN();
      // ---- reducer CTA 0: winner over all records -> a 6-word decision pushed into every CTA's
      //      mailbox (winner CTA, position, column, coef, flags); every CTA then reads v from
      //      the winner's buffer.
      if (cta == kRed) {
        double gk = -1.0;
        long long gi = LLONG_MAX;
        int gs = -1;
        unsigned gw[4] = {0, 0, 0, 0};
        for (int c = tid; c < G; c += nthr) {
          unsigned w[4];
          if (!ll_read<4>(p.qll + ((size_t)pb * G + c) * kQWords, tag, w)) {
            s_abort = 1;
            continue;
          }
          const double v = ll_d(w[0], w[1]);
          const int ps = static_cast<int>(w[2]);
          if ((v >= 0.0 || v != v) && better(v, ps, gk, gi)) {
            gk = v;
            gi = ps;
            gs = c;
#pragma unroll
            for (int u = 0; u < 4; ++u) gw[u] = w[u];
          }
        }
        BlockBest gb = block_argmax(gk, gi, gs, par);
        if (gs >= 0 && gs == gb.slot) {  // the thread that loaded the winning record
          const bool gstop = (j == 0 && p.guard_mode != 0 && gb.key < p.guard_limit);
          s_qhdr[0] = static_cast<unsigned>(gs);
          s_qhdr[1] = gw[2];
          s_qhdr[2] = gw[3];
          s_qhdr[3] = gstop ? 2u : 0u;
        }
        if (gb.slot < 0 && tid == 0) s_qhdr[3] = 4u;  // no candidate anywhere: cannot happen
        __syncthreads();
        unsigned hw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) hw[u] = s_qhdr[u];
        if (s_abort) hw[3] = 4u;
        for (int f = tid; f < G * 4; f += nthr) {
          const int c = f >> 2, u = f & 3;
          if (c != kRed) ll_put(p.qdll + ((size_t)pb * G + c) * kMWords + u, tag, hw[u]);
        }
        if (tid == 0) {
          s_wcta = static_cast<int>(hw[0]);
          s_wpos = static_cast<int>(hw[1]);
          s_wcol = static_cast<int>(hw[2]);
          s_qflags = static_cast<int>(hw[3]);
        }
      } else {
        if (tid < 4) {
          unsigned w[1];
          if (!ll_read<1>(p.qdll + ((size_t)pb * G + cta) * kMWords + tid, tag, w)) {
            s_abort = 1;
            w[0] = 0;
          }
          s_qhdr[tid] = w[0];
        }
        __syncthreads();
        if (tid == 0) {
          s_wcta = static_cast<int>(s_qhdr[0]);
          s_wpos = static_cast<int>(s_qhdr[1]);
          s_wcol = static_cast<int>(s_qhdr[2]);
          s_qflags = static_cast<int>(s_qhdr[3]);
          if (s_abort) s_qflags |= 4;
        }
      }
      par ^= 1;
      __syncthreads();
      const int wpos = s_wpos;
      const int wcol = s_wcol;
      // replay bookkeeping (factor.py:586-599), position j <-> wpos: every thread reads the
      // displaced column now; thread 0 rewrites `win` after the next barrier
      const int moved = (wpos != j) ? win[j] : -1;
      if (!(s_qflags & 6)) {  // fetch the winner's Householder vector, coef and skip flag
        const u64* src = p.qcll + ((size_t)pb * G + s_wcta) * QS;
        for (int r = j + tid; r < P; r += nthr) {
          unsigned w[2];
          if (!ll_read<2>(src + 2 * r, tag, w)) s_abort = 1;
          vcur[r] = ll_d(w[0], w[1]);
        }
        if (tid == nthr - 1) {
          unsigned w[3];
          if (!ll_read<3>(src + 2 * P, tag, w)) s_abort = 1;
          s_coef = ll_d(w[0], w[1]);
          s_skip = static_cast<int>(w[2]);
        }
      }
      __syncthreads();
      PROF_END(1);
      PROF_BEGIN();
      if (s_abort || (s_qflags & 4)) {
        if (tid == 0) atomicExch(&p.st->status, 99);
        s_abort = 1;
        break;
      }
      if (s_qflags & 2) {
        if (cta == 0 && tid == 0) p.st->status = p.guard_mode == 1 ? 1 : 2;
        s_abort = 2;
        break;
      }
      if (tid == 0 && moved >= 0) {
        win[j] = wcol;
        if (wpos < Wn) win[wpos] = moved;
      }
      if (regmode) {
        if (own && r0 + tid == wcol) {
          mypos = j;
          mysel = true;
        }
        if (own && moved >= 0 && r0 + tid == moved) mypos = wpos;
      } else if (tid == 0) {
        if (wcol >= r0 && wcol < r0 + rcnt) {
          lpos[wcol - r0] = j;
          qsel[wcol - r0] = 1;
        }
        if (moved >= 0 && moved >= r0 && moved < r0 + rcnt) lpos[moved - r0] = wpos;
      }
      // ---- reflect the remaining columns and refresh their residual norms
      PROF_END(10);
      PROF_BEGIN();
      if (j + 1 < p.qn) {
        if (!regmode) __syncthreads();
        const int skip = s_skip;
        const double coef = s_coef;
        if (regmode) {
          if (own && !mysel) reflect_fused(vcur, vprv, j, coef, skip);
          pend = !skip;
        } else {
          for (int c = tid; c < rcnt; c += nthr) {
            if (qsel[c]) continue;
            double ss = 0.0, am = 0.0;
            if (!skip) {
              double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
              int r = j;
              for (; r + 4 <= P; r += 4) {
                d0 = __fma_rn(vvec[r], bsm(r, c), d0);
                d1 = __fma_rn(vvec[r + 1], bsm(r + 1, c), d1);
                d2 = __fma_rn(vvec[r + 2], bsm(r + 2, c), d2);
                d3 = __fma_rn(vvec[r + 3], bsm(r + 3, c), d3);
              }
              for (; r < P; ++r) d0 = __fma_rn(vvec[r], bsm(r, c), d0);
              const double wv = __dmul_rn(coef, __dadd_rn(__dadd_rn(d0, d1), __dadd_rn(d2, d3)));
              for (r = j; r < P; ++r) {
                double& x = bsm(r, c);
                const double y = __dsub_rn(x, __dmul_rn(vvec[r], wv));
                x = y;
                if (r > j) {
                  am = fmax(am, fabs(y));
                  ss = __fma_rn(y, y, ss);
                }
              }
            } else {
              for (int r = j + 1; r < P; ++r) {
                const double y = bsm(r, c);
                am = fmax(am, fabs(y));
                ss = __fma_rn(y, y, ss);
              }
            }
            qnorm[c] = safe_norm(ss, am, [&](int r) { return bsm(r, c); }, j + 1, P);
          }
        }
      }
      __syncthreads();
      PROF_END(6);
    }
    if (regmode && own) lpos[tid] = mypos;
  }
  if (prof) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->cyc[0]), (unsigned long long)(prof_now() - c_q0));
  __syncthreads();
  if (s_abort) {
    if (cta == 0 && tid == 0) p.st->seq = seq;
    return;
  }
  {
    // Prefetch this CTA's row slice of the panel's candidate pivot columns (the QRCP
    // selection, positions [0, Wn)) into L2: most SBKP pivot columns come from here.
    const int nl = (rcnt + 15) / 16;
    const int wx = min(Wn, m0);
    for (int f = tid; f < wx * nl; f += nthr) {
      const int x = f / nl, line = f - x * nl;
      const double* ptr = p.A + (k0 + r0 + 16 * line) + (int64_t)(k0 + win[x]) * n;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
    }
  }

  // =====================================================================
  // Phase 2: SBKP pivot steps (factor.py:602-634) with left-looking columns.
  // =====================================================================
  const int Ls = p.Ls;
  double* Lsm = reinterpret_cast<double*>(region);  // [Ls][R]
  double* ck = Lsm + (size_t)Ls * R;
  double* cr = ck + R;
  double* dg = cr + R;
  // q = 1 mode (factor.py:607-620, 486-489): own sketch columns [P][R] + the two pivot columns
  double* Bq = dg + R;
  double* skr = Bq + (size_t)P * R;
  double* skp0 = vvec;
  const bool q1 = p.q1 != 0;
  const double* A = p.A;
  const double alpha = p.alpha;
  const int width = p.width;

  for (int i = tid; i < rcnt; i += nthr) {
    int64_t x = k0 + r0 + i;
    dg[i] = A[x * (n + 1)];
  }
  if (q1)
    for (int f = tid; f < P * rcnt; f += nthr) {
      const int i = f / P, r = f - i * P;
      Bq[r * R + i] = p.B[(size_t)(k0 + r0 + i) * P + r];
    }
  int pk = win[0];
  bool first_guard = true;
  __syncthreads();

  int t = 0;
  int end_reason = 0;  // 1: 2x2 defer, 2: q=1 guard defer (for the op counters)
  // Operation counters of the steps (metrics.py:28-43), kept by CTA 0 / thread 0 and committed
  // only when the panel completes (a tripped attempt is relaunched and recharged).
  long long c_mul = 0, c_add = 0, c_div = 0, c_cmp = 0;
  while (t < width && k0 + t < n) {
    if (q1) {
      // ---- q = 1: sketch column argmax (factor.py:607-620), then swap(k, k + jl)
      if (n - (k0 + t) > 1) {
        if (cta == 0 && tid == 0) {  // column_norms of the active sketch (factor.py:608-610)
          const long long mm = n - (k0 + t);
          c_mul += (long long)P * (mm - 1);
          c_add += (long long)P * (mm - 1);
          c_cmp += mm - 1;
        }
        double bk1 = -1.0;
        long long bi1 = LLONG_MAX;
        int bs1 = -1;
        for (int i = tid; i < rcnt; i += nthr) {
          const int lp = lpos[i];
          if (lp < t) continue;
          double am = 0.0;
          for (int r = 0; r < P; ++r) am = fmax(am, fabs(Bq[r * R + i]));
          double nv = 0.0;
          if (am > 0.0) {
            double ss = 0.0;
            for (int r = 0; r < P; ++r) {
              const double x = fabs(Bq[r * R + i]) / am;
              ss = __fma_rn(x, x, ss);
            }
            nv = am * sqrt(ss);
          }
          if (better(nv, lp, bk1, bi1)) {
            bk1 = nv;
            bi1 = lp;
            bs1 = i;
          }
        }
        BlockBest lb1 = block_argmax(bk1, bi1, bs1, par);
        par ^= 1;
        const long long nseq1 = seq + 1;
        const int pb1 = static_cast<int>(nseq1 & 1);
        const unsigned tag1 = static_cast<unsigned>(nseq1);
        if (lb1.slot >= 0) {
          u64* dst = p.qcll + ((size_t)pb1 * G + cta) * QS;
          for (int r = tid; r < P; r += nthr) ll_put_d(dst + 2 * r, tag1, Bq[r * R + lb1.slot]);
        }
        if (tid == 0) {
          u64* q = p.qll + ((size_t)pb1 * G + cta) * kQWords;
          const bool has = lb1.slot >= 0;
          ll_put_d(q, tag1, has ? lb1.key : -1.0);
          ll_put(q + 2, tag1, has ? static_cast<unsigned>(lb1.idx) : 0x7fffffffu);
          ll_put(q + 3, tag1, has ? static_cast<unsigned>(r0 + lb1.slot) : 0xffffffffu);
        }
        seq = nseq1;
        __syncthreads();  // records out before anyone polls
        if (cta == kRed) {
          double gk = -1.0;
          long long gi = LLONG_MAX;
          int gs = -1, gph = -1;
          for (int c = tid; c < G; c += nthr) {
            unsigned w[4];
            if (!ll_read<4>(p.qll + ((size_t)pb1 * G + c) * kQWords, tag1, w)) {
              s_abort = 1;
              continue;
            }
            const double v = ll_d(w[0], w[1]);
            const int ps = static_cast<int>(w[2]);
            if ((v >= 0.0 || v != v) && better(v, ps, gk, gi)) {
              gk = v;
              gi = ps;
              gs = c;
              gph = static_cast<int>(w[3]);
            }
          }
          BlockBest gb = block_argmax(gk, gi, gs, par);
          if (gs >= 0 && gs == gb.slot) {
            // guard (factor.py:613-619): trip -> defer (t > 0) or recompute (t == 0); after a
            // recompute the first check decides "stop"
            unsigned fl = 0;
            if (p.guard_mode != 0 && gb.key < p.guard_limit) {
              if (p.guard_mode == 2 && first_guard) fl = 2;  // stop
              else if (t > 0) fl = 8;                        // defer
              else fl = 1;                                   // trip: recompute
            }
            s_qhdr[0] = static_cast<unsigned>(gs);
            s_qhdr[1] = static_cast<unsigned>(gb.idx);
            s_qhdr[2] = static_cast<unsigned>(gph);
            s_qhdr[3] = fl;
          }
          if (gb.slot < 0 && tid == 0) s_qhdr[3] = 4u;
          __syncthreads();
          unsigned hw[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) hw[u] = s_qhdr[u];
          if (s_abort) hw[3] |= 4u;
          for (int f = tid; f < G * 4; f += nthr) {
            const int c = f >> 2, u = f & 3;
            if (c != kRed) ll_put(p.qdll + ((size_t)pb1 * G + c) * kMWords + u, tag1, hw[u]);
          }
          if (tid == 0) {
            s_gs1 = static_cast<int>(hw[0]);
            s_wpos = static_cast<int>(hw[1]);
            s_wcol = static_cast<int>(hw[2]);
            s_qflags = static_cast<int>(hw[3]);
          }
        } else {
          if (tid < 4) {
            unsigned w[1];
            if (!ll_read<1>(p.qdll + ((size_t)pb1 * G + cta) * kMWords + tid, tag1, w)) {
              s_abort = 1;
              w[0] = 4;
            }
            s_qhdr[tid] = w[0];
          }
          __syncthreads();
          if (tid == 0) {
            s_gs1 = static_cast<int>(s_qhdr[0]);
            s_wpos = static_cast<int>(s_qhdr[1]);
            s_wcol = static_cast<int>(s_qhdr[2]);
            s_qflags = static_cast<int>(s_qhdr[3]) | (s_abort ? 4 : 0);
          }
        }
        par ^= 1;
        __syncthreads();
        first_guard = false;
        if (s_abort || (s_qflags & 4)) {
          if (tid == 0) atomicExch(&p.st->status, 99);
          break;
        }
        if (s_qflags & 8) {  // defer: flush this panel, retest at t == 0
          end_reason = 2;
          break;
        }
        if (s_qflags & 3) {
          if (cta == 0 && tid == 0) p.st->status = (s_qflags & 2) ? 2 : 1;
          s_abort = 2;
          break;
        }
        // pivot sketch column (for the per-step downdate) from the winner's LL buffer
        {
          const u64* src = p.qcll + ((size_t)pb1 * G + s_gs1) * QS;
          for (int r = tid; r < P; r += nthr) {
            unsigned w[2];
            ll_read<2>(src + 2 * r, tag1, w);
            skp0[r] = ll_d(w[0], w[1]);
          }
        }
        // swap(k, k + jl) as bookkeeping
        const int jl = s_wpos, pw = s_wcol;
        if (tid == 0 && jl != t) {
          const int pold = win[t];
          win[t] = pw;
          if (jl < Wn) win[jl] = pold;
          if (pw >= r0 && pw < r0 + rcnt) lpos[pw - r0] = t;
          if (pold >= r0 && pold < r0 + rcnt) lpos[pold - r0] = jl;
        }
        __syncthreads();
      }
      // pivot and its W row: all entries were written before the exchange(s) of this step
      pk = win[t];
      for (int s3 = tid; s3 < t; s3 += nthr) wrow[s3] = __ldcg(p.W + (k0 + pk) + (int64_t)s3 * n);
      __syncthreads();
    }
    // ---- phase A: pivot column (rows of the active block owned here)
    PROF_BEGIN();
    if (tid == 0) {
      s_akk = 0.0;
      s_gerr = 0;
    }
    __syncthreads();
    double bk = -1.0;
    long long bi = LLONG_MAX;
    int bs = -1;
    for (int i = tid; i < rcnt; i += nthr) {
      const int lp = lpos[i];
      if (lp < t) continue;
      const int64_t row = k0 + r0 + i;
      const double av = sym_at(A, n, row, k0 + pk);  // issued before the dot: latency overlaps it
      const double dot = row_dot4(Lsm + i, R, Ls, p.Lbuf + row + (int64_t)k0 * n, n, wrow, t);
      double c = __dsub_rn(av, dot);
      ck[i] = c;
      if (lp > t) {
        double key = fabs(c);
        if (better(key, lp, bk, bi)) {
          bk = key;
          bi = lp;
          bs = i;
        }
      }
      if (r0 + i == pk) s_akk = c;
    }
    PROF_END(2);
    PROF_BEGIN();
    BlockBest lb = block_argmax(bk, bi, bs, par);
    par ^= 1;
    const long long nseq = seq + 1;
    const int pb = static_cast<int>(nseq & 1);
    const unsigned tag = static_cast<unsigned>(nseq);
    if (q1 && lb.slot >= 0) {
      u64* dst = p.qcll + ((size_t)pb * G + cta) * QS;
      for (int r = tid; r < P; r += nthr) ll_put_d(dst + 2 * r, tag, Bq[r * R + lb.slot]);
    }
    if (tid == 0) {
      u64* q = p.xll + ((size_t)pb * G + cta) * kXWords;
      const bool has = lb.slot >= 0;
      ll_put_d(q + 0, tag, has ? lb.key : -1.0);
      ll_put_d(q + 2, tag, has ? ck[lb.slot] : 0.0);
      ll_put_d(q + 4, tag, has ? dg[lb.slot] : 0.0);
      ll_put_d(q + 6, tag, s_akk);
      ll_put(q + 8, tag, has ? static_cast<unsigned>(lb.idx) : 0x7fffffffu);
      ll_put(q + 9, tag, has ? static_cast<unsigned>(r0 + lb.slot) : 0xffffffffu);
      ll_put(q + 10, tag, ((pk >= r0 && pk < r0 + rcnt) ? 1u : 0u) | (s_lerr ? 2u : 0u));
    }
    seq = nseq;
    __syncthreads();  // record out before anyone polls
    PROF_END(8);
    PROF_BEGIN();

    // ---- reducer CTA 0 reads all records and pushes the decision inputs (12 LL words) into
    //      every CTA's mailbox
    if (cta == kRed) {
      double gk = -1.0;
      long long gi = LLONG_MAX;
      int gs = -1;
      XRec mine;
      mine.key = -1.0;
      for (int c = tid; c < G; c += nthr) {
        unsigned w[11];
        if (!ll_read<11>(p.xll + ((size_t)pb * G + c) * kXWords, tag, w)) {
          s_abort = 1;
          continue;
        }
        XRec r;
        r.key = ll_d(w[0], w[1]);
        r.val = ll_d(w[2], w[3]);
        r.diag = ll_d(w[4], w[5]);
        r.akk = ll_d(w[6], w[7]);
        r.lidx = static_cast<int>(w[8]);
        r.phys = static_cast<int>(w[9]);
        r.has_akk = w[10] & 1u;
        r.err = (w[10] >> 1) & 1u;
        if (r.has_akk) s_gakk = r.akk;
        if (r.err) s_gerr = 1;
        if ((r.key >= 0.0 || r.key != r.key) && better(r.key, r.lidx, gk, gi)) {
          gk = r.key;
          gi = r.lidx;
          gs = c;
          mine = r;
        }
      }
      BlockBest gb = block_argmax(gk, gi, gs, par);
      if (gb.slot >= 0 && gs == gb.slot) s_win = mine;  // the thread holding the winning record
      if (tid == 0) s_hascand = gb.slot >= 0 ? 1 : 0;
      __syncthreads();
      {
        unsigned hw[12];
        const u64 kb = static_cast<u64>(__double_as_longlong(s_win.key));
        const u64 vb = static_cast<u64>(__double_as_longlong(s_win.val));
        const u64 db = static_cast<u64>(__double_as_longlong(s_win.diag));
        const u64 ab = static_cast<u64>(__double_as_longlong(s_gakk));
        hw[0] = static_cast<unsigned>(kb);
        hw[1] = static_cast<unsigned>(kb >> 32);
        hw[2] = static_cast<unsigned>(vb);
        hw[3] = static_cast<unsigned>(vb >> 32);
        hw[4] = static_cast<unsigned>(db);
        hw[5] = static_cast<unsigned>(db >> 32);
        hw[6] = static_cast<unsigned>(ab);
        hw[7] = static_cast<unsigned>(ab >> 32);
        hw[8] = static_cast<unsigned>(s_win.lidx);
        hw[9] = static_cast<unsigned>(s_win.phys);
        hw[10] = (s_hascand ? 1u : 0u) | (s_gerr ? 2u : 0u) | (s_abort ? 4u : 0u);
        hw[11] = static_cast<unsigned>(gb.slot);
        for (int f = tid; f < G * 12; f += nthr) {
          const int c = f / 12, u = f - c * 12;
          if (c != kRed) ll_put(p.sdll + ((size_t)pb * G + c) * kMWords + u, tag, hw[u]);
        }
      }
      if (tid == 0) s_gs2 = gb.slot;
      // The decision will need the partner column r unless the 1x1 test passes: start pulling it
      // into L2 now, while the workers are still waiting for this broadcast.
      if (s_hascand && !(fabs(s_gakk) >= __dmul_rn(alpha, s_win.key))) {
        const double* colr = p.A + (int64_t)(k0 + s_win.phys) * n;
        for (int64_t r = k0 + 16 * tid; r < n; r += 16 * nthr) asm volatile("prefetch.global.L2 [%0];" ::"l"(colr + r));
      }
    } else {
      if (tid < 12) {
        unsigned w[1];
        if (!ll_read<1>(p.sdll + ((size_t)pb * G + cta) * kMWords + tid, tag, w)) {
          s_abort = 1;
          w[0] = 0;
        }
        s_dhdr[tid] = w[0];
      }
      __syncthreads();
      if (tid == 0) {
        s_win.key = ll_d(s_dhdr[0], s_dhdr[1]);
        s_win.val = ll_d(s_dhdr[2], s_dhdr[3]);
        s_win.diag = ll_d(s_dhdr[4], s_dhdr[5]);
        s_gakk = ll_d(s_dhdr[6], s_dhdr[7]);
        s_win.lidx = static_cast<int>(s_dhdr[8]);
        s_win.phys = static_cast<int>(s_dhdr[9]);
        s_hascand = s_dhdr[10] & 1u;
        s_gs2 = static_cast<int>(s_dhdr[11]);
        if (s_dhdr[10] & 2u) s_gerr = 1;
        if (s_dhdr[10] & 4u) s_abort = 1;
      }
    }
    par ^= 1;
    __syncthreads();
    PROF_END(3);
    PROF_BEGIN();
    if (s_abort) {
      if (cta == 0 && tid == 0) atomicExch(&p.st->status, 99);
      break;
    }
    if (s_gerr) break;
    const double akk = s_gakk;
    const bool has_cand = s_hascand != 0;
    double lam = 0.0, ckr = 0.0, dr = 0.0;
    int r_rel = -1, pr = -1;
    if (has_cand) {
      lam = s_win.key;
      ckr = s_win.val;
      dr = s_win.diag;
      r_rel = s_win.lidx;
      pr = s_win.phys;
    }

    const double athr = __dmul_rn(alpha, lam);
    // ---- BKPP (pivot.py:146-171): when the 1x1 test fails, form column r in every CTA and find
    //      sigma = max_{i != r} |c_r(i)| with a second exchange; a_rr comes from r's owner.
    bool cr_done = false;
    double sigma = 0.0;
    if (STRAT == 1 && has_cand && lam != 0.0 && !(fabs(akk) >= athr)) {
      for (int s2 = tid; s2 < t; s2 += nthr) wrrow[s2] = __ldcg(p.W + (k0 + pr) + (int64_t)s2 * n);
      const double av0 = (tid < rcnt) ? sym_at(A, n, k0 + r0 + tid, k0 + pr) : 0.0;
      if (tid == 0) s_bkhas = 0;
      __syncthreads();  // wrrow ready
      double sk = -1.0;
      long long si = LLONG_MAX;
      int ss = -1;
      for (int i = tid; i < rcnt; i += nthr) {
        const double a_ip = (i == tid) ? av0 : sym_at(A, n, k0 + r0 + i, k0 + pr);
        const int lp = lpos[i];
        if (lp < t) continue;
        const int64_t row = k0 + r0 + i;
        const double dot = row_dot4(Lsm + i, R, Ls, p.Lbuf + row + (int64_t)k0 * n, n, wrrow, t);
        const double c = __dsub_rn(a_ip, dot);
        cr[i] = c;
        if (r0 + i == pr) {
          s_bkarr = c;
          s_bkhas = 1;
        } else if (better(fabs(c), lp, sk, si)) {
          sk = fabs(c);
          si = lp;
          ss = i;
        }
      }
      const BlockBest lb2 = block_argmax(sk, si, ss, par);
      par ^= 1;
      const long long nseq2 = seq + 1;
      const int pb2 = static_cast<int>(nseq2 & 1);
      const unsigned tag2 = static_cast<unsigned>(nseq2);
      if (tid == 0) {
        u64* q = p.xll + ((size_t)pb2 * G + cta) * kXWords;
        ll_put_d(q + 0, tag2, lb2.slot >= 0 ? lb2.key : -1.0);
        ll_put(q + 2, tag2, lb2.slot >= 0 ? static_cast<unsigned>(lb2.idx) : 0x7fffffffu);
        ll_put_d(q + 3, tag2, s_bkhas ? s_bkarr : 0.0);
        ll_put(q + 5, tag2, s_bkhas ? 1u : 0u);
      }
      seq = nseq2;
      __syncthreads();  // record out before anyone polls
      if (cta == kRed) {
        double gk = -1.0;
        long long gi = LLONG_MAX;
        int gs = -1;
        for (int c = tid; c < G; c += nthr) {
          unsigned w[6];
          if (!ll_read<6>(p.xll + ((size_t)pb2 * G + c) * kXWords, tag2, w)) {
            s_abort = 1;
            continue;
          }
          const double v = ll_d(w[0], w[1]);
          if (w[5]) s_bkarr = ll_d(w[3], w[4]);
          if ((v >= 0.0 || v != v) && better(v, static_cast<int>(w[2]), gk, gi)) {
            gk = v;
            gi = static_cast<int>(w[2]);
            gs = c;
          }
        }
        const BlockBest gb = block_argmax(gk, gi, gs, par);
        __syncthreads();  // s_bkarr from the owner's record
        const u64 kb = static_cast<u64>(__double_as_longlong(gb.slot >= 0 ? gb.key : -1.0));
        const u64 ab = static_cast<u64>(__double_as_longlong(s_bkarr));
        const unsigned hw[5] = {static_cast<unsigned>(kb), static_cast<unsigned>(kb >> 32), static_cast<unsigned>(ab),
                                static_cast<unsigned>(ab >> 32), s_abort ? 4u : 0u};
        for (int f = tid; f < G * 5; f += nthr) {
          const int c = f / 5, u = f - c * 5;
          if (c != kRed) ll_put(p.sdll + ((size_t)pb2 * G + c) * kMWords + u, tag2, hw[u]);
        }
        if (tid < 5) s_dhdr[tid] = hw[tid];
      } else {
        if (tid < 5) {
          unsigned w[1];
          if (!ll_read<1>(p.sdll + ((size_t)pb2 * G + cta) * kMWords + tid, tag2, w)) {
            s_abort = 1;
            w[0] = 4u;
          }
          s_dhdr[tid] = w[0];
        }
      }
      par ^= 1;
      __syncthreads();
      if (s_abort || (s_dhdr[4] & 4u)) {
        if (tid == 0) atomicExch(&p.st->status, 99);
        s_abort = 1;
        break;
      }
      sigma = ll_d(s_dhdr[0], s_dhdr[1]);
      dr = ll_d(s_dhdr[2], s_dhdr[3]);  // a_rr = c_r(r): the 1x1-swap pivot / the 2x2 block's d22
      cr_done = true;
    }

    // pivot-block sources: c0 = the column that ends at position t, c1 = at t + 1 (2x2); their
    // physical rows, W rows and formed values.  Defaults: SBKP / BKPP.
    double* c0v = ck;
    double* c1v = cr;
    const double* c0w = wrow;
    const double* c1w = wrrow;
    int c0phys = pk;
    double d3a = akk, d3b = ckr;  // 2x2 block d11, d21 (d22 = dr)
    int pre_pos = -1, pre_phys = -1;  // bbk: swap(k, p) before swap(k + 1, r) (factor.py:628-629)
    int bbk_kind = -1;
    long long bbk_iters = 0;
    if (STRAT == 2 && has_cand && lam != 0.0 && !(fabs(akk) >= athr)) {
      // ---- BBK rook walk (pivot.py:189-218): form column imax, rowmax = max_{i != imax} |c(i)|
      //      (one exchange per hop); stop at a 1x1-swap (|a_ii| >= alpha rowmax) or a 2x2 (p, imax)
      int ppos = t, pphys = pk, ipos = r_rel, iphys = pr;
      double colmax = lam, app = akk;
      double* cpv = ck;
      const double* cpw = wrow;
      // third column / W-row buffers in global scratch (the rook path is off the rcp critical path)
      double* const cx = p.bkscr + (size_t)cta * (R + Wn);
      double* const wx = cx + R;
      int nb = 0;
      for (long long it = 0; it <= n - (k0 + t); ++it) {
        double* ccv = nb ? cx : cr;
        double* ccw = nb ? wx : wrrow;
        for (int s2 = tid; s2 < t; s2 += nthr) ccw[s2] = __ldcg(p.W + (k0 + iphys) + (int64_t)s2 * n);
        const double av0 = (tid < rcnt) ? sym_at(A, n, k0 + r0 + tid, k0 + iphys) : 0.0;
        if (tid == 0) s_bkhas = 0;
        __syncthreads();  // ccw ready
        double sk = -1.0;
        long long si = LLONG_MAX;
        int ss = -1;
        for (int i = tid; i < rcnt; i += nthr) {
          const double a_ip = (i == tid) ? av0 : sym_at(A, n, k0 + r0 + i, k0 + iphys);
          const int lp = lpos[i];
          if (lp < t) continue;
          const int64_t row = k0 + r0 + i;
          const double dot = row_dot4(Lsm + i, R, Ls, p.Lbuf + row + (int64_t)k0 * n, n, ccw, t);
          const double c = __dsub_rn(a_ip, dot);
          ccv[i] = c;
          if (r0 + i == iphys) {
            s_bkarr = c;
            s_bkcp = cpv[i];
            s_bkhas = 1;
          } else if (better(fabs(c), lp, sk, si)) {
            sk = fabs(c);
            si = lp;
            ss = i;
          }
        }
        const BlockBest lb2 = block_argmax(sk, si, ss, par);
        par ^= 1;
        const long long nseq2 = seq + 1;
        const int pb2 = static_cast<int>(nseq2 & 1);
        const unsigned tag2 = static_cast<unsigned>(nseq2);
        if (tid == 0) {
          u64* q = p.xll + ((size_t)pb2 * G + cta) * kXWords;
          const bool hv = lb2.slot >= 0;
          ll_put_d(q + 0, tag2, hv ? lb2.key : -1.0);
          ll_put(q + 2, tag2, hv ? static_cast<unsigned>(lb2.idx) : 0x7fffffffu);
          ll_put(q + 3, tag2, hv ? static_cast<unsigned>(r0 + lb2.slot) : 0xffffffffu);
          ll_put_d(q + 4, tag2, s_bkhas ? s_bkarr : 0.0);
          ll_put_d(q + 6, tag2, s_bkhas ? s_bkcp : 0.0);
          ll_put(q + 8, tag2, s_bkhas ? 1u : 0u);
        }
        seq = nseq2;
        __syncthreads();  // record out before anyone polls
        if (cta == kRed) {
          double gk = -1.0;
          long long gi = LLONG_MAX;
          int gs = -1;
          unsigned gph = 0;
          for (int c = tid; c < G; c += nthr) {
            unsigned w[9];
            if (!ll_read<9>(p.xll + ((size_t)pb2 * G + c) * kXWords, tag2, w)) {
              s_abort = 1;
              continue;
            }
            const double v = ll_d(w[0], w[1]);
            if (w[8]) {
              s_bkarr = ll_d(w[4], w[5]);
              s_bkcp = ll_d(w[6], w[7]);
            }
            if ((v >= 0.0 || v != v) && better(v, static_cast<int>(w[2]), gk, gi)) {
              gk = v;
              gi = static_cast<int>(w[2]);
              gs = c;
              gph = w[3];
            }
          }
          const BlockBest gb = block_argmax(gk, gi, gs, par);
          if (gs >= 0 && gs == gb.slot) s_bkjph = static_cast<int>(gph);
          __syncthreads();
          const u64 kb = static_cast<u64>(__double_as_longlong(gb.slot >= 0 ? gb.key : -1.0));
          const u64 ab = static_cast<u64>(__double_as_longlong(s_bkarr));
          const u64 cb = static_cast<u64>(__double_as_longlong(s_bkcp));
          const unsigned hw[9] = {static_cast<unsigned>(kb), static_cast<unsigned>(kb >> 32),
                                  gb.slot >= 0 ? static_cast<unsigned>(gb.idx) : 0x7fffffffu,
                                  gb.slot >= 0 ? static_cast<unsigned>(s_bkjph) : 0xffffffffu,
                                  static_cast<unsigned>(ab), static_cast<unsigned>(ab >> 32),
                                  static_cast<unsigned>(cb), static_cast<unsigned>(cb >> 32), s_abort ? 4u : 0u};
          for (int f = tid; f < G * 9; f += nthr) {
            const int c = f / 9, u = f - c * 9;
            if (c != kRed) ll_put(p.sdll + ((size_t)pb2 * G + c) * kMWords + u, tag2, hw[u]);
          }
          if (tid < 9) s_dhdr[tid] = hw[tid];
        } else {
          if (tid < 9) {
            unsigned w[1];
            if (!ll_read<1>(p.sdll + ((size_t)pb2 * G + cta) * kMWords + tid, tag2, w)) {
              s_abort = 1;
              w[0] = 4u;
            }
            s_dhdr[tid] = w[0];
          }
        }
        par ^= 1;
        __syncthreads();
        if (s_abort || (s_dhdr[8] & 4u)) {
          bbk_kind = -2;
          break;
        }
        ++bbk_iters;
        const double rowmax = ll_d(s_dhdr[0], s_dhdr[1]);
        const int jpos = static_cast<int>(s_dhdr[2]);
        const int jphys = static_cast<int>(s_dhdr[3]);
        const double aii = ll_d(s_dhdr[4], s_dhdr[5]);
        const double cpi = ll_d(s_dhdr[6], s_dhdr[7]);
        __syncthreads();  // s_dhdr / s_bk* reused by the next hop
        if (fabs(aii) >= __dmul_rn(alpha, rowmax)) {  // 1x1 with swap(k, imax)
          bbk_kind = 2;
          c0v = ccv;
          c0w = ccw;
          c0phys = iphys;
          dr = aii;
          r_rel = ipos;
          pr = iphys;
          break;
        }
        if (jpos == ppos || rowmax <= colmax) {  // 2x2 (p, imax)
          bbk_kind = 3;
          c0v = cpv;
          c0w = cpw;
          c0phys = pphys;
          c1v = ccv;
          c1w = ccw;
          d3a = app;
          d3b = cpi;
          dr = aii;
          r_rel = ipos;
          pr = iphys;
          if (ppos != t) {
            pre_pos = ppos;
            pre_phys = pphys;
          }
          if (ipos == t) bbk_kind = -3;  // walk returned to k with a 2x2: not supported (ties only)
          break;
        }
        ppos = ipos;  // hop: p <- imax, imax <- jmax
        pphys = iphys;
        cpv = ccv;
        cpw = ccw;
        app = aii;
        colmax = rowmax;
        ipos = jpos;
        iphys = jphys;
        nb ^= 1;
      }
      if (bbk_kind < 0) {
        if (tid == 0) atomicExch(&p.st->status, bbk_kind == -3 ? 96 : 99);
        s_abort = 1;
        break;
      }
      cr_done = true;
    }

    // ---- decision: 0 skip, 1 1x1, 2 1x1-swap r, 3 2x2 (k, r)
    //      SBKP (pivot.py:111-128), BKPP (pivot.py:146-171) or BBK (pivot.py:189-218)
    int kind, s;
    if (!has_cand || lam == 0.0) {
      kind = 0;
      s = 1;
    } else if (fabs(akk) >= athr) {
      kind = 1;
      s = 1;
    } else if (STRAT == 2) {
      kind = bbk_kind;
      s = kind == 3 ? 2 : 1;
    } else if (STRAT == 1) {
      if (__dmul_rn(fabs(akk), sigma) >= __dmul_rn(athr, lam)) {
        kind = 1;
        s = 1;
      } else if (fabs(dr) >= __dmul_rn(alpha, sigma)) {
        kind = 2;
        s = 1;
      } else {
        kind = 3;
        s = 2;
      }
    } else if (fabs(dr) >= athr) {
      kind = 2;
      s = 1;
    } else {
      kind = 3;
      s = 2;
    }
    const bool deferred = s == 2 && t > 0 && t + 2 > width;
    if (cta == 0 && tid == 0) {
      // _decide: form column k, scan, diag of r (factor.py:350-367, 414-427)
      const long long mm = n - (k0 + t);
      const long long colc = t > 0 ? (long long)t * mm : 0;
      c_mul += colc;
      c_add += colc;
      c_cmp += mm >= 2 ? mm - 2 : 0;
      if (STRAT == 2) {  // each rook hop: _form_column(imax) + its scan (pivot.py:207-213)
        c_mul += colc * bbk_iters;
        c_add += colc * bbk_iters;
        c_cmp += (mm >= 2 ? mm - 2 : 0) * bbk_iters;
      } else if (STRAT == 1) {
        if (cr_done) {  // _form_column(r) + the scan for sigma (pivot.py:162-166)
          c_mul += colc;
          c_add += colc;
          c_cmp += mm >= 2 ? mm - 2 : 0;
        }
      } else if (kind >= 2 && t > 0) {  // _diag_entry(r)
        c_mul += t;
        c_add += t;
      }
      if (!deferred) {  // _eliminate re-forms the column(s) (factor.py:449-489)
        c_mul += colc * s;
        c_add += colc * s;
        const long long w = mm - s;
        if (kind != 0) {
          if (s == 1) {
            c_div += w;
          } else {
            c_div += 2 * w;
            c_mul += 4 * w + 2;
            c_add += 2 * w + 1;
          }
        }
        if (q1 && w > 0) {
          c_mul += (long long)s * P * w;
          c_add += (long long)s * P * w;
        }
      }
    }
    if (deferred) {  // defer (factor.py:622-623)
      end_reason = 1;
      break;
    }

    // ---- symmetric swaps as permutation bookkeeping (factor.py:624-630)
    int p_t = pk, p_t1 = -1;
    if (kind == 3 && pre_pos >= 0) {  // bbk: swap(k, p) first (factor.py:628-629)
      if (tid == 0) {
        const int col_t = win[t];
        win[t] = pre_phys;
        if (pre_pos < Wn) win[pre_pos] = col_t;
        if (pre_phys >= r0 && pre_phys < r0 + rcnt) lpos[pre_phys - r0] = t;
        if (col_t >= r0 && col_t < r0 + rcnt) lpos[col_t - r0] = pre_pos;
      }
      p_t = pre_phys;
    }
    if (kind == 2) {  // swap(k, r)
      if (tid == 0) {
        win[t] = pr;
        if (r_rel < Wn) win[r_rel] = pk;
        if (pr >= r0 && pr < r0 + rcnt) lpos[pr - r0] = t;
        if (pk >= r0 && pk < r0 + rcnt) lpos[pk - r0] = r_rel;
      }
      p_t = pr;
    } else if (kind == 3) {  // swap(k+1, r)
      if (r_rel != t + 1 && tid == 0) {
        const int p1 = win[t + 1];  // (after the bbk swap(k, p), which never touches r's position)
        win[t + 1] = pr;
        if (r_rel < Wn) win[r_rel] = p1;
        if (pr >= r0 && pr < r0 + rcnt) lpos[pr - r0] = t + 1;
        if (p1 >= r0 && p1 < r0 + rcnt) lpos[p1 - r0] = r_rel;
      }
      p_t1 = pr;
    }

    // ---- phase B: partner column when needed, multipliers, writes
    const int64_t kglob = k0 + t;
    if (kind >= 2 && !cr_done) {
      for (int s2 = tid; s2 < t; s2 += nthr) wrrow[s2] = __ldcg(p.W + (k0 + pr) + (int64_t)s2 * n);
      if (q1) {  // partner's sketch column (per-step downdate, factor.py:486-489)
        const u64* src = p.qcll + ((size_t)pb * G + s_gs2) * QS;
        for (int r = tid; r < P; r += nthr) {
          unsigned w[2];
          ll_read<2>(src + 2 * r, tag, w);
          skr[r] = ll_d(w[0], w[1]);
        }
      }
      const double av0 = (tid < rcnt) ? sym_at(A, n, k0 + r0 + tid, k0 + pr) : 0.0;
      __syncthreads();  // wrrow ready, swaps (lpos) visible
      for (int i = tid; i < rcnt; i += nthr) {
        const double a_ip = (i == tid) ? av0 : sym_at(A, n, k0 + r0 + i, k0 + pr);
        if (lpos[i] < t) continue;
        const int64_t row = k0 + r0 + i;
        const double dot = row_dot4(Lsm + i, R, Ls, p.Lbuf + row + (int64_t)k0 * n, n, wrrow, t);
        cr[i] = __dsub_rn(a_ip, dot);
      }
    }
    // D block and its checks (factor.py:202-226, 455-466) — identical in every CTA
    double d11 = 0.0, d21 = 0.0, d22 = 0.0, det = 1.0;
    int num_kind = 0;
    if (kind <= 1) {
      d11 = akk;
      if (!isfinite(d11)) num_kind = 3;
    } else if (kind == 2) {
      d11 = dr;
      if (!isfinite(d11)) num_kind = 3;
    } else {
      d11 = d3a;
      d21 = d3b;
      d22 = dr;
      det = __dsub_rn(__dmul_rn(d11, d22), __dmul_rn(d21, d21));
      if (det == 0.0) {
        num_kind = 2;
      } else if (!isfinite(d11) || !isfinite(d21) || !isfinite(d22)) {
        num_kind = 3;
      } else {
        double a21 = fabs(d21);
        double dt = __dsub_rn(__dmul_rn(d11, d22), __dmul_rn(a21, a21));
        double bound = __dmul_rn(__dmul_rn(__dmul_rn(__dsub_rn(1.0, __dmul_rn(alpha, alpha)), a21), a21),
                                 __dsub_rn(1.0, 1e-12));
        if (fabs(dt) < bound) num_kind = 4;
      }
    }
    if (num_kind != 0) {
      if (cta == 0 && tid == 0) atomicMin(&p.st->err, (kglob << 8) | num_kind);
      break;
    }
    __syncthreads();  // cr complete; lpos / win updates visible
    bool lerr = false;
    for (int i = tid; i < rcnt; i += nthr) {
      const int lp = lpos[i];
      if (lp < t) continue;
      const int64_t row = k0 + r0 + i;
      if (kind <= 1) {
        const double c = c0v[i];
        p.W[row + (int64_t)t * n] = c;
        if (lp > t) {
          double l = (kind == 0) ? 0.0 : __ddiv_rn(c, d11);
          if (!isfinite(l)) lerr = true;
          p.Lbuf[row + kglob * n] = l;
          if (t < Ls) Lsm[(size_t)t * R + i] = l;
          dg[i] = __fma_rn(-l, c, dg[i]);
          if (q1)
            for (int r = 0; r < P; ++r) Bq[r * R + i] = __dsub_rn(Bq[r * R + i], __dmul_rn(skp0[r], l));
        }
      } else if (kind == 2) {
        const double c = (STRAT == 2 ? c0v : cr)[i];
        p.W[row + (int64_t)t * n] = c;
        if (lp > t) {
          double l = __ddiv_rn(c, d11);
          if (!isfinite(l)) lerr = true;
          p.Lbuf[row + kglob * n] = l;
          if (t < Ls) Lsm[(size_t)t * R + i] = l;
          dg[i] = __fma_rn(-l, c, dg[i]);
          if (q1)
            for (int r = 0; r < P; ++r) Bq[r * R + i] = __dsub_rn(Bq[r * R + i], __dmul_rn(skr[r], l));
        }
      } else {
        const double c0 = c0v[i], c1 = c1v[i];
        p.W[row + (int64_t)t * n] = c0;
        p.W[row + (int64_t)(t + 1) * n] = c1;
        if (lp > t + 1) {
          double l1 = __ddiv_rn(__dsub_rn(__dmul_rn(c0, d22), __dmul_rn(d21, c1)), det);
          double l2 = __ddiv_rn(__dsub_rn(__dmul_rn(d11, c1), __dmul_rn(d21, c0)), det);
          if (!isfinite(l1) || !isfinite(l2)) lerr = true;
          p.Lbuf[row + kglob * n] = l1;
          p.Lbuf[row + (kglob + 1) * n] = l2;
          if (t < Ls) Lsm[(size_t)t * R + i] = l1;
          if (t + 1 < Ls) Lsm[(size_t)(t + 1) * R + i] = l2;
          dg[i] = __fma_rn(-l2, c1, __fma_rn(-l1, c0, dg[i]));
          if (q1)
            for (int r = 0; r < P; ++r)
              Bq[r * R + i] = __dsub_rn(Bq[r * R + i], __dadd_rn(__dmul_rn(skp0[r], l1), __dmul_rn(skr[r], l2)));
        } else if (lp == t + 1) {
          // partner row of the 2x2 block: L[k+1, k] is exactly zero
          p.Lbuf[row + kglob * n] = 0.0;
          if (t < Ls) Lsm[(size_t)t * R + i] = 0.0;
        }
      }
    }
    if (lerr) {
      atomicMin(&p.st->err, (kglob << 8) | 3);
      s_lerr = 1;
    }
    if (cta == 0 && tid == 0) {
      p.d_diag[kglob] = d11;
      p.d_off[kglob] = (kind == 3) ? d21 : 0.0;
      p.pattern[kglob] = (kind == 3) ? 1 : 0;
      p.perm_out[kglob] = p.perm_cur[k0 + p_t];
      if (kind == 3) {
        p.d_diag[kglob + 1] = d22;
        p.d_off[kglob + 1] = 0.0;
        p.pattern[kglob + 1] = 2;
        p.perm_out[kglob + 1] = p.perm_cur[k0 + p_t1];
      }
      if (p.trace_kind) {
        p.trace_kind[kglob] = static_cast<int8_t>(kind);
        p.trace_r[kglob] = (kind >= 2) ? (k0 + r_rel) : -1;
      }
      p.st->n_steps += 1;
      if (kind == 3) p.st->n_2x2 += 1;
    }
    PROF_END(4);

    // ---- next pivot: its W row (older entries from memory, this step's entries recomputed
    //      redundantly with the owner's exact arithmetic from an smem copy of its L row)
    PROF_BEGIN();
    const int tn = t + s;
    if (!q1 && tn < width && k0 + tn < n) {
      const int pn = win[tn];  // win updated by tid 0 before the barrier above
      const int64_t rown = k0 + pn;
      for (int s3 = tid; s3 < t; s3 += nthr) {
        lnext[s3] = __ldcg(p.Lbuf + rown + (int64_t)(k0 + s3) * n);
        wnext[s3] = __ldcg(p.W + rown + (int64_t)s3 * n);
      }
      const double an0 = (tid == 0) ? sym_at(A, n, rown, k0 + (kind == 2 ? pr : c0phys)) : 0.0;
      const double an1 = (tid == 4 && kind == 3) ? sym_at(A, n, rown, k0 + pr) : 0.0;
      __syncthreads();
      if (tid < 32) {
        // chain_dot4 split over lanes: lane q (q < 4) accumulates chain q of the c0 dot, lanes 4..7
        // the c1 dot (2x2); same terms, same order, same ((c0+c1)+(c2+c3)) combination
        const int q = tid & 3;
        const double* wsel = (tid >= 4) ? c1w : (kind == 2 ? (STRAT == 2 ? c0w : wrrow) : c0w);
        double c = 0.0;
        if (tid < 8)
          for (int s3 = q; s3 < t; s3 += 4) c = __fma_rn(lnext[s3], wsel[s3], c);
        const double pr1 = __dadd_rn(c, __shfl_xor_sync(0xffffffffu, c, 1));
        const double tot = __dadd_rn(pr1, __shfl_xor_sync(0xffffffffu, pr1, 2));
        if (tid == 0) wnext[t] = __dsub_rn(an0, tot);
        if (tid == 4 && kind == 3) wnext[t + 1] = __dsub_rn(an1, tot);
      }
      __syncthreads();
      for (int s3 = tid; s3 < tn; s3 += nthr) wrow[s3] = wnext[s3];
      pk = pn;
    }
    t = tn;
    __syncthreads();
    PROF_END(5);
  }

  // ---- q = 1: the updated sketch of the rows still active, in the new logical order
  if (q1 && s_abort == 0)
    for (int f = tid; f < P * rcnt; f += nthr) {
      const int i = f / P, r = f - i * P;
      if (lpos[i] >= t) p.Bout[(size_t)(k0 + lpos[i]) * P + r] = Bq[r * R + i];
    }
  // ---- publish the panel's permutation and outcome
  for (int i = tid; i < rcnt; i += nthr) {
    const int lp = lpos[i];
    p.log_of_phys[k0 + r0 + i] = k0 + lp;
    p.phys_of_log[k0 + lp] = k0 + r0 + i;
  }
  if (cta == 0 && tid == 0) {
    p.st->seq = seq;
    p.st->k_end = k0 + t;
    p.st->t_end = t;
    p.st->end_reason = end_reason;
    if (s_abort == 0) {
      p.st->cnt[0] += c_mul;
      p.st->cnt[1] += c_add;
      p.st->cnt[2] += c_div;
      p.st->cnt[3] += c_cmp;
    }
  }
  if (prof) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->cyc[7]), (unsigned long long)(prof_now() - c_kernel0));
  __syncthreads();
  stamp_end(ts_panel ? ts_panel + 1 : nullptr);
#undef PROF_BEGIN
#undef PROF_END
}

// Finalises panel desc_in (ok, k_end, t) for the gather / Schur / sketch kernels of the same
// panel, logs it, and writes the next panel's descriptor.  Guard events and numerical errors
// stop the chain (run = 0) and record the panel index for the host.
__global__ void panel_commit_kernel(PanelDesc* din, PanelDesc* dout, PanelLog* plog, PanelState* st, int64_t n,
                                    int b, int q, int P, long long snap_cap) {
  const PanelDesc d = *din;
  PanelDesc o = d;
  o.run = 0;
  o.ok = 0;
  o.pidx = d.pidx + 1;
  if (!d.run) {
    din->ok = 0;
    *dout = o;
    return;
  }
  if (st->status != 0 || st->err != LLONG_MAX) {
    din->ok = 0;
    if (st->stop_pidx < 0) st->stop_pidx = d.pidx;
    *dout = o;
    return;
  }
  const int k_end = st->k_end, t = st->t_end;
  const int m0 = (int)(n - d.k0);
  const int width = m0 < b ? m0 : b;
  int qn = 0;
  if (q > 1 && m0 > 1) {
    qn = q < width ? q : width;
    qn = qn < m0 ? qn : m0;
    qn = qn < P ? qn : P;
  }
  din->k_end = k_end;
  din->t = t;
  din->ok = 1;
  plog[d.pidx] = PanelLog{d.k0, k_end, m0, qn, d.snap_off};
  st->panels_done = d.pidx + 1;
  o.k0 = k_end;
  o.snap_off = d.snap_off + m0;
  o.run = (k_end < n) ? 1 : 0;
  if (o.snap_off + (n - k_end) > snap_cap) {  // cannot happen (every panel eliminates a column)
    st->status = 97;
    if (st->stop_pidx < 0) st->stop_pidx = d.pidx + 1;
    o.run = 0;
  }
  *dout = o;
}

cudaError_t launch_panel_commit(PanelDesc* din, PanelDesc* dout, PanelLog* plog, PanelState* st, int64_t n, int b,
                                int q, int P, long long snap_cap, cudaStream_t stream) {
  panel_commit_kernel<<<1, 1, 0, stream>>>(din, dout, plog, st, n, b, q, P, snap_cap);
  return cudaGetLastError();
}

cudaError_t panel_init_attributes(int max_dyn_smem) {
  cudaError_t e = cudaFuncSetAttribute(panel_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(panel_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(panel_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem);
  return e;
}

int panel_static_smem_bytes() {
  cudaFuncAttributes attr;
  int mx = 0;
  if (cudaFuncGetAttributes(&attr, panel_kernel<0>) != cudaSuccess) return 4096;
  mx = static_cast<int>(attr.sharedSizeBytes);
  if (cudaFuncGetAttributes(&attr, panel_kernel<1>) != cudaSuccess) return 4096;
  mx = mx > static_cast<int>(attr.sharedSizeBytes) ? mx : static_cast<int>(attr.sharedSizeBytes);
  if (cudaFuncGetAttributes(&attr, panel_kernel<2>) != cudaSuccess) return 4096;
  mx = mx > static_cast<int>(attr.sharedSizeBytes) ? mx : static_cast<int>(attr.sharedSizeBytes);
  return mx;
}

cudaError_t launch_panel(const PanelParams& prm, int G, size_t smem, cudaStream_t st) {
  PanelParams copy = prm;
  void* args[] = {&copy};
  const void* fn = prm.strategy == 2   ? reinterpret_cast<const void*>(panel_kernel<2>)
                   : prm.strategy == 1 ? reinterpret_cast<const void*>(panel_kernel<1>)
                                       : reinterpret_cast<const void*>(panel_kernel<0>);
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kPanelThreads), args, smem, st);
}

}  // namespace rcp
