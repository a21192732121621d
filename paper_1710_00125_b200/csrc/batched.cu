// Batched RCP factorization of many small symmetric matrices (BASELINE config C5:
// 65536 x n = 256, b = q = 16, P = 24), plus the matching batched solve.
//
// Same algorithm as the single-matrix driver (capi.cu + panel.cu), re-laid out for a
// matrix that one CTA can own: every synchronisation is a CTA barrier, nothing goes back
// to the host, and one persistent grid (two CTAs per SM) pulls matrices from an atomic
// counter.  Thread i of the CTA owns logical row/column i of its matrix:
//   * the sketch column B[:, i] lives in thread i's registers (x[]), so QRCP
//     (sketch.py:135-169) is register-resident and swaps move registers via smem;
//   * the panel's L and W columns (factor.py:350-367, W = unscaled columns) live in smem;
//   * the trailing matrix lives in per-CTA global scratch (L2-resident) in the panel's
//     start order; inside a panel symmetric swaps (factor.py:333-348) are bookkeeping
//     (pol[]), and the trailing update (factor.py:369-379) gathers through it while
//     writing the next panel's compact trailing block (lower triangle only; reads of the
//     upper part go through the transposed index);
//   * L columns are stored keyed by the ORIGINAL row index, so later row swaps never move
//     them; the final L (final pivot order) is one coalesced row gather.
// The decision logic (first-index argmax, thresholds, alpha, defer rule, 2x2 formulas with
// IEEE division and no FMA contraction, the checks of factor.py:455-466, the guard with
// the continuing normal stream) follows the reference line by line; see panel.cu for the
// corresponding cross-references.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "../../include/rcp_b200.h"
#include "rcp_common.cuh"

#ifndef RCP_BATCH_PROF
#define RCP_BATCH_PROF 0
#endif

using namespace rcp;

namespace {

constexpr int BT = 256;  // threads per CTA == largest supported n
constexpr int BW = BT / 32;
constexpr int kMaxB = 32;
constexpr int kMaxThr = 24;  // guard thresholds precomputed on the host

struct BatchParams {
  int count, n, P, b, q, armed;
  double alpha;
  double thr[kMaxThr];  // thr[j] = eps ** ((j + 1) / robust_r)  (factor.py:316, 406), host pow
  const double* A;
  int64_t lda, a_stride;
  const double* omegaT;  // n x PM (zero padded): omegaT[j * PM + r] = Omega[r, j]
  const double* z;       // normal stream; z[0, P n) = Omega row-major
  int64_t z_len;
  double* ws;
  int64_t ws_stride;  // doubles per CTA
  int64_t* perm;
  double* L;
  double* d_diag;
  double* d_off;
  int8_t* pattern;
  rcp_batch_stats* mstats;
  int* next;
  int dbg;  // debug: stop after stage dbg (0 = off)
};

struct Shm {
  double* Lp;   // b columns x BT
  double* Wp;   // (b + 1) columns x BT
  double* scr;  // aliases Lp/Wp: QRCP register exchange (P x BT)
  double* c0s;  // formed pivot column
  double* xs;   // 2 x PM: swap exchange of sketch columns
  double* vsh;  // Householder vector + coefficient
  double* B1s;  // P x b
  double* Ys;   // P x b
  double* redk;
  double* cand;  // 2 x BW x (PM + 2): per-warp QRCP candidate reflectors (double-buffered)
  int* redi;
  int* pol;    // logical position -> storage index (relative to the panel start)
  int* permv;  // logical position -> original index
};

// Block-wide first-index argmax (numpy semantics); one barrier; result in every thread.
__device__ __forceinline__ void bargmax(double& key, int& idx, const Shm& S, int& par) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double k2 = __shfl_down_sync(0xffffffffu, key, o);
    const int i2 = __shfl_down_sync(0xffffffffu, idx, o);
    if (better(k2, i2, key, idx)) {
      key = k2;
      idx = i2;
    }
  }
  if (lane == 0) {
    S.redk[par * BW + warp] = key;
    S.redi[par * BW + warp] = idx;
  }
  __syncthreads();
  key = S.redk[par * BW];
  idx = S.redi[par * BW];
#pragma unroll
  for (int w = 1; w < BW; ++w) {
    const double k2 = S.redk[par * BW + w];
    const int i2 = S.redi[par * BW + w];
    if (better(k2, i2, key, idx)) {
      key = k2;
      idx = i2;
    }
  }
  par ^= 1;
}

__device__ __forceinline__ double bmax(double v, const Shm& S, int& par) {
  int idx = 0;
  bargmax(v, idx, S, par);
  return v;
}

// Scaled Euclidean norm of x[lo, P) (core.py:122-142).
template <int PM>
__device__ __forceinline__ double sc_norm(const double (&x)[PM], int lo, int P) {
  double am = 0.0;
#pragma unroll
  for (int r = 0; r < PM; ++r)
    if (r >= lo && r < P) am = fmax(am, fabs(x[r]));
  if (!(am > 0.0)) return 0.0;
  double ss = 0.0;
#pragma unroll
  for (int r = 0; r < PM; ++r)
    if (r >= lo && r < P) {
      const double v = fabs(x[r]) / am;
      ss = __fma_rn(v, v, ss);
    }
  return am * sqrt(ss);
}

// Residual column norm for the QRCP pivot choice: plain sqrt(sum x^2) when that is safe
// from overflow/underflow, the scaled form of core.py:122-142 otherwise (same ordering up
// to rounding; exact ties, e.g. zero columns, stay exact ties).
template <int PM>
__device__ __forceinline__ double res_norm(const double (&x)[PM], int lo, int P) {
  double ss = 0.0;
#pragma unroll
  for (int r = 0; r < PM; ++r)
    if (r >= lo && r < P) ss = __fma_rn(x[r], x[r], ss);
  if (ss == 0.0) return 0.0;
  if (ss >= 1e-280 && ss <= 1e280) return sqrt(ss);
  return sc_norm<PM>(x, lo, P);
}

// c = Lp[:, row] . Wp[:, col] over the first t panel columns (fixed order, every caller
// that needs the same value gets the same bits).
__device__ __forceinline__ double panel_dot(const double* Lp, const double* Wp, int row, int col, int t) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int s = 0;
  for (; s + 4 <= t; s += 4) {
    a0 = __fma_rn(Lp[s * BT + row], Wp[s * BT + col], a0);
    a1 = __fma_rn(Lp[(s + 1) * BT + row], Wp[(s + 1) * BT + col], a1);
    a2 = __fma_rn(Lp[(s + 2) * BT + row], Wp[(s + 2) * BT + col], a2);
    a3 = __fma_rn(Lp[(s + 3) * BT + row], Wp[(s + 3) * BT + col], a3);
  }
  if (s < t) a0 = __fma_rn(Lp[s * BT + row], Wp[s * BT + col], a0);
  if (s + 1 < t) a1 = __fma_rn(Lp[(s + 1) * BT + row], Wp[(s + 1) * BT + col], a1);
  if (s + 2 < t) a2 = __fma_rn(Lp[(s + 2) * BT + row], Wp[(s + 2) * BT + col], a2);
  return (a0 + a1) + (a2 + a3);
}

template <int PM, int MINB>
__global__ void __launch_bounds__(BT, MINB) batched_factor_kernel(BatchParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int n = p.n, P = p.P, b = p.b;
  const int SC = max(2 * b + 1, PM);
  Shm S;
  {
    double* d = reinterpret_cast<double*>(smem_raw);
    S.Lp = d;
    S.Wp = d + (size_t)b * BT;
    S.scr = d;
    d += (size_t)SC * BT;
    S.c0s = d;
    d += BT;
    S.xs = d;
    d += 2 * PM;
    S.vsh = d;
    d += PM + 2;
    S.B1s = d;
    d += PM * b;
    S.Ys = d;
    d += PM * b;
    S.redk = d;
    d += 2 * BW;
    S.cand = d;
    d += 2 * BW * (PM + 2);
    int* ip = reinterpret_cast<int*>(d);
    S.redi = ip;
    ip += 2 * BW;
    S.pol = ip;
    ip += BT;
    S.permv = ip;
  }
  __shared__ int s_mat, s_skip;
  __shared__ double s_tsw[2];
  double* ws = p.ws + (size_t)blockIdx.x * (size_t)p.ws_stride;
  double* Abuf[2] = {ws, ws + (size_t)n * n};
  double* Lst = ws + 2 * (size_t)n * n;  // L entries keyed by (original row, column)
  double* Bx = ws + 3 * (size_t)n * n;   // sketch, P x n (ld n)
  const double alpha = p.alpha;
  const int i = tid;  // owned logical row / column
  const bool live = i < n;
  int par = 0;

  for (;;) {
    __syncthreads();
    if (tid == 0) s_mat = atomicAdd(p.next, 1);
    __syncthreads();
    const int mat = s_mat;
    if (mat >= p.count) break;
    const double* A = p.A + (size_t)mat * (size_t)p.a_stride;
    const int64_t lda = p.lda;
    int64_t* perm_o = p.perm + (size_t)mat * n;
    double* Lo = p.L + (size_t)mat * n * n;
    double* dd = p.d_diag + (size_t)mat * n;
    double* dof = p.d_off + (size_t)mat * n;
    int8_t* pat = p.pattern + (size_t)mat * n;
    rcp_batch_stats* ms = p.mstats + mat;

#if RCP_BATCH_PROF
    long long pf[4] = {0, 0, 0, 0}, pf_t = clock64();
#define PF(k)                         \
  {                                   \
    const long long now_ = clock64(); \
    pf[k] += now_ - pf_t;             \
    pf_t = now_;                      \
  }
#else
#define PF(k)
#endif
    // ---- input checks (core.py:48-53, factor.py:280-281) and max|A|
    int asym = 0, nonfin = 0;
    double mx = 0.0;
    if (live) {
#pragma unroll 8
      for (int j = 0; j < n; ++j) {
        const double v = A[(size_t)j * lda + i];  // (i, j)
        const double w = A[(size_t)i * lda + j];  // (j, i)
        asym |= !(v == w);
        nonfin |= !isfinite(v);
        mx = fmax(mx, fabs(v));
      }
    }
    asym = __syncthreads_or(asym);
    nonfin = __syncthreads_or(nonfin);
    if (asym || nonfin) {
      if (tid == 0) {
        rcp_batch_stats z{};
        z.status = asym ? RCP_ERR_NOT_SYMMETRIC : RCP_ERR_NONFINITE_INPUT;
        z.deficient_from = -1;
        *ms = z;
      }
      continue;
    }
    const double amax = bmax(mx, S, par);
    if (p.dbg == 1) continue;

    // ---- B = Omega A (factor.py:307-309): thread i forms sketch column i
    // the sketch lives in per-CTA global scratch Bx[r * n + i] (L1/L2-resident), loaded into
    // registers only for the QRCP of each panel
    double nrm0 = 0.0;
    {
      double x[PM];
#pragma unroll
      for (int r = 0; r < PM; ++r) x[r] = 0.0;
      if (live) {
        for (int j = 0; j < n; ++j) {
          const double a = A[(size_t)j * lda + i];  // A[j, i] (symmetric: coalesced)
          const double* om = p.omegaT + (size_t)j * PM;
#pragma unroll
          for (int r = 0; r < PM; r += 2) {
            const double2 o2 = __ldg(reinterpret_cast<const double2*>(om + r));
            x[r] = __fma_rn(o2.x, a, x[r]);
            x[r + 1] = __fma_rn(o2.y, a, x[r + 1]);
          }
        }
#pragma unroll
        for (int r = 0; r < PM; ++r)
          if (r < P) Bx[(size_t)r * n + i] = x[r];
        nrm0 = sc_norm<PM>(x, 0, P);
      }
    }
    const double beta = p.armed ? bmax(nrm0, S, par) : 0.0;

    if (p.dbg == 2) continue;
    if (live) S.permv[i] = i;
    int c_mul = 0, c_add = 0, c_div = 0, c_cmp = 0;  // thread 0's op counters (n <= 256: < 2^31)
    int64_t zoff = (int64_t)P * n;
    int recomputes = 0, n2x2 = 0, nsteps = 0, npanels = 0, def_from = -1, kdone = 0;
    int status = RCP_OK, num_kind = 0, num_step = 0;
    double dmax = 0.0;
    const double* Acur = A;
    int64_t ldA = lda;
    int nb = 0;  // next scratch buffer
    int k = 0;
    if (p.armed && beta == 0.0) {  // zero sketch: deficient from the start (factor.py:510-511)
      if (live) {
        dd[i] = 0.0;
        dof[i] = 0.0;
        pat[i] = 3;
      }
      def_from = 0;
      k = n;
    }

    while (k < n) {
      const int k0 = k;
      const int m = n - k0;
      const int width = min(b, m);
      ++npanels;
      if (live && i >= k0) S.pol[i] = i - k0;
      const bool act0 = live && i >= k0;
      __syncthreads();

      PF(3);
      // ---- guard + partial QRCP + replay (factor.py:570-600)
      if (p.q > 1 && m > 1) {
        if (tid == 0) {
          c_mul += (int)P * (m - 1);
          c_add += (int)P * (m - 1);
          c_cmp += m - 1;
        }
        double y[PM];
#pragma unroll
        for (int r = 0; r < PM; ++r) y[r] = (act0 && r < P) ? Bx[(size_t)r * n + i] : 0.0;
        double tsel = bmax(act0 ? sc_norm<PM>(y, 0, P) : 0.0, S, par);
        if (p.armed && tsel < p.thr[recomputes] * beta) {
          // fresh projection of the active block from the continuing stream (factor.py:392-404)
          if (zoff + (int64_t)P * m > p.z_len || recomputes + 1 >= kMaxThr) {
            status = RCP_ERR_NEED_NORMALS;
            break;
          }
          if (act0) {
#pragma unroll
            for (int r = 0; r < PM; ++r) y[r] = 0.0;
            const int ci = i - k0;
            for (int j = 0; j < m; ++j) {
              // T(ci, j) = T(j, ci); trailing blocks hold only their lower triangle
              const double a = ci >= j ? Acur[(size_t)j * ldA + ci] : Acur[(size_t)ci * ldA + j];
              const double* zz = p.z + zoff + j;
#pragma unroll
              for (int r = 0; r < PM; ++r)
                if (r < P) y[r] = __fma_rn(__ldg(zz + (size_t)r * m), a, y[r]);
            }
#pragma unroll
            for (int r = 0; r < PM; ++r)
              if (r < P) Bx[(size_t)r * n + i] = y[r];
          }
          zoff += (int64_t)P * m;
          ++recomputes;
          tsel = bmax(act0 ? sc_norm<PM>(y, 0, P) : 0.0, S, par);
          if (tsel < p.thr[recomputes] * beta) {  // "stop": deficient tail (factor.py:381-385)
            if (act0) {
              dd[i] = 0.0;
              dof[i] = 0.0;
              pat[i] = 3;
            }
            def_from = k0;
            kdone = k0;
            k = n;
            break;
          }
        }
        const int qn = min(min(p.q, width), min(m, P));
        int slot = act0 ? i - k0 : INT_MAX;
        // y rows >= P are zero (padding), so the loops below run over all PM rows unpredicated
        // on P; rows < s are predicated off (they are finished)
        for (int s = 0; s < qn; ++s) {
          // One barrier per QRCP step.  Each warp's best column publishes its Householder vector
          // (speculative: computed before the winner is known) next to its key; after the
          // barrier every thread reads the winner's vector and reflects its own column.
          const bool cand_ok = slot >= s && slot != INT_MAX;
          double key = -1.0;
          int idx = INT_MAX;
          if (__any_sync(0xffffffffu, cand_ok)) {
            // residual norm: 4 independent FMA chains over rows > s, then row s
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, x0 = 0.0;
#pragma unroll
            for (int r = 0; r < PM; ++r) {
              if (r == s) x0 = y[r];
              if (r > s) {
                if ((r & 3) == 0) a0 = __fma_rn(y[r], y[r], a0);
                else if ((r & 3) == 1) a1 = __fma_rn(y[r], y[r], a1);
                else if ((r & 3) == 2) a2 = __fma_rn(y[r], y[r], a2);
                else a3 = __fma_rn(y[r], y[r], a3);
              }
            }
            const double rest = (a0 + a1) + (a2 + a3);
            const double ss = __fma_rn(x0, x0, rest);
            if (cand_ok) {
              key = (ss == 0.0 || (ss >= 1e-280 && ss <= 1e280)) ? sqrt(ss) : sc_norm<PM>(y, s, PM);
              idx = slot;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const double k2 = __shfl_xor_sync(0xffffffffu, key, o);
              const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
              if (better(k2, i2, key, idx)) {
                key = k2;
                idx = i2;
              }
            }
            if (slot == idx) {  // reflector of this column (sketch.py:158-168)
              double* cw = S.cand + ((size_t)par * BW + warp) * (PM + 2);
              const double xn = key;  // = ||y[s:]||
              const double v0 = x0 + copysign(xn, x0 != 0.0 ? x0 : 1.0);
              const double vv = __fma_rn(v0, v0, rest);
#pragma unroll
              for (int r = 0; r < PM; ++r)
                if (r >= s) cw[r] = r == s ? v0 : y[r];
              cw[PM] = (xn == 0.0 || vv == 0.0) ? 0.0 : 2.0 / vv;  // 0: no reflection
            }
          }
          if (lane == 0) {
            S.redk[par * BW + warp] = key;
            S.redi[par * BW + warp] = idx;
          }
          __syncthreads();
          int ww = 0;
          key = S.redk[par * BW];
          idx = S.redi[par * BW];
#pragma unroll
          for (int w = 1; w < BW; ++w) {
            const double k2 = S.redk[par * BW + w];
            const int i2 = S.redi[par * BW + w];
            if (better(k2, i2, key, idx)) {
              key = k2;
              idx = i2;
              ww = w;
            }
          }
          const double* cv = S.cand + ((size_t)par * BW + ww) * (PM + 2);
          par ^= 1;
          const int sw = idx;
          const bool winner = (slot == sw);
          if (winner) slot = s;
          else if (slot == s) slot = sw;
          if (slot <= s || slot == INT_MAX) continue;
          const double coef = cv[PM];
          if (coef == 0.0) continue;
          double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
          for (int r = 0; r < PM; ++r)
            if (r >= s) {
              if ((r & 3) == 0) d0 = __fma_rn(cv[r], y[r], d0);
              else if ((r & 3) == 1) d1 = __fma_rn(cv[r], y[r], d1);
              else if ((r & 3) == 2) d2 = __fma_rn(cv[r], y[r], d2);
              else d3 = __fma_rn(cv[r], y[r], d3);
            }
          const double u = coef * ((d0 + d1) + (d2 + d3));
#pragma unroll
          for (int r = 0; r < PM; ++r)
            if (r >= s) y[r] = __dsub_rn(y[r], __dmul_rn(cv[r], u));
        }
        if (tid == 0)
          for (int s = 0; s < qn; ++s) {
            c_cmp += m - 1 - s;
            c_mul += 2LL * P * (m - s);
            c_add += 2LL * P * (m - s);
          }
        // replay: column at panel slot i-k0 moves to logical k0 + slot (same transpositions)
        int pvi = 0;
        if (act0) {
          pvi = S.permv[i];
#pragma unroll
          for (int r = 0; r < PM; ++r) y[r] = r < P ? Bx[(size_t)r * n + i] : 0.0;
        }
        __syncthreads();
        if (act0) {
          S.permv[k0 + slot] = pvi;
          S.pol[k0 + slot] = i - k0;
#pragma unroll
          for (int r = 0; r < PM; ++r)
            if (r < P) Bx[(size_t)r * n + k0 + slot] = y[r];
        }
        __syncthreads();
      }

      if (p.dbg == 3) {
        status = 99;
        break;
      }
      PF(0);
      // ---- SBKP steps (factor.py:602-634)
      // element (a, c) of the symmetric active block, read from its lower triangle (the only part
      // the trailing update stores; the input A is full, so the same rule holds for panel 0)
      auto T = [&](int a, int c) -> double {
        return a >= c ? Acur[(size_t)c * ldA + a] : Acur[(size_t)a * ldA + c];
      };
      double tk = act0 ? T(S.pol[i], S.pol[k0]) : 0.0;
      int t = 0;
      bool deferred = false;
      while (t < width && k0 + t < n) {
        const int kk = k0 + t;
        const int mm = n - kk;
        const bool act = live && i >= kk;
        double c = 0.0;
        if (act) {
          c = __dsub_rn(tk, panel_dot(S.Lp, S.Wp, i, kk, t));
          S.c0s[i] = c;
        }
        double lam = (act && i > kk) ? fabs(c) : -1.0;
        int r = (act && i > kk) ? i : INT_MAX;
        bargmax(lam, r, S, par);
        const double akk = S.c0s[kk];
        int kind, s;
        double dr = 0.0, tr = 0.0;
        if (mm == 1 || lam == 0.0) {
          kind = 0;
          s = 1;
        } else if (fabs(akk) >= alpha * lam) {
          kind = 1;
          s = 1;
        } else {
          const int pr = S.pol[r];
          if (act) tr = T(S.pol[i], pr);
          dr = __dsub_rn(T(pr, pr), panel_dot(S.Lp, S.Wp, r, r, t));
          if (fabs(dr) >= alpha * lam) {
            kind = 2;
            s = 1;
          } else {
            kind = 3;
            s = 2;
          }
        }
        deferred = s == 2 && t > 0 && t + 2 > width;
        if (p.dbg == 9) {  // debug: every thread must have taken the same decision
          __shared__ long long s_chk[4];
          __syncthreads();
          if (tid == 0) {
            s_chk[0] = kind;
            s_chk[1] = r;
            s_chk[2] = __double_as_longlong(dr);
            s_chk[3] = __double_as_longlong(lam);
          }
          __syncthreads();
          const int bad = (s_chk[0] != kind) | ((s_chk[1] != r) << 1) |
                          ((s_chk[2] != __double_as_longlong(dr)) << 2) | ((s_chk[3] != __double_as_longlong(lam)) << 3);
          if (__syncthreads_or(bad)) {
            if (bad) atomicOr(&s_skip, bad << 8);
            __syncthreads();
            status = 98;
            num_kind = s_skip >> 8;
            num_step = kk;
            break;
          }
        }
        if (tid == 0) {  // op counters of _decide / _eliminate (factor.py:350-367, 414-489)
          const long long colc = t > 0 ? (int)t * mm : 0;
          c_mul += colc;
          c_add += colc;
          c_cmp += mm >= 2 ? mm - 2 : 0;
          if (kind >= 2 && t > 0) {
            c_mul += t;
            c_add += t;
          }
          if (!deferred) {
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
          }
        }
        if (deferred) break;  // defer (factor.py:622-623)

        // symmetric swaps as bookkeeping + register/smem row exchanges (factor.py:624-630)
        int sa = -1, sb = -1;
        if (kind == 2) {
          sa = kk;
          sb = r;
        } else if (kind == 3 && r != kk + 1) {
          sa = kk + 1;
          sb = r;
        }
        if (sa >= 0) {
          __syncthreads();  // every thread has read pol / Lp / Wp rows for this decision
          if (tid == sa || tid == sb) s_tsw[tid == sa ? 0 : 1] = tr;
          if (tid >= 128 && tid < 128 + P) {  // sketch columns
            double* bc = Bx + (size_t)(tid - 128) * n;
            const double u = bc[sa];
            bc[sa] = bc[sb];
            bc[sb] = u;
          }
          if (tid < t) {
            double* Lc = S.Lp + (size_t)tid * BT;
            const double u = Lc[sa];
            Lc[sa] = Lc[sb];
            Lc[sb] = u;
          } else if (tid >= 32 && tid < 32 + t) {
            double* Wc = S.Wp + (size_t)(tid - 32) * BT;
            const double u = Wc[sa];
            Wc[sa] = Wc[sb];
            Wc[sb] = u;
          } else if (tid == 64) {
            int u = S.pol[sa];
            S.pol[sa] = S.pol[sb];
            S.pol[sb] = u;
            u = S.permv[sa];
            S.permv[sa] = S.permv[sb];
            S.permv[sb] = u;
          } else if (tid == 65 && kind == 3) {
            const double u = S.c0s[sa];
            S.c0s[sa] = S.c0s[sb];
            S.c0s[sb] = u;
          }
        }
        __syncthreads();
        if (sa >= 0 && (tid == sa || tid == sb)) tr = s_tsw[tid == sa ? 1 : 0];

        // D block and checks (factor.py:202-226, 455-466): identical in every thread
        double d11, d21 = 0.0, d22 = 0.0, det = 1.0;
        int nk = 0;
        if (kind <= 1) {
          d11 = akk;
          if (!isfinite(d11)) nk = 3;
        } else if (kind == 2) {
          d11 = dr;
          if (!isfinite(d11)) nk = 3;
        } else {
          d11 = akk;
          d21 = S.c0s[kk + 1];
          d22 = dr;
          det = __dsub_rn(__dmul_rn(d11, d22), __dmul_rn(d21, d21));
          if (det == 0.0) {
            nk = 2;
          } else if (!isfinite(d11) || !isfinite(d21) || !isfinite(d22)) {
            nk = 3;
          } else {
            const double a21 = fabs(d21);
            const double dt = __dsub_rn(__dmul_rn(d11, d22), __dmul_rn(a21, a21));
            const double bound =
                __dmul_rn(__dmul_rn(__dmul_rn(__dsub_rn(1.0, __dmul_rn(alpha, alpha)), a21), a21), __dsub_rn(1.0, 1e-12));
            if (fabs(dt) < bound) nk = 4;
          }
        }
        if (nk) {
          status = RCP_ERR_NUMERICAL;
          num_kind = nk;
          num_step = kk;
          break;
        }
        // multipliers and writes (factor.py:467-480): W keeps the unscaled columns
        int lerr = 0;
        if (act) {
          if (kind <= 1) {
            S.Wp[(size_t)t * BT + i] = c;
            if (i > kk) {
              const double l = kind == 0 ? 0.0 : __ddiv_rn(c, d11);
              if (!isfinite(l)) lerr = 1;
              S.Lp[(size_t)t * BT + i] = l;
            }
          } else if (kind == 2) {
            const double c0 = __dsub_rn(tr, panel_dot(S.Lp, S.Wp, i, kk, t));
            S.Wp[(size_t)t * BT + i] = c0;
            if (i > kk) {
              const double l = __ddiv_rn(c0, d11);
              if (!isfinite(l)) lerr = 1;
              S.Lp[(size_t)t * BT + i] = l;
            }
          } else {
            const double c0 = S.c0s[i];
            const double c1 = __dsub_rn(tr, panel_dot(S.Lp, S.Wp, i, kk + 1, t));
            S.Wp[(size_t)t * BT + i] = c0;
            S.Wp[(size_t)(t + 1) * BT + i] = c1;
            if (i > kk + 1) {
              const double l1 = __ddiv_rn(__dsub_rn(__dmul_rn(c0, d22), __dmul_rn(d21, c1)), det);
              const double l2 = __ddiv_rn(__dsub_rn(__dmul_rn(d11, c1), __dmul_rn(d21, c0)), det);
              if (!isfinite(l1) || !isfinite(l2)) lerr = 1;
              S.Lp[(size_t)t * BT + i] = l1;
              S.Lp[(size_t)(t + 1) * BT + i] = l2;
            } else if (i == kk + 1) {
              S.Lp[(size_t)t * BT + i] = 0.0;  // L[k+1, k] of a 2x2 block is exactly zero
            }
          }
        }
        if (tid == 0) {
          dd[kk] = d11;
          dof[kk] = kind == 3 ? d21 : 0.0;
          pat[kk] = kind == 3 ? 1 : 0;
          dmax = fmax(dmax, fabs(d11));
          if (kind == 3) {
            dd[kk + 1] = d22;
            dof[kk + 1] = 0.0;
            pat[kk + 1] = 2;
            dmax = fmax(dmax, fmax(fabs(d21), fabs(d22)));
            ++n2x2;
          }
          ++nsteps;
        }
        // prefetch the next pivot column (pol is final for this step)
        const int kn = kk + s;
        if (t + s < width && kn < n && live && i >= kn) tk = T(S.pol[i], S.pol[kn]);
        lerr = __syncthreads_or(lerr);
        if (lerr) {
          status = RCP_ERR_NUMERICAL;
          num_kind = 3;
          num_step = kk;
          break;
        }
        t += s;
        if (p.dbg == 4) {
          status = 99;
          break;
        }
      }
      if (p.dbg == 5) status = 99;
      if (status != RCP_OK) break;
      (void)deferred;
      const int k_end = k0 + t;
      const int mp = n - k_end;

      PF(1);
      // L columns of this panel, keyed by original row index (rows never move afterwards)
      if (act0) {
        double* dst = Lst + (size_t)S.permv[i] * n + k0;
        for (int s = 0; s < t; ++s)
          if (i > k0 + s) __stcs(dst + s, S.Lp[(size_t)s * BT + i]);  // read once at the end: evict-first
      }

      if (mp > 0 && t > 0) {
        // ---- trailing update A22 -= L21 W21^T (factor.py:369-379). The reference mirrors the
        // lower result into the upper part (mirror_lower); here only the lower triangle is
        // stored and every reader takes (a, c) with a < c from (c, a) -- the same values.
        // Warp work unit: a 32-row strip I x an 8-column group g of the lower triangle; lane =
        // row.  Stores are coalesced across lanes; the C-in gather (through pol) of the next
        // unit is issued before this unit's FMAs.
        double* An = Abuf[nb];
        const int ng = (mp + 7) >> 3;
        int uI = 0, ug = warp;
        while (uI * 32 < mp && ug >= min(4 * uI + 4, ng)) {
          ug -= min(4 * uI + 4, ng);
          ++uI;
        }
#define RCP_LOAD_CIN(I_, g_, cin_)                                                   \
  {                                                                                  \
    const int ii_ = k_end + 32 * (I_) + lane;                                        \
    const int j0_ = k_end + 8 * (g_);                                                \
    const int pi_ = ii_ < n ? S.pol[ii_] : 0;                                        \
    _Pragma("unroll") for (int c2 = 0; c2 < 8; ++c2) {                               \
      const int j_ = j0_ + c2;                                                       \
      const int pj_ = (ii_ < n && j_ < n && ii_ >= j_) ? S.pol[j_] : -1;                      \
      cin_[c2] = pj_ < 0 ? 0.0 : (pi_ >= pj_ ? Acur[(size_t)pj_ * ldA + pi_] : Acur[(size_t)pi_ * ldA + pj_]); \
    }                                                                                \
  }
        double cin[8];
        if (uI * 32 < mp) RCP_LOAD_CIN(uI, ug, cin);
        while (uI * 32 < mp) {
          // next unit of this warp
          int nI = uI, ngp = ug + BW;
          while (nI * 32 < mp && ngp >= min(4 * nI + 4, ng)) {
            ngp -= min(4 * nI + 4, ng);
            ++nI;
          }
          double cnx[8];
          if (nI * 32 < mp) RCP_LOAD_CIN(nI, ngp, cnx);
          const int ii = k_end + 32 * uI + lane;
          const int j0 = k_end + 8 * ug;
          double acc[8];
#pragma unroll
          for (int c2 = 0; c2 < 8; ++c2) acc[c2] = 0.0;
          const int ir = min(ii, BT - 1);
          for (int s2 = 0; s2 < t; ++s2) {
            const double lv = S.Lp[(size_t)s2 * BT + ir];
            const double* Wc = S.Wp + (size_t)s2 * BT;
#pragma unroll
            for (int c2 = 0; c2 < 8; ++c2) acc[c2] = __fma_rn(lv, Wc[j0 + c2], acc[c2]);  // j0 + c2 <= n + 7 stays inside smem
          }
          if (ii < n) {
#pragma unroll
            for (int c2 = 0; c2 < 8; ++c2) {
              const int j = j0 + c2;
              if (j < n && ii >= j) {
                const double v = __dsub_rn(cin[c2], acc[c2]);
                An[(size_t)(j - k_end) * mp + (ii - k_end)] = v;  // lower triangle only
              }
            }
          }
#pragma unroll
          for (int c2 = 0; c2 < 8; ++c2) cin[c2] = cnx[c2];
          uI = nI;
          ug = ngp;
        }
#undef RCP_LOAD_CIN
        if (tid == 0) {
          c_mul += (int)t * ((int)mp * (mp + 1) / 2);
          c_add += (int)t * ((int)mp * (mp + 1) / 2);
        }
        // ---- sketch correction B2 -= (B1 L11^-T) L21^T (factor.py:554-565)
        if (p.q > 1) {
          if (tid < P) {
            for (int s = 0; s < t; ++s) {
              double yv = Bx[(size_t)tid * n + k0 + s];
              for (int u = 0; u < s; ++u) yv = __fma_rn(-S.Ys[tid * b + u], S.Lp[(size_t)u * BT + k0 + s], yv);
              S.Ys[tid * b + s] = yv;
            }
          }
          __syncthreads();
          if (live && i >= k_end) {
            for (int q = 0; q < P; ++q) {
              double acc = 0.0;
              for (int s = 0; s < t; ++s) acc = __fma_rn(S.Ys[q * b + s], S.Lp[(size_t)s * BT + i], acc);
              double* bq = Bx + (size_t)q * n + i;
              *bq = __dsub_rn(*bq, acc);
            }
          }
          if (tid == 0) {
            c_mul += (int)t * P * mp + (int)(t * (t - 1) / 2) * mp;
            c_add += (int)t * P * mp + (int)(t * (t - 1) / 2) * mp;
          }
        }
        Acur = An;
        ldA = mp;
        nb ^= 1;
      }
      if (p.dbg == 6 || (p.dbg > 100 && npanels >= p.dbg - 100)) {
        status = 99;
        break;
      }
      __syncthreads();  // trailing block + Lst visible; Lp/Wp free for the next panel
      PF(2);
      k = k_end;
      kdone = k_end;
    }

    if (status != RCP_OK) {
      if (tid == 0) {
        rcp_batch_stats z{};
        z.status = status;
        z.num_kind = num_kind;
        z.num_step = num_step;
        z.recompute_count = recomputes;
        z.deficient_from = -1;
        z.amax = amax;
        *ms = z;
      }
      continue;
    }
    __syncthreads();
    if (p.dbg == 7) continue;
    // ---- outputs: perm, L in final order (one coalesced row gather), statistics
    if (live) perm_o[i] = S.permv[i];
    double mm = 0.0;
    for (int row = warp; row < n; row += BW) {
      const double* src = Lst + (size_t)S.permv[row] * n;
      double* dst = Lo + (size_t)row * n;
      for (int c = lane; c < n; c += 32) {
        double v;
        if (c < row) {
          v = c < kdone ? __ldcs(src + c) : 0.0;
          mm = fmax(mm, fabs(v));
        } else {
          v = c == row ? 1.0 : 0.0;
        }
        __stcs(dst + c, v);  // output: streaming store, keeps the other CTAs' trailing blocks in L2
      }
    }
    mm = bmax(mm, S, par);
    if (tid == 0) {
      rcp_batch_stats z{};
      z.status = RCP_OK;
      z.recompute_count = recomputes;
      z.deficient_from = def_from;
      z.n_2x2 = n2x2;
      z.n_steps = nsteps;
      z.n_panels = npanels;
      z.amax = amax;
      z.dmax = dmax;
      z.max_multiplier = n > 1 ? mm : 0.0;
      z.rho_cheap = amax == 0.0 ? (dmax == 0.0 ? 1.0 : INFINITY) : dmax / amax;
      z.mults = c_mul;
      z.adds = c_add;
      z.divs = c_div;
      z.comps = c_cmp;
#if RCP_BATCH_PROF
      PF(3);
      z.mults = pf[0];  // QRCP (guard + QRCP + replay)
      z.adds = pf[1];   // SBKP steps
      z.divs = pf[2];   // L store + trailing update + sketch correction
      z.comps = pf[3];  // validation + sketch + outputs
#endif
      *ms = z;
    }
  }
}

// ---------------------------------------------------------------- batched solve
// x = P^T L^-T D^-1 L^-1 P b per matrix (solve.py:34-76); one CTA per matrix, L rows read
// coalesced (row-major), 16-row blocks.
constexpr int SB = 16;

__global__ void __launch_bounds__(BT) batched_solve_kernel(int count, int n, const int64_t* __restrict__ perm,
                                                           const double* __restrict__ L,
                                                           const double* __restrict__ d_diag,
                                                           const double* __restrict__ d_off,
                                                           const int8_t* __restrict__ pattern,
                                                           const double* b, double* x, int32_t* singular) {
  __shared__ double y[BT];
  __shared__ double part[BW][SB];
  __shared__ int s_sing;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int mat = blockIdx.x; mat < count; mat += gridDim.x) {
    const int64_t* pm = perm + (size_t)mat * n;
    const double* Lm = L + (size_t)mat * n * n;
    const double* dg = d_diag + (size_t)mat * n;
    const double* df = d_off + (size_t)mat * n;
    const int8_t* pt = pattern + (size_t)mat * n;
    __syncthreads();
    if (tid < n) y[tid] = b[(size_t)mat * n + pm[tid]];  // y = b[perm]
    if (tid == 0) s_sing = 0;
    __syncthreads();
    // forward: unit lower L (solve.py:69-71)
    for (int r0 = 0; r0 < n; r0 += SB) {
      const int rb = min(SB, n - r0);
      // y[r0 + a] -= L[r0 + a, :r0] . y[:r0]; warp w handles rows a = w, w + BW
      for (int a = warp; a < rb; a += BW) {
        const double* Lr = Lm + (size_t)(r0 + a) * n;
        double acc = 0.0;
        for (int j = lane; j < r0; j += 32) acc = __fma_rn(Lr[j], y[j], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) part[0][a] = acc;
      }
      __syncthreads();
      if (warp == 0) {
        double v = lane < rb ? __dsub_rn(y[r0 + lane], part[0][lane]) : 0.0;
        const double* Lb = Lm + (size_t)(r0 + (lane < rb ? lane : 0)) * n + r0;
        for (int j = 0; j < rb; ++j) {
          const double yj = __shfl_sync(0xffffffffu, v, j);
          if (lane > j && lane < rb) v = __fma_rn(-Lb[j], yj, v);
        }
        if (lane < rb) y[r0 + lane] = v;
      }
      __syncthreads();
    }
    // block diagonal (solve.py:47-62): exact-zero blocks give zeros and the singular flag
    double out = 0.0;
    if (tid < n) {
      const int8_t pk = pt[tid];
      const double v = y[tid];
      int sg = 0;
      if (pk == 1) {
        const double d11 = dg[tid], d21 = df[tid], d22 = dg[tid + 1];
        const double det = __dsub_rn(__dmul_rn(d11, d22), __dmul_rn(d21, d21));
        if (det == 0.0) sg = 1;
        else out = __ddiv_rn(__dsub_rn(__dmul_rn(d22, v), __dmul_rn(d21, y[tid + 1])), det);
      } else if (pk == 2) {
        const double d11 = dg[tid - 1], d21 = df[tid - 1], d22 = dg[tid];
        const double det = __dsub_rn(__dmul_rn(d11, d22), __dmul_rn(d21, d21));
        if (det == 0.0) sg = 1;
        else out = __ddiv_rn(__dsub_rn(__dmul_rn(d11, v), __dmul_rn(d21, y[tid - 1])), det);
      } else {
        const double d = dg[tid];
        if (d == 0.0) sg = 1;
        else out = __ddiv_rn(v, d);
      }
      if (sg) atomicOr(&s_sing, 1);
    }
    __syncthreads();
    if (tid < n) y[tid] = out;
    __syncthreads();
    // backward with L^T (solve.py:72-73): blocks from the bottom; after a block is solved,
    // y[:r0] -= L[r0:r0+rb, :r0]^T x[r0:r0+rb] (rows of L read coalesced)
    for (int r1 = n; r1 > 0; r1 -= SB) {
      const int r0 = max(0, r1 - SB);
      const int rb = r1 - r0;
      if (warp == 0) {
        double v = lane < rb ? y[r0 + lane] : 0.0;
        for (int j = rb - 1; j >= 0; --j) {
          const double xj = __shfl_sync(0xffffffffu, v, j);
          if (lane < j) v = __fma_rn(-Lm[(size_t)(r0 + j) * n + r0 + lane], xj, v);
        }
        if (lane < rb) y[r0 + lane] = v;
      }
      __syncthreads();
      if (tid < r0) {
        double acc = 0.0;
        for (int a = 0; a < rb; ++a) acc = __fma_rn(Lm[(size_t)(r0 + a) * n + tid], y[r0 + a], acc);
        y[tid] = __dsub_rn(y[tid], acc);
      }
      __syncthreads();
    }
    if (tid < n) x[(size_t)mat * n + pm[tid]] = y[tid];  // x[perm] = v
    if (tid == 0 && singular) singular[mat] = s_sing;
  }
}

__global__ void transpose_omega_kernel(const double* __restrict__ om, int P, int PM, int n, double* __restrict__ omT) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n)
    for (int r = 0; r < PM; ++r) omT[(size_t)j * PM + r] = r < P ? om[(size_t)r * n + j] : 0.0;
}

int pick_pm(int P) {
  if (P <= 8) return 8;
  if (P <= 16) return 16;
  if (P <= 24) return 24;
  if (P <= 32) return 32;
  if (P <= 48) return 48;
  return 64;
}

size_t factor_smem(int PM, int b) {
  const int SC = std::max(2 * b + 1, PM);
  size_t d = (size_t)SC * BT + BT + 2 * PM + PM + 2 + 2 * (size_t)PM * b + 2 * BW + 2 * BW * (size_t)(PM + 2);
  return d * 8 + (2 * BW + 2 * BT) * 4;
}

template <int PM, int MINB>
cudaError_t launch_pm(const BatchParams& prm, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(batched_factor_kernel<PM, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  batched_factor_kernel<PM, MINB><<<grid, BT, smem, st>>>(prm);
  return cudaGetLastError();
}

int resident_ctas(int PM) {
  if (const char* e = std::getenv("RCP_BATCH_MINB")) return std::atoi(e) == 1 ? 1 : 2;
  return PM <= 32 ? 2 : 1;
}

int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

int64_t ws_stride_doubles(int64_t n, int PM) { return ((3 * n * n + (int64_t)PM * n + 31) / 32) * 32; }

}  // namespace

extern "C" {

size_t rcp_batched_workspace_bytes(int64_t n, const rcp_config* cfg) {
  if (!cfg || n < 1 || n > BT || cfg->p < 1 || cfg->p > 64 || cfg->b < 1 || cfg->b > kMaxB) return 0;
  const int grid = sm_count() * resident_ctas(pick_pm(cfg->p));
  const size_t om_bytes = ((size_t)n * pick_pm(cfg->p) * 8 + 255) & ~size_t(255);
  return (size_t)grid * (size_t)ws_stride_doubles(n, pick_pm(cfg->p)) * 8 + 256 + om_bytes;
}

int rcp_factor_batched(const rcp_config* cfg, int64_t count, int64_t n, const double* a, int64_t lda,
                       int64_t a_stride, const double* normals, int64_t normals_len, void* workspace,
                       size_t workspace_bytes, int64_t* perm, double* L, double* d_diag, double* d_off,
                       int8_t* pattern, rcp_batch_stats* mstats, void* cuda_stream) {
  if (!cfg || count < 0 || n < 1 || lda < n || a_stride < n * lda - (lda - n)) return RCP_ERR_INVALID_ARG;
  if (cfg->p < 1 || cfg->b < 1 || cfg->robust_r < 0 || cfg->p < cfg->q) return RCP_ERR_INVALID_ARG;
  if (!(cfg->q == 1 || cfg->q == cfg->b)) return RCP_ERR_INVALID_ARG;
  if (n > BT || cfg->b > kMaxB || cfg->p > 64 || cfg->q == 1) return RCP_ERR_UNSUPPORTED;
  if (cfg->strategy != RCP_STRATEGY_RCP) return RCP_ERR_UNSUPPORTED;  // batched kernel: rcp only
  if (count > INT_MAX || normals_len < (int64_t)cfg->p * n) return RCP_ERR_INVALID_ARG;
  if (count == 0) return RCP_OK;
  const size_t need = rcp_batched_workspace_bytes(n, cfg);
  if (!workspace || workspace_bytes < need) return RCP_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  const int P = cfg->p;
  const int PM = pick_pm(P);
  int grid = sm_count() * resident_ctas(PM);
  if (const char* g = std::getenv("RCP_BATCH_GRID")) grid = std::max(1, std::min(grid, std::atoi(g)));

  // workspace: [counter | omegaT (n x P) | per-CTA scratch]
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  int* counter = reinterpret_cast<int*>(ws);
  double* omegaT = reinterpret_cast<double*>(ws + 256);
  const size_t om_bytes = ((size_t)n * PM * 8 + 255) & ~size_t(255);
  double* scratch = reinterpret_cast<double*>(ws + 256 + om_bytes);
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return RCP_ERR_CUDA;
  // Omega^T (n x P) from the row-major Omega at the head of the normal stream
  transpose_omega_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(normals, P, PM, (int)n, omegaT);
  if (cudaGetLastError() != cudaSuccess) return RCP_ERR_CUDA;
  BatchParams prm{};
  prm.count = (int)count;
  prm.n = (int)n;
  prm.P = P;
  prm.b = cfg->b;
  prm.q = cfg->q;
  prm.armed = cfg->robust_r >= 1;
  prm.alpha = std::sqrt(2.0) / 2.0;
  {  // thresholds exactly as the reference accumulates them: delta = 1/r, then delta += 1/r per
     // recompute, threshold = eps**delta (factor.py:316, 400-401)
    double delta = prm.armed ? 1.0 / cfg->robust_r : 0.0;
    for (int j = 0; j < kMaxThr; ++j) {
      prm.thr[j] = prm.armed ? std::pow(DBL_EPSILON, delta) : 0.0;
      if (prm.armed) delta += 1.0 / cfg->robust_r;
    }
  }
  prm.A = a;
  prm.lda = lda;
  prm.a_stride = a_stride;
  prm.omegaT = omegaT;
  prm.z = normals;
  prm.z_len = normals_len;
  prm.ws = scratch;
  prm.ws_stride = ws_stride_doubles(n, pick_pm(cfg->p));
  prm.perm = perm;
  prm.L = L;
  prm.d_diag = d_diag;
  prm.d_off = d_off;
  prm.pattern = pattern;
  prm.mstats = mstats;
  prm.next = counter;
  if (const char* dbg = std::getenv("RCP_BATCH_DBG")) prm.dbg = std::atoi(dbg);
  const size_t smem = factor_smem(PM, cfg->b);
  switch (PM) {
    case 8: e = launch_pm<8, 2>(prm, grid, smem, st); break;
    case 16: e = launch_pm<16, 2>(prm, grid, smem, st); break;
    case 24:
      e = resident_ctas(24) == 1 ? launch_pm<24, 1>(prm, grid, smem, st) : launch_pm<24, 2>(prm, grid, smem, st);
      break;
    case 32: e = launch_pm<32, 2>(prm, grid, smem, st); break;
    case 48: e = launch_pm<48, 1>(prm, grid, smem, st); break;
    default: e = launch_pm<64, 1>(prm, grid, smem, st); break;
  }
  return e == cudaSuccess ? RCP_OK : RCP_ERR_CUDA;
}

int rcp_solve_batched(int64_t count, int64_t n, const int64_t* perm, const double* L, const double* d_diag,
                      const double* d_off, const int8_t* pattern, const double* b, double* x, int32_t* singular,
                      void* cuda_stream) {
  if (count < 0 || n < 1 || n > BT || count > INT_MAX) return RCP_ERR_INVALID_ARG;
  if (count == 0) return RCP_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  const int grid = (int)std::min<int64_t>(count, (int64_t)sm_count() * 8);
  batched_solve_kernel<<<grid, BT, 0, st>>>((int)count, (int)n, perm, L, d_diag, d_off, pattern, b, x, singular);
  return cudaGetLastError() == cudaSuccess ? RCP_OK : RCP_ERR_CUDA;
}

}  // extern "C"
