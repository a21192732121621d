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
// local best candidate (plus the data the decision needs) and a release flag; every
// CTA then reads all G records and reduces them identically, so all CTAs take the
// same decision without a second barrier.  Values a CTA needs from rows it does not
// own (the next pivot's W row entries of the columns produced in this step) are
// recomputed redundantly with the same bitwise-deterministic dot routine.
#include <cfloat>
#include <climits>
#include "panel.cuh"
#include "rcp_common.cuh"

namespace rcp {

namespace {

constexpr int kPanelThreads = 256;
constexpr int kWarps = kPanelThreads / 32;

struct BlockBest {
  double key;
  long long idx;
  int slot;
};

// Block-wide argmax with numpy first-index semantics; result broadcast to all threads.
__device__ BlockBest block_argmax(double key, long long idx, int slot) {
  __shared__ double sk[kWarps];
  __shared__ long long si[kWarps];
  __shared__ int ss[kWarps];
  __shared__ BlockBest res;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double k2 = __shfl_down_sync(0xffffffffu, key, off);
    long long i2 = __shfl_down_sync(0xffffffffu, idx, off);
    int s2 = __shfl_down_sync(0xffffffffu, slot, off);
    if (better(k2, i2, key, idx)) {
      key = k2;
      idx = i2;
      slot = s2;
    }
  }
  if (lane == 0) {
    sk[warp] = key;
    si[warp] = idx;
    ss[warp] = slot;
  }
  __syncthreads();
  if (warp == 0) {
    key = lane < kWarps ? sk[lane] : -1.0;
    idx = lane < kWarps ? si[lane] : LLONG_MAX;
    slot = lane < kWarps ? ss[lane] : -1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      double k2 = __shfl_down_sync(0xffffffffu, key, off);
      long long i2 = __shfl_down_sync(0xffffffffu, idx, off);
      int s2 = __shfl_down_sync(0xffffffffu, slot, off);
      if (better(k2, i2, key, idx)) {
        key = k2;
        idx = i2;
        slot = s2;
      }
    }
    if (lane == 0) res = BlockBest{key, idx, slot};
  }
  __syncthreads();
  BlockBest out = res;
  __syncthreads();
  return out;
}

// Deterministic sum over vals[lo, hi) by warp 0 (lane-strided partials + fixed tree);
// every CTA obtains the same bits for the same input.  Returns the value in lane 0.
__device__ double warp0_sum_sq(const double* vals, int lo, int hi) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int r = lo + lane; r < hi; r += 32) acc = __fma_rn(vals[r], vals[r], acc);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, off));
  return acc;
}

RCP_D void xpublish(long long* flags, int cta, long long seq) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(flags + cta, seq);
  }
}

// Waits for all G flags to reach seq.  A watchdog (~4 s of SM clock) turns a lost
// peer into an error instead of a hung GPU; returns false on timeout.
__device__ bool xwait(const long long* flags, int G, long long seq, PanelState* st) {
  __shared__ int s_timeout;
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < G; c += blockDim.x) {
    long long t0 = clock64();
    while (ld_acquire(flags + c) < seq) {
      if (clock64() - t0 > 8000000000LL) {
        s_timeout = 1;
        atomicExch(&st->status, 99);
        break;
      }
    }
  }
  __syncthreads();
  return s_timeout == 0;
}

// Euclidean norm from a fused (sum of squares, max |x|) pass.  Falls back to the
// reference's scaled formulation (core.py:122-142) when the plain sum could have
// overflowed or underflowed.
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

}  // namespace

__global__ void __launch_bounds__(kPanelThreads, 1) panel_kernel(PanelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int cta = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const int64_t n = p.n;
  const int k0 = p.k0, P = p.P, R = p.R, G = p.G, Wn = p.Wn;
  const int m0 = static_cast<int>(n - k0);
  const int r0 = cta * R;
  const int rcnt = max(0, min(R, m0 - r0));

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
  double* wrow = reinterpret_cast<double*>(carve(sizeof(double) * Wn));
  double* wrrow = reinterpret_cast<double*>(carve(sizeof(double) * Wn));
  unsigned char* region = sp;  // QRCP and SBKP phases reuse the rest

  __shared__ long long s_seq;
  __shared__ int s_stop;
  __shared__ double s_coef;
  __shared__ int s_skip;
  __shared__ double s_gakk;
  __shared__ int s_gerr, s_lerr, s_wcta;
  __shared__ double s_akk;

  for (int x = tid; x < Wn; x += nthr) win[x] = x;
  for (int i = tid; i < rcnt; i += nthr) lpos[i] = r0 + i;
  if (tid == 0) {
    s_seq = p.st->seq;
    s_stop = 0;
    s_lerr = 0;
  }
  __syncthreads();
  long long seq = s_seq;

  // =====================================================================
  // Phase 1: guard + partial QRCP on the sketch (q = b mode).
  // =====================================================================
  if (p.qn > 0) {
    const int Rs = p.Rs, Rg = R - Rs;
    double* Bs = reinterpret_cast<double*>(region);
    double* qnorm = Bs + (size_t)P * Rs;
    int* qsel = reinterpret_cast<int*>(qnorm + R);
    double* qg = p.qscr + (size_t)cta * P * (Rg > 0 ? Rg : 0);
    auto bel = [&](int r, int c) -> double& {
      return c < Rs ? Bs[r * Rs + c] : qg[(size_t)r * Rg + (c - Rs)];
    };
    for (int f = tid; f < P * rcnt; f += nthr) {
      int c = f / P, r = f - c * P;
      bel(r, c) = p.B[(size_t)(k0 + r0 + c) * P + r];
    }
    for (int c = tid; c < rcnt; c += nthr) qsel[c] = 0;
    __syncthreads();
    for (int c = tid; c < rcnt; c += nthr) {
      double ss = 0.0, am = 0.0;
      for (int r = 0; r < P; ++r) {
        double x = bel(r, c);
        am = fmax(am, fabs(x));
        ss = __fma_rn(x, x, ss);
      }
      qnorm[c] = safe_norm(ss, am, [&](int r) { return bel(r, c); }, 0, P);
    }
    __syncthreads();

    for (int j = 0; j < p.qn; ++j) {
      // ---- local candidate: largest residual norm, ties to the lowest position
      double bk = -1.0;
      long long bi = LLONG_MAX;
      int bs = -1;
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
      BlockBest lb = block_argmax(bk, bi, bs);
      const long long nseq = seq + 1;
      const int par = static_cast<int>(nseq & 1);
      if (lb.slot >= 0) {
        double* dst = p.qcol + ((size_t)par * G + cta) * P;
        for (int r = j + tid; r < P; r += nthr) dst[r] = bel(r, lb.slot);
      }
      if (tid == 0) {
        QRec rec;
        rec.norm = lb.slot >= 0 ? lb.key : -1.0;
        rec.pos = lb.slot >= 0 ? static_cast<int>(lb.idx) : INT_MAX;
        rec.col = lb.slot >= 0 ? r0 + lb.slot : -1;
        p.qrec[(size_t)par * G + cta] = rec;
      }
      seq = nseq;
      xpublish(p.flags, cta, seq);
      if (!xwait(p.flags, G, seq, p.st)) {
        s_stop = 1;
        break;
      }

      // ---- global winner (every CTA reduces the same records identically)
      double gk = -1.0;
      long long gi = LLONG_MAX;
      int gs = -1;
      for (int c = tid; c < G; c += nthr) {
        const QRec* rc = p.qrec + (size_t)par * G + c;
        double v = __ldcg(&rc->norm);
        int ps = __ldcg(&rc->pos);
        if (v >= 0.0 || v != v) {
          if (better(v, ps, gk, gi)) {
            gk = v;
            gi = ps;
            gs = c;
          }
        }
      }
      BlockBest gb = block_argmax(gk, gi, gs);
      const int wcta = gb.slot;
      const int wpos = static_cast<int>(gb.idx);
      const int wcol = __ldcg(&p.qrec[(size_t)par * G + wcta].col);

      if (j == 0 && p.guard_mode != 0) {
        // tsel = max column norm of B[:, k:] (factor.py:576-583 / 405-408)
        bool below = gb.key < p.guard_limit;
        if (below) {
          if (cta == 0 && tid == 0) p.st->status = p.guard_mode == 1 ? 1 : 2;
          s_stop = 1;
          break;
        }
      }

      // ---- Householder vector from the winner column (sketch.py:159-168)
      const double* src = p.qcol + ((size_t)par * G + wcta) * P;
      for (int r = j + tid; r < P; r += nthr) vvec[r] = __ldcg(src + r);
      __syncthreads();
      if (tid < 32) {
        double xn2 = warp0_sum_sq(vvec, j, P);
        double xn = sqrt(xn2);
        double x0 = vvec[j];
        double v0 = x0;
        int skip = 0;
        if (tid == 0) {
          if (xn == 0.0) {
            skip = 1;
          } else {
            v0 = __dadd_rn(x0, copysign(xn, x0 != 0.0 ? x0 : 1.0));
          }
        }
        skip = __shfl_sync(0xffffffffu, skip, 0);
        v0 = __shfl_sync(0xffffffffu, v0, 0);
        if (!skip) {
          if (tid == 0) vvec[j] = v0;
          __syncwarp();
          double vn2 = warp0_sum_sq(vvec, j, P);
          if (tid == 0) {
            if (vn2 == 0.0) {
              s_skip = 1;
            } else {
              s_skip = 0;
              s_coef = 2.0 / vn2;
            }
          }
        } else if (tid == 0) {
          s_skip = 1;
        }
        // ---- replay bookkeeping (factor.py:586-599): position j <-> wpos
        if (tid == 0 && wpos != j) {
          int cj = win[j];
          win[j] = wcol;
          if (wpos < Wn) win[wpos] = cj;
          // owner updates of lpos are done below by all CTAs (cj owner)
          s_wcta = cj;  // reuse as scratch: column that moves to wpos
        } else if (tid == 0) {
          s_wcta = -1;
        }
      }
      __syncthreads();
      {
        const int moved = s_wcta;
        if (tid == 0) {
          if (wcol >= r0 && wcol < r0 + rcnt) {
            lpos[wcol - r0] = j;
            qsel[wcol - r0] = 1;
          }
          if (moved >= 0 && moved >= r0 && moved < r0 + rcnt) lpos[moved - r0] = wpos;
        }
      }
      __syncthreads();

      // ---- reflect the remaining columns and refresh their residual norms
      if (j + 1 < p.qn) {
        const int skip = s_skip;
        const double coef = s_coef;
        for (int c = tid; c < rcnt; c += nthr) {
          if (qsel[c]) continue;
          double ss = 0.0, am = 0.0;
          if (!skip) {
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
            int r = j;
            for (; r + 4 <= P; r += 4) {
              d0 = __fma_rn(vvec[r], bel(r, c), d0);
              d1 = __fma_rn(vvec[r + 1], bel(r + 1, c), d1);
              d2 = __fma_rn(vvec[r + 2], bel(r + 2, c), d2);
              d3 = __fma_rn(vvec[r + 3], bel(r + 3, c), d3);
            }
            for (; r < P; ++r) d0 = __fma_rn(vvec[r], bel(r, c), d0);
            const double wv = __dmul_rn(coef, __dadd_rn(__dadd_rn(d0, d1), __dadd_rn(d2, d3)));
            {
              double& x = bel(j, c);
              x = __dsub_rn(x, __dmul_rn(vvec[j], wv));
            }
            for (r = j + 1; r < P; ++r) {
              double& x = bel(r, c);
              double y = __dsub_rn(x, __dmul_rn(vvec[r], wv));
              x = y;
              am = fmax(am, fabs(y));
              ss = __fma_rn(y, y, ss);
            }
          } else {
            for (int r = j + 1; r < P; ++r) {
              double y = bel(r, c);
              am = fmax(am, fabs(y));
              ss = __fma_rn(y, y, ss);
            }
          }
          qnorm[c] = safe_norm(ss, am, [&](int r) { return bel(r, c); }, j + 1, P);
        }
        __syncthreads();
      }
    }
  }

  if (s_stop) {
    if (cta == 0 && tid == 0) p.st->seq = seq;
    return;
  }

  // =====================================================================
  // Phase 2: SBKP pivot steps (factor.py:602-634) with left-looking columns.
  // =====================================================================
  const int Ls = p.Ls;
  double* Lsm = reinterpret_cast<double*>(region);  // [Ls][R]
  double* ck = Lsm + (size_t)Ls * R;
  double* cr = ck + R;
  double* dg = cr + R;
  double* acol = dg + R;
  const double* A = p.A;
  const double alpha = p.alpha;
  const int width = p.width;

  for (int i = tid; i < rcnt; i += nthr) {
    int64_t x = k0 + r0 + i;
    dg[i] = A[x * (n + 1)];
  }
  __syncthreads();
  int pk = win[0];
  for (int i = tid; i < rcnt; i += nthr) acol[i] = sym_lower(A, n, k0 + r0 + i, k0 + pk);
  __syncthreads();

  int t = 0;
  while (t < width && k0 + t < n) {
    // ---- phase A: pivot column (rows of the active block owned here)
    if (tid == 0) s_akk = 0.0;
    __syncthreads();
    double bk = -1.0;
    long long bi = LLONG_MAX;
    int bs = -1;
    for (int i = tid; i < rcnt; i += nthr) {
      const int lp = lpos[i];
      if (lp < t) continue;
      const int64_t row = k0 + r0 + i;
      double dot = chain_dot4(
          [&](int s) { return s < Ls ? Lsm[(size_t)s * R + i] : __ldcg(p.Lbuf + row + (int64_t)(k0 + s) * n); },
          wrow, t);
      double c = __dsub_rn(acol[i], dot);
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
    BlockBest lb = block_argmax(bk, bi, bs);
    const long long nseq = seq + 1;
    const int par = static_cast<int>(nseq & 1);
    if (tid == 0) {
      XRec rec;
      rec.key = lb.slot >= 0 ? lb.key : -1.0;
      rec.val = lb.slot >= 0 ? ck[lb.slot] : 0.0;
      rec.diag = lb.slot >= 0 ? dg[lb.slot] : 0.0;
      rec.lidx = lb.slot >= 0 ? static_cast<int>(lb.idx) : INT_MAX;
      rec.phys = lb.slot >= 0 ? r0 + lb.slot : -1;
      rec.has_akk = (pk >= r0 && pk < r0 + rcnt) ? 1 : 0;
      rec.akk = s_akk;
      rec.err = s_lerr;
      p.xrec[(size_t)par * G + cta] = rec;
    }
    seq = nseq;
    xpublish(p.flags, cta, seq);
    if (!xwait(p.flags, G, seq, p.st)) break;

    // ---- identical reduction of all records in every CTA
    if (tid == 0) s_gerr = 0;
    __syncthreads();
    double gk = -1.0;
    long long gi = LLONG_MAX;
    int gs = -1;
    for (int c = tid; c < G; c += nthr) {
      const XRec* rc = p.xrec + (size_t)par * G + c;
      double v = __ldcg(&rc->key);
      int li = __ldcg(&rc->lidx);
      if (v >= 0.0 || v != v) {
        if (better(v, li, gk, gi)) {
          gk = v;
          gi = li;
          gs = c;
        }
      }
      if (__ldcg(&rc->has_akk)) s_gakk = __ldcg(&rc->akk);
      if (__ldcg(&rc->err)) s_gerr = 1;
    }
    BlockBest gb = block_argmax(gk, gi, gs);
    if (s_gerr) break;
    const double akk = s_gakk;
    const bool has_cand = gb.slot >= 0;
    double lam = 0.0, ckr = 0.0, dr = 0.0;
    int r_rel = -1, pr = -1;
    if (has_cand) {
      const XRec* rc = p.xrec + (size_t)par * G + gb.slot;
      lam = __ldcg(&rc->key);
      ckr = __ldcg(&rc->val);
      dr = __ldcg(&rc->diag);
      r_rel = __ldcg(&rc->lidx);
      pr = __ldcg(&rc->phys);
    }

    // ---- SBKP decision (pivot.py:111-128): 0 skip, 1 1x1, 2 1x1-swap, 3 2x2
    int kind, s;
    const double athr = __dmul_rn(alpha, lam);
    if (!has_cand || lam == 0.0) {
      kind = 0;
      s = 1;
    } else if (fabs(akk) >= athr) {
      kind = 1;
      s = 1;
    } else if (fabs(dr) >= athr) {
      kind = 2;
      s = 1;
    } else {
      kind = 3;
      s = 2;
    }
    if (s == 2 && t > 0 && t + 2 > width) break;  // defer (factor.py:622-623)

    // ---- symmetric swaps as permutation bookkeeping (factor.py:624-630)
    int p_t = pk, p_t1 = -1;
    if (kind == 2) {
      // swap(k, r)
      if (tid == 0) {
        win[t] = pr;
        if (r_rel < Wn) win[r_rel] = pk;
      }
      if (tid == 0) {
        if (pr >= r0 && pr < r0 + rcnt) lpos[pr - r0] = t;
        if (pk >= r0 && pk < r0 + rcnt) lpos[pk - r0] = r_rel;
      }
      p_t = pr;
    } else if (kind == 3) {
      if (r_rel != t + 1) {
        if (tid == 0) {
          const int p1 = win[t + 1];
          win[t + 1] = pr;
          if (r_rel < Wn) win[r_rel] = p1;
          if (pr >= r0 && pr < r0 + rcnt) lpos[pr - r0] = t + 1;
          if (p1 >= r0 && p1 < r0 + rcnt) lpos[p1 - r0] = r_rel;
        }
      }
      p_t1 = pr;
    }
    __syncthreads();

    // ---- phase B: partner column when needed, multipliers, writes
    const int64_t kglob = k0 + t;
    if (kind >= 2) {
      for (int s2 = tid; s2 < t; s2 += nthr) wrrow[s2] = __ldcg(p.W + (k0 + pr) + (int64_t)s2 * n);
      __syncthreads();
      for (int i = tid; i < rcnt; i += nthr) {
        if (lpos[i] < t) continue;
        const int64_t row = k0 + r0 + i;
        double dot = chain_dot4(
            [&](int s3) { return s3 < Ls ? Lsm[(size_t)s3 * R + i] : __ldcg(p.Lbuf + row + (int64_t)(k0 + s3) * n); },
            wrrow, t);
        cr[i] = __dsub_rn(sym_lower(A, n, row, k0 + pr), dot);
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
      d11 = akk;
      d21 = ckr;
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
    __syncthreads();  // cr complete before use; lpos updates visible
    bool lerr = false;
    for (int i = tid; i < rcnt; i += nthr) {
      const int lp = lpos[i];
      if (lp < t) continue;
      const int64_t row = k0 + r0 + i;
      if (kind <= 1) {
        const double c = ck[i];
        p.W[row + (int64_t)t * n] = c;
        if (lp > t) {
          double l = (kind == 0) ? 0.0 : __ddiv_rn(c, d11);
          if (!isfinite(l)) lerr = true;
          p.Lbuf[row + kglob * n] = l;
          if (t < Ls) Lsm[(size_t)t * R + i] = l;
          dg[i] = __fma_rn(-l, c, dg[i]);
        }
      } else if (kind == 2) {
        const double c = cr[i];
        p.W[row + (int64_t)t * n] = c;
        if (lp > t) {
          double l = __ddiv_rn(c, d11);
          if (!isfinite(l)) lerr = true;
          p.Lbuf[row + kglob * n] = l;
          if (t < Ls) Lsm[(size_t)t * R + i] = l;
          dg[i] = __fma_rn(-l, c, dg[i]);
        }
      } else {
        const double c0 = ck[i], c1 = cr[i];
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

    // ---- next pivot: its W row (older entries from memory, this step's entries
    //      recomputed redundantly with the owner's exact arithmetic) + A column prefetch
    const int tn = t + s;
    __syncthreads();
    if (tn < width && k0 + tn < n) {
      const int pn = win[tn];
      if (tid == 0) {
        const int64_t rown = k0 + pn;
        auto lrow = [&](int s3) { return __ldcg(p.Lbuf + rown + (int64_t)(k0 + s3) * n); };
        double v0, v1 = 0.0;
        if (kind <= 1) {
          v0 = __dsub_rn(sym_lower(A, n, rown, k0 + pk), chain_dot4(lrow, wrow, t));
        } else if (kind == 2) {
          v0 = __dsub_rn(sym_lower(A, n, rown, k0 + pr), chain_dot4(lrow, wrrow, t));
        } else {
          v0 = __dsub_rn(sym_lower(A, n, rown, k0 + pk), chain_dot4(lrow, wrow, t));
          v1 = __dsub_rn(sym_lower(A, n, rown, k0 + pr), chain_dot4(lrow, wrrow, t));
        }
        s_coef = v0;  // scratch broadcast
        s_gakk = v1;
      }
      __syncthreads();
      const double v0 = s_coef, v1 = s_gakk;
      for (int s3 = tid; s3 < tn; s3 += nthr) {
        double w;
        if (s3 < t) {
          w = __ldcg(p.W + (k0 + pn) + (int64_t)s3 * n);
        } else {
          w = (s3 == t) ? v0 : v1;
        }
        wrow[s3] = w;
      }
      for (int i = tid; i < rcnt; i += nthr) {
        if (lpos[i] >= tn) acol[i] = sym_lower(A, n, k0 + r0 + i, k0 + pn);
      }
      pk = pn;
    }
    t = tn;
    __syncthreads();
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
  }
}

cudaError_t panel_init_attributes(int max_dyn_smem) {
  return cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem);
}

int panel_static_smem_bytes() {
  cudaFuncAttributes attr;
  if (cudaFuncGetAttributes(&attr, panel_kernel) != cudaSuccess) return 4096;
  return static_cast<int>(attr.sharedSizeBytes);
}

cudaError_t launch_panel(const PanelParams& prm, int G, size_t smem, cudaStream_t st) {
  PanelParams copy = prm;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(panel_kernel), dim3(G), dim3(kPanelThreads), args,
                                     smem, st);
}

}  // namespace rcp
