// Trailing Schur update, second generation: two MMA warps per SM sub-partition.
//
// schur_ws_kernel (schur_ws.cuh) runs one MMA warp per sub-partition; its DMMA pipe stalls at
// ~0.7 because a single warp cannot fill the fixed issue gap between its own consecutive
// DMMA.8x8x4 (profiles/r02_ncu_schur_c3_stalls.txt).  Here a CTA works on a 128x128 "supertile"
// = two adjacent 128x64 tiles of the same row block:
//   warps 0-3   MMA group 0: left  half (columns n0 .. n0+63),   64x32 warp tiles
//   warps 4-7   MMA group 1: right half (columns n0+64 .. +127), 64x32 warp tiles
//   warps 8-9   producer:  cp.async ring, one stage = -L21[128 x 16] + W21[128 x 16], chunk-major
//                          (no row padding: 3 stages + both C tiles fit in 227 KB)
//   warps 10-11 epilogue:  per half: C-in gather through the panel permutation into the half's
//                          C tile, then lower (column-wise) + mirror (row-wise) stores
// Warps w and w+4 share a sub-partition, so each has two independent DMMA streams.  The A operand
// stage is shared by both groups.  Each half has ONE C tile (2 x 66.5 KB; double-buffering both
// would need 266 KB): the gather of the next supertile's half is issued right after the drain of
// the current one and has the whole next mainloop (twice as long per group) to land.
// Register budget (launch 384 x 168): setmaxnreg 216 for the MMA groups, 72 for warps 8-11.
// Arithmetic is the same as schur_ws_kernel (zero-initialised accumulators, k ascending, one
// add into C-in): outputs are bit-identical.
#pragma once
#include <cuda.h>

#include "schur_ws.cuh"

namespace rcp {

namespace ws2 {

using ws::BM;
using ws::BN;
using ws::mbar_arrive;
using ws::mbar_arrive_cpasync;
using ws::mbar_init;
using ws::mbar_wait;
using ws::named_sync;
constexpr int SN = 2 * BN;  // supertile width
#ifndef RCP_WS2_KS
#define RCP_WS2_KS 16
#endif
constexpr int KS = RCP_WS2_KS;        // k-columns per operand stage (8 or 16)
constexpr int STAGES = 48 / KS;       // 96 KB of operand stages either way
constexpr int kMmaWarps = 8, kThreads = 384, kProdThreads = 64, kEpiThreads = 64;
constexpr int kCStride = BM + 2;
#ifndef RCP_WS2_MMAREGS
#define RCP_WS2_MMAREGS 208
#endif
#ifndef RCP_WS2_AUXREGS
#define RCP_WS2_AUXREGS 88
#endif
constexpr int kMmaRegs = RCP_WS2_MMAREGS, kAuxRegs = RCP_WS2_AUXREGS;

struct Smem {
  double a[STAGES][BM * KS];  // element (row, k) at opidx(BM, row, k)
  double b[STAGES][SN * KS];
  double c[2][BN][kCStride];
  int colmap[2][BN];
  unsigned long long full[STAGES], empty[STAGES], cin[2], accd[2];
};

// Operand stage layout, chunk-major: element (row, k) of a ROWS x 16 slice lives at
// (k / 4) * ROWS * 4 + row * 4 + (k & 3).  A DMMA fragment load (rows g = 0..7, k = 4c + q) reads
// 32 consecutive doubles: bank-conflict free without padding, and every fragment address is the
// thread's base plus an immediate (no per-chunk address arithmetic in the mainloop).
RCP_HD int opidx(int rows, int row, int k) { return (k >> 2) * rows * 4 + row * 4 + (k & 3); }

// Supertile s of the lower triangle (diagonal included): row block I holds I + 1 supertiles.
RCP_HD void super_of(long long s, int64_t& m0, int64_t& n0) {
  long long I = static_cast<long long>((sqrt(8.0 * (double)s + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) / 2 > s) --I;
  while ((I + 1) * (I + 2) / 2 <= s) ++I;
  m0 = I * BM;
  n0 = (s - I * (I + 1) / 2) * SN;
}
// Supertile list of one panel's update: nbi (nbi + 1) / 2 lower-triangle supertiles, then
// nbi * nbp2 sketch supertiles (sketch rows n0 .. n0+127 of the 128-row block m0).
RCP_HD bool super_at(long long s, long long s_tri, int nbp2, int64_t& m0, int64_t& n0) {
  if (s < s_tri) {
    super_of(s, m0, n0);
    return false;
  }
  const long long sx = s - s_tri;
  m0 = (sx / nbp2) * BM;
  n0 = (sx % nbp2) * SN;
  return true;
}

#ifndef RCP_WS2_SETMAXNREG
#define RCP_WS2_SETMAXNREG 1
#endif
// The supertiles CTA `cta` of a `grid`-CTA launch takes on device `part` of `nparts` sharing the update:
// s = first, first + step, ...  (supertiles dealt round robin to the devices, then to their CTAs).
RCP_HD void super_sequence(bool multi, int part, int nparts, int cta, int grid, long long& first, long long& step) {
  first = multi ? part + (long long)nparts * cta : (long long)cta;
  step = multi ? (long long)nparts * grid : (long long)grid;
}

template <int N>
RCP_D void setmaxnreg_inc() {
#if RCP_WS2_SETMAXNREG
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
#endif
}
template <int N>
RCP_D void setmaxnreg_dec() {
#if RCP_WS2_SETMAXNREG
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
#endif
}

// Raw-address copies / stores for the interior-tile fast paths; kHints adds L2 cache policies
// (operand panels evict_last: every CTA re-reads them; C-in / C-out streams evict_first).
typedef unsigned long long u64a;
template <bool H>
RCP_D void cpa8(unsigned s, u64a g, u64a pol) {
  if (H) asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(s), "l"(g), "l"(pol) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(g) : "memory");
}
template <bool H>
RCP_D void cpa16(unsigned s, u64a g, u64a pol) {
  if (H) asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(g), "l"(pol) : "memory");
  else asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
template <bool H>
RCP_D void stg(u64a g, double v, u64a pol) {
  if (H) asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(g), "d"(v), "l"(pol) : "memory");
  else asm volatile("st.global.f64 [%0], %1;" ::"l"(g), "d"(v) : "memory");
}
// TMA: 3-D tiled load of one operand stage.  The tensor map views a K-contiguous panel
// [rows][tpad] as {4 (k inside a chunk), rows, tpad / 4 (chunks)} with box {4, 128, 4}, so the box
// lands in shared memory chunk-major ([chunk][row][4]) -- the layout the fragment loads want.
template <bool H>
RCP_D void tma_load_3d(unsigned dst, const CUtensorMap* tm, int c0, int c1, int c2, unsigned bar, u64a pol) {
  if (H)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(dst), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
RCP_D void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ws::sa(b)), "r"(bytes) : "memory");
}
RCP_D u64a policy_evict_last() {
  u64a p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

}  // namespace ws2

// kHints: 0 none, 1 operand panels evict_last, 2 also C-in / C-out evict_first
// kMulti: the update is shared by `nparts` devices (dist.cuh): this launch takes every nparts-th
// supertile; a worker resolves C-in / C-out / the descriptor from rank 0's signal (dyn)
// kTma: operand stages filled by TMA (one elected thread, mbarrier transaction counts) instead of
// 64 threads' cp.async.
template <int kHints, bool kTma, bool kMulti>
__global__ void __launch_bounds__(ws2::kThreads, 1)
schur_ws2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmY, const double* __restrict__ Lneg, const double* __restrict__ Wg, int tpad, int Kl,
                 const double* __restrict__ ain, double* __restrict__ aout, const int* __restrict__ phys, int64_t n,
                 int64_t k, int64_t mp, const PanelDesc* __restrict__ d, const double* __restrict__ ysk,
                 const double* __restrict__ bin, double* __restrict__ bout, int P,
                 unsigned long long* __restrict__ tstamp, int part, int nparts, const SchurDyn* __restrict__ dyn) {
  using namespace ws2;
  if (kMulti && dyn) {  // multi-GPU worker: buffers resolved on the device from rank 0's signal
    if (!dyn->go) return;
    ain = dyn->ain;
    aout = dyn->aout;
    d = dyn->d;
  }
  if (d) {  // device-driven: the panel outcome comes from the committed descriptor
    if (!d->ok || d->t <= 0 || d->k_end >= n) return;
    k = d->k_end;
    mp = n - k;
    Kl = ((d->t + kBK - 1) / kBK) * kBK;
  }
  const long long nbi = (mp + BM - 1) / BM;
  const int nbp2 = ysk ? (P + SN - 1) / SN : 0;  // sketch supertiles per 128-row block
  const long long s_tri = nbi * (nbi + 1) / 2;
  const long long s_all = s_tri + nbi * nbp2;
  unsigned long long* const ts_schur = (tstamp && d) ? tstamp + 4 * (size_t)d->pidx + 2 : nullptr;
  stamp_start(ts_schur);
  extern __shared__ __align__(128) unsigned char smem_ws2[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_ws2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = Kl / KS;
  long long x0, xs;
  super_sequence(kMulti, part, nparts, (int)blockIdx.x, (int)gridDim.x, x0, xs);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sm.full[s], kTma ? 1 : kProdThreads);
      mbar_init(&sm.empty[s], kMmaWarps);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&sm.cin[h], kEpiThreads);
      mbar_init(&sm.accd[h], kMmaWarps / 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp < kMmaWarps) {
    // ======================= MMA groups =======================
    setmaxnreg_inc<kMmaRegs>();
    // Identity shuffles: ptxas otherwise re-derives lane / warp / fragment offsets from S2R SR_TID.X
    // inside the k-loop (a ~50-cycle special-register read per stage); a SHFL result is not
    // rematerialised, so these stay in registers.
    const int mlane = __shfl_sync(0xffffffffu, lane, lane), mwarp = __shfl_sync(0xffffffffu, warp, lane);
    const int h = mwarp >> 2, w = mwarp & 3;
    const int g = mlane >> 2, q = mlane & 3;
    const int wm0 = (w >> 1) * 64, wc0 = (w & 1) * 32;  // rows of A / columns inside the half
    constexpr int MF = 8, NF = 4;
    // fragment offsets inside a stage: row (base + 8 i + g), k = 4 c + q
    const int aoff = (wm0 + g) * 4 + q;
    const int boff = (h * BN + wc0 + g) * 4 + q;
    unsigned stage = 0, sphase = 0;
    int it = 0;
    for (long long x = x0; x < s_all; x += xs, ++it) {
      double acc[MF][NF][2];
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      // Fragments are double-buffered across chunks AND stages: the first chunk of the next stage is
      // fetched during the last chunk's DMMAs of the current one (no LDS burst at a stage boundary).
      double af[2][MF], bf[2][NF];
      mbar_wait(&sm.full[stage], sphase);
      {
        const double* as = sm.a[stage] + aoff;
        const double* bs = sm.b[stage] + boff;
#pragma unroll
        for (int i = 0; i < MF; ++i) af[0][i] = as[i * 32];
#pragma unroll
        for (int j = 0; j < NF; ++j) bf[0][j] = bs[j * 32];
      }
      for (int kt = 0; kt < KT; ++kt) {
        const double* as = sm.a[stage] + aoff;
        const double* bs = sm.b[stage] + boff;
        unsigned nstage = stage + 1, nphase = sphase;
        if (nstage == STAGES) {
          nstage = 0;
          nphase ^= 1;
        }
#pragma unroll
        for (int c = 0; c < KS / 4; ++c) {
          const int cb = c & 1;
          if (c + 1 < KS / 4) {
#pragma unroll
            for (int i = 0; i < MF; ++i) af[cb ^ 1][i] = as[(c + 1) * BM * 4 + i * 32];
#pragma unroll
            for (int j = 0; j < NF; ++j) bf[cb ^ 1][j] = bs[(c + 1) * SN * 4 + j * 32];
          } else if (kt + 1 < KT) {
            mbar_wait(&sm.full[nstage], nphase);
            const double* an = sm.a[nstage] + aoff;
            const double* bn = sm.b[nstage] + boff;
#pragma unroll
            for (int i = 0; i < MF; ++i) af[cb ^ 1][i] = an[i * 32];
#pragma unroll
            for (int j = 0; j < NF; ++j) bf[cb ^ 1][j] = bn[j * 32];
          }
#pragma unroll
          for (int j = 0; j < NF; ++j)
#pragma unroll
            for (int i = 0; i < MF; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cb][i], bf[cb][j]);
        }
        __syncwarp();
        if (mlane == 0) mbar_arrive(&sm.empty[stage]);
        stage = nstage;
        sphase = nphase;
      }
      // add into the half's C tile once its C-in has landed
      mbar_wait(&sm.cin[h], it & 1);
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int li = wm0 + 8 * i + g, lj = wc0 + 8 * j + 2 * q;
          sm.c[h][lj][li] = __dadd_rn(sm.c[h][lj][li], acc[i][j][0]);
          sm.c[h][lj + 1][li] = __dadd_rn(sm.c[h][lj + 1][li], acc[i][j][1]);
        }
      __syncwarp();
      if (mlane == 0) mbar_arrive(&sm.accd[h]);
    }
  } else {
    setmaxnreg_dec<kAuxRegs>();
    if (warp < kMmaWarps + 2) {
      // ======================= producer warps =======================
      const int pt = tid - 32 * kMmaWarps;  // 0..63
      constexpr int TPR = KS / 2;           // threads per operand row (16 bytes each)
      constexpr int RPP = 64 / TPR;         // rows per pass of the 64 producer threads
      const int srow = pt / TPR, c16 = pt % TPR;
      const int soff = c16 * 2;
      const int dofs = opidx(BM, srow, soff);  // opidx(row = srow + RPP u, soff) = dofs + 4 RPP u  (BM == SN)
      static_assert(BM == SN, "operand stages share the row count");
      unsigned stage = 0, ephase = 1;  // fresh "empty" barriers count as released
      const u64a pol_keep = kHints >= 1 ? policy_evict_last() : 0;
      if (kTma) {
        if (pt == 0) {  // one elected thread feeds the ring
          for (long long x = x0; x < s_all; x += xs) {
            int64_t m0, n0;
            const bool skt = super_at(x, s_tri, nbp2, m0, n0);
            const CUtensorMap* tb = skt ? &tmY : &tmB;
            for (int kt = 0; kt < KT; ++kt) {
              mbar_wait(&sm.empty[stage], ephase);
              mbar_expect_tx(&sm.full[stage], (unsigned)(sizeof(double) * (BM + SN) * KS));
              tma_load_3d<(kHints >= 1)>(ws::sa(sm.a[stage]), &tmA, 0, (int)m0, kt * (KS / 4), ws::sa(&sm.full[stage]),
                                         pol_keep);
              tma_load_3d<(kHints >= 1)>(ws::sa(sm.b[stage]), tb, 0, (int)n0, kt * (KS / 4), ws::sa(&sm.full[stage]),
                                         pol_keep);
              if (++stage == STAGES) {
                stage = 0;
                ephase ^= 1;
              }
            }
          }
        }
      } else
      for (long long x = x0; x < s_all; x += xs) {
        int64_t m0, n0;
        const bool skt = super_at(x, s_tri, nbp2, m0, n0);
        const double* ab = Lneg + (m0 + srow) * (int64_t)tpad + soff;
        const double* bsrc = skt ? ysk : Wg;
        const int64_t blim = skt ? P : mp;
        const double* bb = bsrc + (n0 + srow) * (int64_t)tpad + soff;
        const int64_t step = RPP * (int64_t)tpad;
        const bool interior = m0 + BM <= mp && n0 + SN <= blim;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&sm.empty[stage], ephase);
          const int64_t k0 = (int64_t)kt * KS;
          double* da = sm.a[stage] + dofs;
          double* db = sm.b[stage] + dofs;
          if (interior) {  // no predicates, immediate strides
            const unsigned t64 = (unsigned)tpad * (8u * RPP);  // bytes between rows r and r + RPP
            const u64a ua = (u64a)(ab + k0), ub = (u64a)(bb + k0);
            const unsigned sda = ws::sa(da), sdb = ws::sa(db);
#pragma unroll
            for (int u = 0; u < BM / RPP; ++u) cpa16<(kHints >= 1)>(sda + u * 4 * RPP * 8, ua + (u64a)u * t64, pol_keep);
#pragma unroll
            for (int u = 0; u < SN / RPP; ++u) cpa16<(kHints >= 1)>(sdb + u * 4 * RPP * 8, ub + (u64a)u * t64, pol_keep);
            mbar_arrive_cpasync(&sm.full[stage]);
            if (++stage == STAGES) {
              stage = 0;
              ephase ^= 1;
            }
            continue;
          }
#pragma unroll
          for (int u = 0; u < BM / RPP; ++u) {
            const bool ok = m0 + srow + RPP * u < mp;
            cp_async16(da + u * 4 * RPP, ok ? ab + u * step + k0 : Lneg, ok);
          }
#pragma unroll
          for (int u = 0; u < SN / RPP; ++u) {
            const bool ok = n0 + srow + RPP * u < blim;
            cp_async16(db + u * 4 * RPP, ok ? bb + u * step + k0 : Lneg, ok);
          }
          mbar_arrive_cpasync(&sm.full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            ephase ^= 1;
          }
        }
      }
    } else {
      // ======================= epilogue warps =======================
      const int et = tid - 32 * kMmaWarps - 64;  // 0..63
      const unsigned n8 = (unsigned)n * 8u;  // column stride in bytes (n < 2^29)
      const u64a pol_stream = kHints >= 2 ? policy_evict_first() : 0;
      auto gather = [&](long long x, int h) {
        int64_t m0, n0;
        const bool skt = super_at(x, s_tri, nbp2, m0, n0);
        n0 += h * BN;
        if (skt) {  // sketch tile: C(i, j) = B[n0 + j, phys[m0 + i]] (threads along j)
          const bool col_ok = n0 + et < P;
          for (int i = 0; i < BM; ++i) {
            const int64_t gi = m0 + i;
            const bool ok = col_ok && gi < mp;
            cp_async8(&sm.c[h][et][i], ok ? bin + (n0 + et) + (int64_t)phys[gi] * P : bin, ok);
          }
          mbar_arrive_cpasync(&sm.cin[h]);
          return;
        }
        sm.colmap[h][et] = (n0 + et < mp) ? phys[n0 + et] : 0;
        if (RCP_FULL_STORAGE && m0 + BM <= mp && n0 + BN <= m0) {
          // interior tile (all rows valid, strictly below the diagonal): one IMAD.WIDE + one
          // LDGSTS per element, column offsets read four at a time
          const int pa = phys[m0 + et], pb = phys[m0 + et + 64];
          named_sync(1, kEpiThreads);
          const u64a ra = (u64a)(ain + pa), rb = (u64a)(ain + pb);
          const unsigned sA = ws::sa(&sm.c[h][0][et]), sB = sA + 64 * 8;
#pragma unroll
          for (int j4 = 0; j4 < BN; j4 += 4) {
            const int4 cm = *reinterpret_cast<const int4*>(&sm.colmap[h][j4]);
            const unsigned cc[4] = {(unsigned)cm.x, (unsigned)cm.y, (unsigned)cm.z, (unsigned)cm.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const u64a off = (u64a)cc[u] * n8;
              cpa8<(kHints >= 2)>(sA + (j4 + u) * kCStride * 8, ra + off, pol_stream);
              cpa8<(kHints >= 2)>(sB + (j4 + u) * kCStride * 8, rb + off, pol_stream);
            }
          }
          mbar_arrive_cpasync(&sm.cin[h]);
          return;
        }
        named_sync(1, kEpiThreads);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int i = et + 64 * hh;
          const int64_t gi = m0 + i;
          const bool row_ok = gi < mp;
          const int pi = row_ok ? phys[gi] : 0;
#pragma unroll 8
          for (int j = 0; j < BN; ++j) {
            const bool ok = row_ok && (n0 + j <= gi);
            cp_async8(&sm.c[h][j][i], ok ? ain + sym_index(n, pi, sm.colmap[h][j]) : ain, ok);
          }
        }
        mbar_arrive_cpasync(&sm.cin[h]);
      };
      auto drain = [&](long long x, int h) {
        int64_t m0, n0;
        const bool skt = super_at(x, s_tri, nbp2, m0, n0);
        n0 += h * BN;
        if (skt) {  // corrected sketch columns k + m0 + i, rows n0 + j (threads along j)
          if (n0 + et < P) {
            const int imax = (int)(mp - m0 < BM ? mp - m0 : BM);
            double* dst = bout + (n0 + et) + (k + m0) * (int64_t)P;
            const double* src = &sm.c[h][et][0];
            int i = 0;
            for (; i + 8 <= imax; i += 8) {
              double v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = src[i + u];
#pragma unroll
              for (int u = 0; u < 8; ++u) dst[(int64_t)(i + u) * P] = v[u];
            }
            for (; i < imax; ++i) dst[(int64_t)i * P] = src[i];
          }
          return;
        }
        if (RCP_FULL_STORAGE && m0 + BM <= mp && n0 + BN <= m0) {  // interior tile
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // lower part: thread = row, columns by immediate strides
            const int i = et + 64 * hh;
            const u64a dst0 = (u64a)(aout + (k + m0 + i) + (k + n0) * n);
            const double* src = &sm.c[h][0][i];
#pragma unroll
            for (int j = 0; j < BN; j += 8) {
              double v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = src[(j + u) * kCStride];
#pragma unroll
              for (int u = 0; u < 8; ++u) stg<(kHints >= 2)>(dst0 + (u64a)(unsigned)(j + u) * n8, v[u], pol_stream);
            }
          }
          {  // mirror: thread = tile column et -> row k+n0+et, 16-byte smem reads
            const u64a dst0 = (u64a)(aout + (k + n0 + et) + (k + m0) * n);
            const double2* src = reinterpret_cast<const double2*>(&sm.c[h][et][0]);
#pragma unroll
            for (int i = 0; i < BM; i += 8) {
              double2 v[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) v[u] = src[i / 2 + u];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                stg<(kHints >= 2)>(dst0 + (u64a)(unsigned)(i + 2 * u) * n8, v[u].x, pol_stream);
                stg<(kHints >= 2)>(dst0 + (u64a)(unsigned)(i + 2 * u + 1) * n8, v[u].y, pol_stream);
              }
            }
          }
          return;
        }
        // lower part: column n0+j, rows m0..m0+127 (threads along rows)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int i = et + 64 * hh;
          const int64_t gi = m0 + i;
          if (gi < mp) {
            const int64_t jl = (mp < gi + 1 ? mp : gi + 1) - n0;
            const int jmax = (int)(jl < BN ? (jl > 0 ? jl : 0) : BN);
            double* dst = aout + (k + gi) + (k + n0) * n;
            const double* src = &sm.c[h][0][i];
            int j = 0;
            for (; j + 8 <= jmax; j += 8, dst += 8 * n) {
              double v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = src[(j + u) * kCStride];
#pragma unroll
              for (int u = 0; u < 8; ++u) dst[u * n] = v[u];
            }
            for (; j < jmax; ++j, dst += n) *dst = src[j * kCStride];
          }
        }
        // mirror of the strictly-lower part: row k+n0+j, columns k+m0+i (threads along j)
        if (RCP_FULL_STORAGE && m0 + BM - 1 > n0) {
          const int64_t gj = n0 + et;
          if (gj < mp) {
            const int imax = (int)(mp - m0 < BM ? mp - m0 : BM);
            // first i with m0 + i > gj
            const int64_t il = gj + 1 - m0;
            int i = (int)(il > 0 ? il : 0);
            double* dst = aout + (k + gj) + (k + m0 + i) * n;
            const double* src = &sm.c[h][et][0];
            for (; i + 8 <= imax; i += 8, dst += 8 * n) {
              double v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = src[i + u];
#pragma unroll
              for (int u = 0; u < 8; ++u) dst[u * n] = v[u];
            }
            for (; i < imax; ++i, dst += n) *dst = src[i];
          }
        }
      };
      if (x0 < s_all) {
        gather(x0, 0);
        gather(x0, 1);
      }
      int it = 0;
      for (long long x = x0; x < s_all; x += xs, ++it) {
        const bool more = x + xs < s_all;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&sm.accd[h], it & 1);
          drain(x, h);
          named_sync(1, kEpiThreads);  // every epilogue thread done reading the half's tile
          if (more) gather(x + xs, h);
        }
      }
    }
  }
  __syncthreads();
  stamp_end(ts_schur ? ts_schur + 1 : nullptr);
}

inline size_t schur_ws2_smem_bytes() { return sizeof(ws2::Smem); }

}  // namespace rcp
