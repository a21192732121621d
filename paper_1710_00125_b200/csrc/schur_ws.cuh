// Warp-specialised persistent trailing Schur update  A22 <- A22 - L21 W21^T
// (factor.py:369-379 + core.py:115-119), FP64 DMMA.
//
// Why: at K = t <= 129 each lower element costs ~24 B of HBM traffic (read C, write C and
// its mirror) for 2t flops (~10.7 flop/B, only ~2x the B200 FP64 ridge), so a tile's
// epilogue is about as long as half its MMA mainloop.  Instead of serialising them, one
// persistent CTA per SM splits its 8 warps into three roles that run concurrently:
//   warps 0-3  MMA:       DMMA.8x8x4 mainloop of the 128x64 tile (4 warps x 64x32), then add
//                         the accumulators into the tile's C buffer
//   warps 4-5  producer:  cp.async operand ring (3 stages of -L21 / W21 k-slices)
//   warps 6-7  epilogue:  C-in gather through the panel permutation into a double-buffered
//                         C tile, then column-wise (lower) and row-wise (mirror) stores
// Roles synchronise through shared-memory mbarriers (cp.async.mbarrier.arrive for data
// arrival), so the tensor pipe keeps issuing while the previous tile drains to HBM.
#pragma once
#include "panel.cuh"
#include "dist.cuh"
#include "gemm_dmma.cuh"

namespace rcp {

namespace ws {

#ifndef RCP_WS_STAGES
#define RCP_WS_STAGES 3
#endif
#ifndef RCP_WS_NBUF
#define RCP_WS_NBUF 2
#endif
constexpr int BM = 128, BN = 64, STAGES = RCP_WS_STAGES;
constexpr int NBUF = RCP_WS_NBUF;  // C tile buffers (1: the epilogue drains tile t during mainloop t+1)
#ifndef RCP_WS_MMA_WARPS
#define RCP_WS_MMA_WARPS 4
#endif
constexpr int kMmaWarps = RCP_WS_MMA_WARPS;  // 4: 64x32 warp tiles, 8: 32x32 warp tiles
constexpr int kThreads = 32 * kMmaWarps + 128;
constexpr int kProdThreads = 64, kEpiThreads = 64;
#ifndef RCP_WS_CSTRIDE
#define RCP_WS_CSTRIDE (BM + 2)
#endif
// C tile column stride: BM + 2 makes the MMA warps' accumulate (lanes g + 4q) bank-conflict free; the
// epilogue's mirror reads then see 2-way conflicts (BM + 1 is the other way round)
constexpr int kCStride = RCP_WS_CSTRIDE;

struct Smem {
  double a[STAGES][BM][kBK + kPad];
  double b[STAGES][BN][kBK + kPad];
  double c[NBUF][BN][kCStride];
  int colmap[NBUF][BN];
  unsigned long long full[STAGES], empty[STAGES], cin[NBUF], accd[NBUF];
};

RCP_D unsigned sa(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
RCP_D void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count));
}
RCP_D void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
RCP_D void mbar_arrive_cpasync(unsigned long long* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(b)) : "memory");
}
RCP_D bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(sa(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for the phase with `parity` to complete; a watchdog (~4 s) traps instead of hanging.
RCP_D void mbar_wait(unsigned long long* b, unsigned parity) {
  if (mbar_try(b, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(b, parity)) {
    if (clock64() - t0 > 8000000000LL) __trap();
  }
}
#ifndef RCP_WS_ORDER
#define RCP_WS_ORDER 2  // DMMA issue order inside a k-step: 2 = B fragment outer (measured -1.3 % at C3)
#endif
RCP_D void st_c(double* p, double v) { *p = v; }  // (streaming stores measured: no difference)
RCP_D void named_sync(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }

// Lower-triangle tile x -> (m0, n0): row block I holds 2I + 2 column blocks of BN = BM / 2.
RCP_HD void tile_of(long long x, int64_t& m0, int64_t& n0) {
  long long I = static_cast<long long>((sqrt(4.0 * (double)x + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) > x) --I;
  while ((I + 1) * (I + 2) <= x) ++I;
  m0 = I * BM;
  n0 = (x - I * (I + 1)) * BN;
}
// Tile list of one panel's update: nbi (nbi + 1) lower-triangle tiles, then nbi * nbp sketch tiles
// (sketch rows n0..n0+BN of the 128-row block m0).  Returns true for a sketch tile.
RCP_HD bool tile_at(long long x, long long tiles_tri, int nbp, int64_t& m0, int64_t& n0) {
  if (x < tiles_tri) {
    tile_of(x, m0, n0);
    return false;
  }
  const long long sx = x - tiles_tri;
  m0 = (sx / nbp) * BM;
  n0 = (sx % nbp) * BN;
  return true;
}
// The tiles CTA `cta` of a `grid`-CTA launch takes on device `part` of `nparts` sharing the update:
// x = first, first + step, ... (tiles dealt round robin to the devices, then to their CTAs).
RCP_HD void tile_sequence(bool multi, int part, int nparts, int cta, int grid, long long& first, long long& step) {
  first = multi ? part + (long long)nparts * cta : (long long)cta;
  step = multi ? (long long)nparts * grid : (long long)grid;
}

}  // namespace ws

template <bool kMulti>
__global__ void __launch_bounds__(ws::kThreads, 1)
schur_ws_kernel(const double* __restrict__ Lneg, const double* __restrict__ Wg, int tpad, int Kl,
                const double* __restrict__ ain, double* __restrict__ aout, const int* __restrict__ phys, int64_t n,
                int64_t k, int64_t mp, long long tiles, const PanelDesc* __restrict__ d, int part, int nparts,
                const SchurDyn* __restrict__ dyn, const double* __restrict__ ysk = nullptr,
                const double* __restrict__ bin = nullptr, double* __restrict__ bout = nullptr, int P = 0,
                unsigned long long* __restrict__ tstamp = nullptr) {
  // With ysk != nullptr (device-driven, single GPU) the sketch correction B2^T -= L21 Y^T
  // (factor.py:554-565, Y = B1 L11^-T from ysolve) rides along as extra tiles after the lower
  // triangle: A operand = the same -L21 rows, B operand = Y rows, C = the sketch columns
  // gathered through the panel permutation (no mirror).
  using namespace ws;
  if (kMulti && dyn) {  // multi-GPU worker: buffers resolved on the device from rank 0's signal
    if (!dyn->go) return;
    ain = dyn->ain;
    aout = dyn->aout;
    d = dyn->d;
  }
  long long tiles_tri = tiles;
  const int nbp = ysk ? (P + BN - 1) / BN : 0;  // sketch tiles per 128-row block
  if (d) {  // device-driven: the panel outcome comes from the committed descriptor
    if (!d->ok || d->t <= 0 || d->k_end >= n) return;
    k = d->k_end;
    mp = n - k;
    Kl = ((d->t + kBK - 1) / kBK) * kBK;
    const long long nbi = (mp + BM - 1) / BM;
    tiles_tri = nbi * (nbi + 1);
    tiles = tiles_tri + nbi * nbp;
  }
  // tile x: lower-triangle tile (returns false) or sketch tile (true): rows m0 of -L21, sketch
  // rows n0 (of Y and B)
  auto tile_at = [&](long long x, int64_t& m0, int64_t& n0) -> bool { return ws::tile_at(x, tiles_tri, nbp, m0, n0); };
  unsigned long long* const ts_schur = (tstamp && d) ? tstamp + 4 * (size_t)d->pidx + 2 : nullptr;
  stamp_start(ts_schur);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = Kl / kBK;
  // tile sequence of this CTA: x0, x0 + xs, ...  (multi-GPU: tiles are dealt round robin to the
  // nparts devices sharing the update, then to their CTAs)
  long long x0, xs;
  tile_sequence(kMulti, part, nparts, (int)blockIdx.x, (int)gridDim.x, x0, xs);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sm.full[s], kProdThreads);
      mbar_init(&sm.empty[s], kMmaWarps);
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&sm.cin[b], kEpiThreads);
      mbar_init(&sm.accd[b], kMmaWarps);
    }
  }
  __syncthreads();

  if (warp < kMmaWarps) {
    // ======================= MMA warps =======================
    const int g = lane >> 2, q = lane & 3;
    constexpr int WM = BM / (kMmaWarps / 2);  // warps tile 2 (N) x kMmaWarps/2 (M)
    const int wm0 = (warp >> 1) * WM, wn0 = (warp & 1) * 32;
    constexpr int MF = WM / 8, NF = 4;
    unsigned stage = 0, sphase = 0;
    int it = 0;
    for (long long x = x0; x < tiles; x += xs, ++it) {
      double acc[MF][NF][2];
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int kt = 0; kt < KT; ++kt) {
        mbar_wait(&sm.full[stage], sphase);
        double af[2][MF], bf[2][NF];
#pragma unroll
        for (int i = 0; i < MF; ++i) af[0][i] = sm.a[stage][wm0 + 8 * i + g][q];
#pragma unroll
        for (int j = 0; j < NF; ++j) bf[0][j] = sm.b[stage][wn0 + 8 * j + g][q];
#pragma unroll
        for (int kk = 0; kk < kBK; kk += 4) {
          const int cb = (kk / 4) & 1;
          if (kk + 4 < kBK) {
#pragma unroll
            for (int i = 0; i < MF; ++i) af[cb ^ 1][i] = sm.a[stage][wm0 + 8 * i + g][kk + 4 + q];
#pragma unroll
            for (int j = 0; j < NF; ++j) bf[cb ^ 1][j] = sm.b[stage][wn0 + 8 * j + g][kk + 4 + q];
          }
#if RCP_WS_ORDER == 1
          // consecutive DMMAs share neither operand register
#pragma unroll
          for (int d = 0; d < NF; ++d)
#pragma unroll
            for (int i = 0; i < MF; ++i) {
              const int j = (i + d) % NF;
              dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cb][i], bf[cb][j]);
            }
#elif RCP_WS_ORDER == 2
#pragma unroll
          for (int j = 0; j < NF; ++j)
#pragma unroll
            for (int i = 0; i < MF; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cb][i], bf[cb][j]);
#else
#pragma unroll
          for (int i = 0; i < MF; ++i)
#pragma unroll
            for (int j = 0; j < NF; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cb][i], bf[cb][j]);
#endif
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          sphase ^= 1;
        }
      }
      // add into the tile's C buffer once its C-in has landed
      const int b = it % NBUF;
      mbar_wait(&sm.cin[b], (it / NBUF) & 1);
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int li = wm0 + 8 * i + g, lj = wn0 + 8 * j + 2 * q;
          sm.c[b][lj][li] = __dadd_rn(sm.c[b][lj][li], acc[i][j][0]);
          sm.c[b][lj + 1][li] = __dadd_rn(sm.c[b][lj + 1][li], acc[i][j][1]);
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.accd[b]);
    }
  } else if (warp < kMmaWarps + 2) {
    // ======================= producer warps =======================
    const int pt = tid - 32 * kMmaWarps;  // 0..63
    const int srow = pt / 8, soff = (pt % 8) * 2;
    unsigned stage = 0, ephase = 1;  // fresh "empty" barriers count as released
    for (long long x = x0; x < tiles; x += xs) {
      int64_t m0, n0;
      const bool skt = tile_at(x, m0, n0);
      const double* ab = Lneg + (m0 + srow) * (int64_t)tpad + soff;
      const double* bsrc = skt ? ysk : Wg;
      const int64_t blim = skt ? P : mp;
      const double* bb = bsrc + (n0 + srow) * (int64_t)tpad + soff;
      const int64_t step = 8 * (int64_t)tpad;
      for (int kt = 0; kt < KT; ++kt) {
        mbar_wait(&sm.empty[stage], ephase);
        const int64_t k0 = (int64_t)kt * kBK;
#pragma unroll
        for (int u = 0; u < BM / 8; ++u) {
          const bool ok = m0 + srow + 8 * u < mp;
          cp_async16(&sm.a[stage][srow + 8 * u][soff], ok ? ab + u * step + k0 : Lneg, ok);
        }
#pragma unroll
        for (int u = 0; u < BN / 8; ++u) {
          const bool ok = n0 + srow + 8 * u < blim;
          cp_async16(&sm.b[stage][srow + 8 * u][soff], ok ? bb + u * step + k0 : Lneg, ok);
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
    auto gather = [&](long long x, int b) {
      int64_t m0, n0;
      if (tile_at(x, m0, n0)) {  // sketch tile: C(i, j) = B[n0 + j, phys[m0 + i]] (threads along j)
        const bool col_ok = n0 + et < P;
        for (int i = 0; i < BM; ++i) {
          const int64_t gi = m0 + i;
          const bool ok = col_ok && gi < mp;
          cp_async8(&sm.c[b][et][i], ok ? bin + (n0 + et) + (int64_t)phys[gi] * P : bin, ok);
        }
        mbar_arrive_cpasync(&sm.cin[b]);
        return;
      }
      sm.colmap[b][et] = (n0 + et < mp) ? phys[n0 + et] : 0;
      named_sync(1, kEpiThreads);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = et + 64 * h;
        const int64_t gi = m0 + i;
        const bool row_ok = gi < mp;
        const int pi = row_ok ? phys[gi] : 0;
        for (int j = 0; j < BN; ++j) {
          const bool ok = row_ok && (n0 + j <= gi);
          cp_async8(&sm.c[b][j][i], ok ? ain + sym_index(n, pi, sm.colmap[b][j]) : ain, ok);
        }
      }
      mbar_arrive_cpasync(&sm.cin[b]);
    };
    for (int b = 0; b < NBUF; ++b)
      if (x0 + (long long)b * xs < tiles) gather(x0 + (long long)b * xs, b);
    int it = 0;
    for (long long x = x0; x < tiles; x += xs, ++it) {
      const int b = it % NBUF;
      int64_t m0, n0;
      const bool skt = tile_at(x, m0, n0);
      mbar_wait(&sm.accd[b], (it / NBUF) & 1);
      if (skt) {  // corrected sketch columns k + m0 + i, rows n0 + j (threads along j)
        if (n0 + et < P) {
          const int imax = (int)(mp - m0 < BM ? mp - m0 : BM);
          double* dst = bout + (n0 + et) + (k + m0) * (int64_t)P;
          for (int i = 0; i < imax; ++i, dst += P) st_c(dst, sm.c[b][et][i]);
        }
        named_sync(1, kEpiThreads);
        if (x + (long long)NBUF * xs < tiles) gather(x + (long long)NBUF * xs, b);
        continue;
      }
      // lower part: column n0+j, rows m0..m0+127 (threads along rows)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = et + 64 * h;
        const int64_t gi = m0 + i;
        if (gi < mp) {
          const int64_t jl = (mp < gi + 1 ? mp : gi + 1) - n0;
          const int jmax = (int)(jl < BN ? (jl > 0 ? jl : 0) : BN);
          double* dst = aout + (k + gi) + (k + n0) * n;
          for (int j = 0; j < jmax; ++j, dst += n) st_c(dst, sm.c[b][j][i]);
        }
      }
      // mirror of the strictly-lower part: row k+n0+j, columns k+m0+i (threads along j)
      if (RCP_FULL_STORAGE && m0 + BM - 1 > n0) {
        const int64_t gj = n0 + et;
        if (gj < mp) {
          double* dst = aout + (k + gj) + (k + m0) * n;
          const int imax = (int)(mp - m0 < BM ? mp - m0 : BM);
          for (int i = 0; i < imax; ++i, dst += n)
            if (m0 + i > gj) st_c(dst, sm.c[b][et][i]);
        }
      }
      named_sync(1, kEpiThreads);  // every epilogue thread done reading buffer b
      if (x + (long long)NBUF * xs < tiles) gather(x + (long long)NBUF * xs, b);
    }
  }
  __syncthreads();
  stamp_end(ts_schur ? ts_schur + 1 : nullptr);
}

inline size_t schur_ws_smem_bytes() { return sizeof(ws::Smem); }



}  // namespace rcp
