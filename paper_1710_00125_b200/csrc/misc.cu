// Bandwidth-bound helper kernels of the RCP path: input validation + copy, sketch
// norms, the per-panel gather (applies the panel's deferred permutation to the
// operands of the trailing update), the small triangular sketch solve, the final
// L assembly, statistics and the deficient-tail fill.
#include <algorithm>
#include <cfloat>
#include "misc.cuh"
#include "panel.cuh"
#include "rcp_common.cuh"

namespace rcp {

namespace {

__device__ double block_max(double v) {
  __shared__ double sm[32];
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = (blockDim.x * blockDim.y + 31) >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? sm[lane] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  }
  return v;  // valid in thread (0, 0)
}

// Exact-symmetry / finiteness check (core.py:48-53, factor.py:278-281), max|A|
// (factor.py:286) and copy into the workspace, 32x32 tiles.
// One 32x32 tile pair per block: tile (I, J) with I >= J and its mirror (J, I), each read once
// from the input and written once to the workspace; the exact-symmetry check compares the two in
// shared memory (core.py:48-53), finiteness and max|A| on the way (factor.py:280-286).
// half != 0: only the upper triangle of a (column-major view: a(r, c) for r <= c, i.e. the
// lower triangle of a row-major host matrix) was transferred and its exact symmetry is
// checked on the host (rcp_factor_host); the kernel mirrors it and checks finiteness / max|A|.
__global__ void validate_copy_kernel(const double* __restrict__ a, int64_t lda, int64_t n,
                                     double* __restrict__ out, int* flags, double* amax, int half) {
  __shared__ double tl[32][33];  // tile (I, J): tl[x][y] = a(bi + y, bj + x)  (x = column offset)
  __shared__ double tu[32][33];  // tile (J, I): tu[x][y] = a(bj + y, bi + x)
  const long long pid = blockIdx.x;
  long long I = static_cast<long long>((sqrt(8.0 * (double)pid + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) / 2 > pid) --I;
  while ((I + 1) * (I + 2) / 2 <= pid) ++I;
  const long long J = pid - I * (I + 1) / 2;
  const int64_t bi = I * 32, bj = J * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  int asym = 0, nonfin = 0;
  double mx = 0.0;
  for (int r = ty; r < 32; r += 8) {  // coalesced along rows (tx) of column bj + r / bi + r
    const int64_t il = bi + tx, jl = bj + r;
    double v = 0.0;
    if (il < n && jl < n && !(half && I != J)) {
      v = a[il + jl * lda];
      out[il + jl * n] = v;
      nonfin |= !isfinite(v);
      mx = fmax(mx, fabs(v));
    }
    tl[r][tx] = v;
    if (I != J) {
      const int64_t iu = bj + tx, ju = bi + r;
      double w = 0.0;
      if (iu < n && ju < n) {
        w = a[iu + ju * lda];
        out[iu + ju * n] = w;
        nonfin |= !isfinite(w);
        mx = fmax(mx, fabs(w));
      }
      tu[r][tx] = w;
    }
  }
  __syncthreads();
  if (half) {  // tile (I, J) = transpose of the transferred tile (J, I)
    if (I != J)
      for (int r = ty; r < 32; r += 8) {
        const int64_t il = bi + tx, jl = bj + r;
        if (il < n && jl < n) out[il + jl * n] = tu[tx][r];
      }
  } else
  for (int r = ty; r < 32; r += 8) {  // a(bi + tx, bj + r) vs a(bj + r, bi + tx)
    const int64_t il = bi + tx, jl = bj + r;
    if (il < n && jl < n) {
      const double v = tl[r][tx];
      const double m = (I != J) ? tu[tx][r] : tl[tx][r];
      if (!(v == m)) asym = 1;
    }
  }
  if (asym) atomicOr(flags + 0, 1);
  if (nonfin) atomicOr(flags + 1, 1);
  double bm = block_max(mx);
  if (threadIdx.x == 0 && threadIdx.y == 0) atomic_max_nonneg(amax, bm);
}

// Scaled column norms of B (P x ncols, col-major ld P) -> max (metrics.norm_1_2, core.py:122-142).
__global__ void sketch_norm_max_kernel(const double* __restrict__ B, int P, int64_t ncols, double* out) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double nv = 0.0;
  if (j < ncols) {
    const double* c = B + j * P;
    double scale = 0.0;
    for (int r = 0; r < P; ++r) scale = fmax(scale, fabs(c[r]));
    if (scale > 0.0) {
      double ss = 0.0;
      for (int r = 0; r < P; ++r) {
        double x = fabs(c[r]) / scale;
        ss = __fma_rn(x, x, ss);
      }
      nv = scale * sqrt(ss);
    }
  }
  double bm = block_max(nv);
  if (threadIdx.x == 0) atomic_max_nonneg(out, bm);
}

// Gather after a panel: applies the panel's permutation to the trailing-update operands.
//   phys[j]        = physical row of new logical k_end + j
//   Lneg[j][s]     = -L(panel col s) at that row   (K-contiguous, ld tpad, zero padded)
//   Wg[j][s]       =  W(panel col s) at that row
//   perm_next      = original index per new logical position
//   snap[x]        = perm at the panel start
//   lorig[o][k0+s] =  L(panel col s) of the still-active row with original index o (row-major by
//                     original index; finalize_rows_kernel reads a row once it is pivoted)
__global__ void gather_kernel(int64_t n, int k0, int k_end, int t, int tpad, int64_t rows_pad,
                              const int* __restrict__ phys_of_log, const double* __restrict__ Lbuf,
                              const double* __restrict__ W, const int* __restrict__ perm_cur,
                              int* __restrict__ perm_next, int* __restrict__ snap,
                              int* __restrict__ phys, double* __restrict__ Lneg, double* __restrict__ Wg,
                              double* __restrict__ L11, const PanelDesc* __restrict__ d, double* __restrict__ lorig) {
  if (d) {  // device-driven: panel geometry from the committed descriptor
    if (!d->ok) return;
    k0 = d->k0;
    k_end = d->k_end;
    t = d->t;
    const int64_t mp_ = n - k_end;
    rows_pad = ((mp_ + 127) / 128) * 128;
    snap += d->snap_off;
  }
  // compact strictly-lower panel block L11 in logical order, stored by columns for ysolve:
  // L11T[c * t + a] = L11[a][c]
  {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x * blockDim.y;
    const int64_t tflat = ((int64_t)blockIdx.x * blockDim.y + threadIdx.y) * blockDim.x + threadIdx.x;
    for (int64_t f = tflat; f < (int64_t)t * t; f += nthreads) {
      const int a = (int)(f / t), c = (int)(f - (int64_t)a * t);
      L11[(int64_t)c * t + a] = (c < a) ? Lbuf[phys_of_log[k0 + a] + (int64_t)(k0 + c) * n] : 0.0;
    }
  }
  const int64_t mp = n - k_end;
  const int64_t m0 = n - k0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.y;
  const int64_t jend = rows_pad > m0 ? rows_pad : m0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; j < jend; j += stride) {
    const bool live = j < mp;
    const int pj = live ? phys_of_log[k_end + j] : 0;
    double* lo = (live && lorig) ? lorig + (int64_t)perm_cur[pj] * n + k0 : nullptr;
    if (j < rows_pad) for (int s = threadIdx.x; s < tpad; s += blockDim.x) {
      double lv = 0.0, wv = 0.0;
      if (live && s < t) {
        const double lb = Lbuf[pj + (int64_t)(k0 + s) * n];
        lv = -lb;
        wv = W[pj + (int64_t)s * n];
        if (lo) lo[s] = lb;
      }
      Lneg[j * tpad + s] = lv;
      Wg[j * tpad + s] = wv;
    }
    if (threadIdx.x == 0) {
      if (live) {
        phys[j] = pj;
        perm_next[k_end + j] = perm_cur[pj];
      }
      if (j < m0) snap[j] = perm_cur[k0 + j];
    }
  }
}

// Y = B1 * L11^{-T}  (P x t), with B1[:, a] = Bin[:, piv[a]] and L11 the panel's
// unit-lower block in logical order.  Algebraically equal to the reference's
// B1 @ solve_triangular(L11, L21^T, trans='T') (factor.py:554-561).  One warp per sketch row:
// column-oriented forward substitution (y[c] -= L11[c][a] y[a] for c > a), the row held in
// registers (lane owns entries lane + 32u), L11 by columns in shared memory.
constexpr int kYsolveWarps = 8;
__global__ void ysolve_kernel(int64_t n, int P, int k0, int t, int tpad, const int* __restrict__ phys_of_log,
                              const double* __restrict__ Bin, const double* __restrict__ L11T,
                              double* __restrict__ Y, const PanelDesc* __restrict__ d) {
  if (d) {
    if (!d->ok || d->t <= 0 || d->k_end >= n) return;
    k0 = d->k0;
    t = d->t;
  }
  extern __shared__ double sm[];  // [t][t]: row a = column a of L11
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {  // stage L11 (t*t doubles, L2-resident): 16-byte loads, 8 in flight per thread
    const int tt = t * t, t2 = tt >> 1;
    const double2* src2 = reinterpret_cast<const double2*>(L11T);
    double2* dst2 = reinterpret_cast<double2*>(sm);
    const int nth = blockDim.x;
    int f = tid;
    for (; f + 7 * nth < t2; f += 8 * nth) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(src2 + f + u * nth);
#pragma unroll
      for (int u = 0; u < 8; ++u) dst2[f + u * nth] = v[u];
    }
    for (; f < t2; f += nth) dst2[f] = __ldcg(src2 + f);
    if ((tt & 1) && tid == 0) sm[tt - 1] = L11T[tt - 1];
  }
  const int r = blockIdx.x * kYsolveWarps + warp;
  constexpr int kU = 6;  // t <= tpad <= 192 (L11 in smem limits t to ~170 anyway)
  double y[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int a = lane + 32 * u;
    y[u] = (r < P && a < t) ? Bin[r + (int64_t)phys_of_log[k0 + a] * P] : 0.0;
  }
  __syncthreads();
  if (r >= P) return;
  for (int a = 0; a < t; ++a) {
    const int ua = a >> 5;
    double src = 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (u == ua) src = y[u];
    const double ya = __shfl_sync(0xffffffffu, src, a & 31);
    const double* col = sm + (size_t)a * t;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = lane + 32 * u;
      if (c > a && c < t) y[u] = __fma_rn(-col[c], ya, y[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int a = lane + 32 * u;
    if (a < tpad) Y[(int64_t)r * tpad + a] = (a < t) ? y[u] : 0.0;
  }
}

// pos_of_orig[snap[x]] = x for one panel's snapshot.
__global__ void invert_snapshot_kernel(int64_t m0, const int* __restrict__ snap, int* __restrict__ pos_of_orig) {
  int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < m0) pos_of_orig[snap[x]] = static_cast<int>(x);
}

// L (row-major, final order) for columns [k0, k_end) of one panel:
// L[i, c] = Lbuf[k0 + pos_p(perm[i]), c] for i > c (factor.py:339-340 applied lazily).
__global__ void assemble_panel_kernel(int64_t n, int k0, int k_end, const int64_t* __restrict__ perm,
                                      const int* __restrict__ pos_of_orig, const double* __restrict__ Lbuf,
                                      double* __restrict__ L, double* maxmult) {
  const int w = k_end - k0;
  double mx = 0.0;
  for (int64_t i = (int64_t)k0 + 1 + blockIdx.x; i < n; i += gridDim.x) {
    const int64_t src = k0 + pos_of_orig[perm[i]];
    const int cmax = static_cast<int>(i < (int64_t)k_end ? i : (int64_t)k_end);
    for (int c = k0 + threadIdx.x; c < cmax; c += blockDim.x) {
      double v = Lbuf[src + (int64_t)c * n];
      L[i * n + c] = v;
      mx = fmax(mx, fabs(v));
    }
  }
  (void)w;
  double bm = block_max(mx);
  if (threadIdx.x == 0) atomic_max_nonneg(maxmult, bm);
}

// Final rows [ra, rb) of L (row-major, final order), written once each row's position is decided:
// L[i, c] = lorig[perm[i]][c] for c < min(i, kp) (the columns of earlier panels, scattered by their
// gathers while the row was active) and, with L11T (the panel [kp, rb) that pivoted these rows),
// the panel's own strictly-lower block for c in [kp, i).  Device-driven (d): the committed panel.
// Same values as the reference's L (factor.py:339-340, 514-538); max |L| for the statistics.
__global__ void finalize_rows_kernel(int64_t n, int64_t ra, int64_t rb, int64_t kp, int t, const int64_t* __restrict__ perm,
                                     const double* __restrict__ lorig, const double* __restrict__ L11T,
                                     double* __restrict__ L, double* maxmult, const PanelDesc* __restrict__ d) {
  if (d) {
    if (!d->ok) return;
    ra = kp = d->k0;
    rb = d->k_end;
    t = d->t;
  }
  double mx = 0.0;
  const int64_t cstep = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = ra + blockIdx.y; i < rb; i += gridDim.y) {
    const double* src = lorig + perm[i] * n;
    double* dst = L + i * n;
    const int64_t cl = i < kp ? i : kp;
    const int64_t ce = L11T ? i : cl;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ce; c += cstep) {
      const double v = (c < cl) ? __ldcs(src + c) : L11T[(c - kp) * t + (i - kp)];
      dst[c] = v;
      mx = fmax(mx, fabs(v));
    }
  }
  const double bm = block_max(mx);
  if (threadIdx.x == 0) atomic_max_nonneg(maxmult, bm);
}

__global__ void unit_diag_kernel(int64_t n, double* L) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) L[i * n + i] = 1.0;
}

__global__ void dmax_kernel(int64_t n, const double* __restrict__ dd, const double* __restrict__ doff, double* out) {
  double mx = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mx = fmax(mx, fmax(fabs(dd[i]), fabs(doff[i])));
  double bm = block_max(mx);
  if (threadIdx.x == 0) atomic_max_nonneg(out, bm);
}

// Deficient tail (factor.py:381-385): zero 1x1 blocks, pattern 3, order as it stands.
__global__ void deficient_fill_kernel(int64_t n, int64_t k0, const int* __restrict__ perm_cur, int64_t* perm_out,
                                      double* dd, double* doff, int8_t* pattern) {
  int64_t x = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < n) {
    dd[x] = 0.0;
    doff[x] = 0.0;
    pattern[x] = 3;
    perm_out[x] = perm_cur[x];
  }
}

// Copy the lower triangle of the trailing block [k:, k:] onto its upper triangle.
__global__ void mirror_lower_kernel(int64_t n, int64_t k, double* A) {
  __shared__ double tile[32][33];
  const int64_t bi = k + (int64_t)blockIdx.y * 32, bj = k + (int64_t)blockIdx.x * 32;
  if (blockIdx.x > blockIdx.y) return;  // only tiles with bi >= bj (lower) are sources
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += 8) {
    int64_t i = bi + tx, j = bj + r;
    tile[r][tx] = (i < n && j < n) ? A[i + j * n] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    int64_t i = bj + tx, j = bi + r;  // destination (i, j) = upper element, source (j, i)
    if (i < n && j < n && i < j) A[i + j * n] = tile[tx][r];
  }
}

__global__ void tstamp_init_kernel(unsigned long long* ts, int64_t count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) ts[2 * i] = ~0ULL;  // start slots (atomicMin); end slots stay 0 (atomicMax)
}

__global__ void iota_kernel(int64_t n, int* p) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = static_cast<int>(i);
}

}  // namespace

// ------------------------------------------------------------------ launchers
cudaError_t launch_validate_copy(const double* a, int64_t lda, int64_t n, double* out, int* flags, double* amax,
                                 cudaStream_t st, int half) {
  const long long nb = (n + 31) / 32;
  dim3 block(32, 8);
  validate_copy_kernel<<<(unsigned)(nb * (nb + 1) / 2), block, 0, st>>>(a, lda, n, out, flags, amax, half);
  return cudaGetLastError();
}

cudaError_t launch_tstamp_init(unsigned long long* ts, int64_t count, cudaStream_t st) {
  tstamp_init_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(ts, count);
  return cudaGetLastError();
}

cudaError_t launch_sketch_norm_max(const double* B, int P, int64_t ncols, double* out, cudaStream_t st) {
  sketch_norm_max_kernel<<<(unsigned)((ncols + 255) / 256), 256, 0, st>>>(B, P, ncols, out);
  return cudaGetLastError();
}

cudaError_t launch_gather(int64_t n, int k0, int k_end, int t, int tpad, int64_t rows_pad, const int* phys_of_log,
                          const double* Lbuf, const double* W, const int* perm_cur, int* perm_next, int* snap,
                          int* phys, double* Lneg, double* Wg, double* L11, cudaStream_t st, const PanelDesc* d,
                          double* lorig) {
  dim3 block(32, 8);
  int64_t rows = rows_pad > (n - k0) ? rows_pad : (n - k0);
  unsigned grid = (unsigned)std::min<int64_t>((rows + 7) / 8, 148 * 16);
  gather_kernel<<<grid, block, 0, st>>>(n, k0, k_end, t, tpad, rows_pad, phys_of_log, Lbuf, W, perm_cur,
                                        perm_next, snap, phys, Lneg, Wg, L11, d, lorig);
  return cudaGetLastError();
}

cudaError_t launch_finalize_rows(int64_t n, int64_t ra, int64_t rb, int64_t kp, int t, const int64_t* perm,
                                 const double* lorig, const double* L11T, double* L, double* maxmult,
                                 int max_rows, cudaStream_t st, const PanelDesc* d) {
  if (!d && rb <= ra) return cudaSuccess;
  const int64_t rows = d ? max_rows : rb - ra;
  dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 16), (unsigned)std::min<int64_t>(std::max<int64_t>(rows, 1), 1024));
  finalize_rows_kernel<<<grid, 256, 0, st>>>(n, ra, rb, kp, t, perm, lorig, L11T, L, maxmult, d);
  return cudaGetLastError();
}

cudaError_t launch_ysolve(int64_t n, int P, int k0, int t, int tpad, const int* phys_of_log, const double* Bin,
                          const double* L11, double* Y, cudaStream_t st, const PanelDesc* d) {
  if (tpad > 192) return cudaErrorInvalidValue;  // register-resident rows: 6 entries per lane
  size_t smem = sizeof(double) * (size_t)t * t;  // t: an upper bound when d != nullptr
  static thread_local size_t smem_set = 0;  // raise the limit only when it grows (one driver call)
  static thread_local int smem_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != smem_dev) {
    smem_set = 0;
    smem_dev = dev;
  }
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(ysolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  ysolve_kernel<<<(unsigned)((P + kYsolveWarps - 1) / kYsolveWarps), 32 * kYsolveWarps, smem, st>>>(
      n, P, k0, t, tpad, phys_of_log, Bin, L11, Y, d);
  return cudaGetLastError();
}

cudaError_t launch_assemble_panel(int64_t n, int k0, int k_end, const int* snap, int* pos_of_orig,
                                  const int64_t* perm, const double* Lbuf, double* L, double* maxmult,
                                  cudaStream_t st) {
  int64_t m0 = n - k0;
  invert_snapshot_kernel<<<(unsigned)((m0 + 255) / 256), 256, 0, st>>>(m0, snap, pos_of_orig);
  int64_t rows = n - k0 - 1;
  if (rows > 0) {
    unsigned grid = (unsigned)std::min<int64_t>(rows, 148 * 8);
    int w = k_end - k0;
    int threads = w >= 128 ? 128 : ((w + 31) / 32) * 32;
    assemble_panel_kernel<<<grid, threads, 0, st>>>(n, k0, k_end, perm, pos_of_orig, Lbuf, L, maxmult);
  }
  return cudaGetLastError();
}

cudaError_t launch_unit_diag(int64_t n, double* L, cudaStream_t st) {
  unit_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, L);
  return cudaGetLastError();
}

cudaError_t launch_dmax(int64_t n, const double* dd, const double* doff, double* out, cudaStream_t st) {
  unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4);
  dmax_kernel<<<grid, 256, 0, st>>>(n, dd, doff, out);
  return cudaGetLastError();
}

cudaError_t launch_deficient_fill(int64_t n, int64_t k0, const int* perm_cur, int64_t* perm_out, double* dd,
                                  double* doff, int8_t* pattern, cudaStream_t st) {
  if (n - k0 <= 0) return cudaSuccess;
  deficient_fill_kernel<<<(unsigned)((n - k0 + 255) / 256), 256, 0, st>>>(n, k0, perm_cur, perm_out, dd, doff,
                                                                          pattern);
  return cudaGetLastError();
}

cudaError_t launch_mirror_lower(int64_t n, int64_t k, double* A, cudaStream_t st) {
  int64_t m = n - k;
  unsigned nb = (unsigned)((m + 31) / 32);
  dim3 grid(nb, nb), block(32, 8);
  mirror_lower_kernel<<<grid, block, 0, st>>>(n, k, A);
  return cudaGetLastError();
}

cudaError_t launch_iota(int64_t n, int* p, cudaStream_t st) {
  iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, p);
  return cudaGetLastError();
}

}  // namespace rcp
