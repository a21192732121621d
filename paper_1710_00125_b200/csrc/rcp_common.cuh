// Shared device helpers for the RCP block-LDL^T kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define RCP_HD __host__ __device__ __forceinline__
#define RCP_D __device__ __forceinline__

namespace rcp {

constexpr int kMaxSMs = 160;

// ---------------------------------------------------------------- memory ordering
// Loads of data written by other CTAs during the same launch go to L2 (.cg) so a
// stale L1 line can never be observed; flags use acquire/release at gpu scope.
RCP_D double ldcg(const double* p) { return __ldcg(p); }
RCP_D int ldcg(const int* p) { return __ldcg(p); }
RCP_D long long ld_acquire(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
RCP_D void st_release(long long* p, long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------- symmetric access
// Trailing blocks are column-major (ld = n).  With RCP_FULL_STORAGE both triangles are kept
// (a pivot column is one contiguous read; the Schur update also writes the mirror); otherwise
// only the lower triangle is valid and (i, j), i < j, is read from (j, i).
#ifndef RCP_FULL_STORAGE
#define RCP_FULL_STORAGE 1
#endif
RCP_HD int64_t sym_index(int64_t ld, int64_t i, int64_t j) {
#if RCP_FULL_STORAGE
  return i + j * ld;
#else
  return (i >= j) ? i + j * ld : j + i * ld;
#endif
}
RCP_D double sym_at(const double* a, int64_t ld, int64_t i, int64_t j) { return a[sym_index(ld, i, j)]; }

// ---------------------------------------------------------------- pivot-column dot
// Dot product of row i of the panel L (Lrow(s)) with the pivot's W row w[s], s < t,
// as 4 interleaved chains combined ((c0+c1)+(c2+c3)).  The GEMV, the redundant
// single-row recomputation and the trailing-diagonal updates all use this exact
// routine so every CTA derives bitwise-identical column entries.
template <class F>
RCP_D double chain_dot4(F lrow, const double* w, int t) {
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  int s = 0;
  for (; s + 4 <= t; s += 4) {
    c0 = __fma_rn(lrow(s), w[s], c0);
    c1 = __fma_rn(lrow(s + 1), w[s + 1], c1);
    c2 = __fma_rn(lrow(s + 2), w[s + 2], c2);
    c3 = __fma_rn(lrow(s + 3), w[s + 3], c3);
  }
  if (s < t) c0 = __fma_rn(lrow(s), w[s], c0);
  if (s + 1 < t) c1 = __fma_rn(lrow(s + 1), w[s + 1], c1);
  if (s + 2 < t) c2 = __fma_rn(lrow(s + 2), w[s + 2], c2);
  return __dadd_rn(__dadd_rn(c0, c1), __dadd_rn(c2, c3));
}

// Same chain arithmetic for a row of the panel L held partly in shared memory (columns
// s < ls, at lsm[s * ldsm]) and partly in global memory (s >= ls, at lg[s * ldg]).
// Chain q accumulates the terms s = q (mod 4) in increasing s, exactly like chain_dot4.
RCP_D double row_dot4(const double* __restrict__ lsm, int ldsm, int ls, const double* __restrict__ lg, int64_t ldg,
                      const double* __restrict__ w, int t) {
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  const int ts = t < ls ? t : ls;
  int s = 0;
  const double* lp = lsm;
  const int st4 = 4 * ldsm;
#pragma unroll 2
  for (; s + 4 <= ts; s += 4, lp += st4) {
    c0 = __fma_rn(lp[0], w[s], c0);
    c1 = __fma_rn(lp[ldsm], w[s + 1], c1);
    c2 = __fma_rn(lp[2 * ldsm], w[s + 2], c2);
    c3 = __fma_rn(lp[3 * ldsm], w[s + 3], c3);
  }
  for (; s < t; ++s) {
    const double x = (s < ls) ? lsm[s * ldsm] : __ldcg(lg + (int64_t)s * ldg);
    switch (s & 3) {
      case 0: c0 = __fma_rn(x, w[s], c0); break;
      case 1: c1 = __fma_rn(x, w[s], c1); break;
      case 2: c2 = __fma_rn(x, w[s], c2); break;
      default: c3 = __fma_rn(x, w[s], c3); break;
    }
  }
  return __dadd_rn(__dadd_rn(c0, c1), __dadd_rn(c2, c3));
}

// ---------------------------------------------------------------- device timestamps
// Kernel durations are stamped on the device (%globaltimer, ns): the host then reads one array per
// factorization instead of issuing a driver call per launch (which can queue behind NVML clients).
RCP_D unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
RCP_D void stamp_start(unsigned long long* s) {
  if (s && threadIdx.x == 0 && blockIdx.x == 0) atomicMin(s, gtimer());
}
RCP_D void stamp_end(unsigned long long* s) {
  if (s && threadIdx.x == 0) atomicMax(s, gtimer());
}

// ---------------------------------------------------------------- argmax comparators
// numpy argmax semantics: NaN wins (first NaN), otherwise largest value, ties to the
// lowest index.
RCP_D bool better(double va, long long ia, double vb, long long ib) {
  bool na = va != va, nb = vb != vb;
  if (na != nb) return na;
  if (!na && va != vb) return va > vb;
  return ia < ib;
}

// ---------------------------------------------------------------- DMMA (FP64 tensor core)
// mma.sync m8n8k4 f64: a = A[g][q], b = B[q][g], c/d = C[g][2q + {0,1}], g = lane>>2, q = lane&3.
RCP_D void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

RCP_D void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
RCP_D void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
// Same with an L2 cache-policy hint (e.g. evict_first for streamed data).
RCP_D void cp_async8_hint(void* smem, const void* gmem, bool pred, unsigned long long policy) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;\n" ::"r"(s), "l"(gmem), "r"(n),
               "l"(policy));
}
RCP_D unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
RCP_D void st_stream(double* p, double v) { __stcs(p, v); }
RCP_D void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RCP_D void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Atomic max for non-negative doubles (bit patterns order like the values).
RCP_D void atomic_max_nonneg(double* addr, double v) {
  if (!(v >= 0.0)) {  // NaN: record as +inf so it is visible to the host
    v = __longlong_as_double(0x7ff0000000000000LL);
  }
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace rcp
