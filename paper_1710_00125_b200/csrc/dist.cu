// Multi-GPU trailing update over NVLink peer memory (see dist.cuh for the protocol).
#include <algorithm>

#include "dist.cuh"
#include "misc.cuh"
#include "rcp_common.cuh"

namespace rcp {

namespace {

constexpr unsigned long long kWatchdogNs = 120ull * 1000000000ull;  // a stuck peer -> error, not a hang

RCP_D unsigned long long ld_acq_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
RCP_D int ld_acq_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
RCP_D void st_rel_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
RCP_D void st_rel_sys(int* p, int v) { asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
RCP_D unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void dist_signal_kernel(DistShared* sh, unsigned long long seq, int curA, int desc_idx) {
  sh->info_curA = curA;
  sh->info_desc = desc_idx;
  __threadfence_system();  // the panel's descriptor, operands and info before the counter
  st_rel_sys(&sh->ready, seq);
}

__global__ void dist_wait_done_kernel(DistShared* sh, int world, unsigned long long seq) {
  const int r = threadIdx.x + 1;
  if (r < world) {
    const unsigned long long t0 = now_ns();
    while (ld_acq_sys(&sh->done[r]) < seq) {
      if (ld_acq_sys(&sh->error)) break;
      if (now_ns() - t0 > kWatchdogNs) {
        st_rel_sys(&sh->error, 1);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

__global__ void dist_finish_kernel(DistShared* sh) {
  __threadfence_system();
  st_rel_sys(&sh->finished, 1);
}

__global__ void worker_wait_kernel(DistShared* sh, unsigned long long seq, double* A0, double* A1,
                                   const PanelDesc* desc, SchurDyn* dyn) {
  const unsigned long long t0 = now_ns();
  int go = 0;
  for (;;) {
    if (ld_acq_sys(&sh->ready) >= seq) {
      go = 1;
      break;
    }
    if (ld_acq_sys(&sh->finished) || ld_acq_sys(&sh->error)) break;
    if (now_ns() - t0 > kWatchdogNs) {
      st_rel_sys(&sh->error, 1);
      break;
    }
    __nanosleep(512);
  }
  SchurDyn d{};
  d.go = go;
  if (go) {
    const int ca = *reinterpret_cast<volatile int*>(&sh->info_curA);
    const int di = *reinterpret_cast<volatile int*>(&sh->info_desc);
    d.ain = ca ? A1 : A0;
    d.aout = ca ? A0 : A1;
    d.d = desc + di;
  }
  *dyn = d;
}

// Copy the panel's update operands (rank 0's gather output) into local memory: the Schur
// kernel re-reads them per tile, which must not cross NVLink.
__global__ void worker_copy_kernel(const SchurDyn* __restrict__ dyn, int64_t n, int tpad,
                                   const double* __restrict__ Lneg0, const double* __restrict__ Wg0,
                                   const int* __restrict__ phys0, double* __restrict__ Lneg, double* __restrict__ Wg,
                                   int* __restrict__ phys) {
  const SchurDyn d = *dyn;
  if (!d.go) return;
  const volatile PanelDesc* vd = d.d;
  const int ok = vd->ok, t = vd->t, k_end = vd->k_end;
  if (!ok || t <= 0 || k_end >= n) return;
  const int64_t mp = n - k_end;
  const int64_t rows = ((mp + 127) / 128) * 128;
  const int64_t tot2 = rows * tpad / 2;  // tpad is a multiple of 16
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double2* l2 = reinterpret_cast<const double2*>(Lneg0);
  const double2* w2 = reinterpret_cast<const double2*>(Wg0);
  double2* lo = reinterpret_cast<double2*>(Lneg);
  double2* wo = reinterpret_cast<double2*>(Wg);
  for (int64_t f = t0; f < tot2; f += stride) {
    lo[f] = l2[f];
    wo[f] = w2[f];
  }
  for (int64_t j = t0; j < mp; j += stride) phys[j] = phys0[j];
}

__global__ void worker_done_kernel(DistShared* sh, int rank, unsigned long long seq) {
  __threadfence_system();  // this panel's peer stores into rank 0's matrix before the counter
  st_rel_sys(&sh->done[rank], seq);
}

}  // namespace

cudaError_t launch_dist_signal(DistShared* sh, unsigned long long seq, int curA, int desc_idx, cudaStream_t st) {
  dist_signal_kernel<<<1, 1, 0, st>>>(sh, seq, curA, desc_idx);
  return cudaGetLastError();
}

cudaError_t launch_dist_wait_done(DistShared* sh, int world, unsigned long long seq, cudaStream_t st) {
  dist_wait_done_kernel<<<1, kMaxWorld, 0, st>>>(sh, world, seq);
  return cudaGetLastError();
}

cudaError_t launch_dist_finish(DistShared* sh, cudaStream_t st) {
  dist_finish_kernel<<<1, 1, 0, st>>>(sh);
  return cudaGetLastError();
}

cudaError_t launch_worker_panel(DistShared* sh, int rank, int world, unsigned long long seq, double* A0, double* A1,
                                const PanelDesc* desc, const double* Lneg0, const double* Wg0, const int* phys0,
                                int64_t n, int tpad, const WorkerBufs& wb, cudaStream_t st) {
  worker_wait_kernel<<<1, 1, 0, st>>>(sh, seq, A0, A1, desc, wb.dyn);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  worker_copy_kernel<<<148 * 4, 256, 0, st>>>(wb.dyn, n, tpad, Lneg0, Wg0, phys0, wb.Lneg, wb.Wg, wb.phys);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = launch_schur_update_dyn(n, wb.Lneg, wb.Wg, tpad, wb.phys, wb.dyn, rank, world, st);
  if (e != cudaSuccess) return e;
  worker_done_kernel<<<1, 1, 0, st>>>(sh, rank, seq);
  return cudaGetLastError();
}

}  // namespace rcp
