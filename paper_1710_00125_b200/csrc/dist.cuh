// Multi-GPU trailing update: rank 0 owns the matrix and runs the panels; every rank (rank 0
// included) updates the tiles x = rank (mod world) of each panel's trailing Schur update,
// reading the C-in tiles from and writing the results into rank 0's buffers through NVLink
// peer memory (CUDA IPC mapping of rank 0's workspace).  Synchronisation is by sequence
// counters in rank 0's memory, release/acquire at system scope:
//   rank 0:  panel p -> commit -> gather -> signal(s) -> Schur part 0 -> wait(done[r] >= s)
//   rank r:  wait(ready >= s) -> copy operands -> Schur part r -> done[r] = s
// The same kernels run in a single-process emulation (world "virtual" ranks on one device,
// enqueued in dependency order on one stream) used by the parity tests.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "panel.cuh"

namespace rcp {

constexpr int kMaxWorld = 16;

struct DistShared {             // lives in rank 0's workspace
  unsigned long long ready;     // last signalled panel (sequence number, 1-based)
  int info_curA;                // A_in buffer index of that panel
  int info_desc;                // its descriptor index (pidx & 1)
  int finished;                 // rank 0 is done: workers exit
  int error;                    // watchdog fired somewhere
  int pad[2];
  unsigned long long done[kMaxWorld];  // per rank: last completed sequence number
};

// Arguments a worker's Schur kernel resolves on the device (they depend on rank 0's state).
struct SchurDyn {
  const double* ain;
  double* aout;
  const PanelDesc* d;
  int go;  // 0: nothing to do (rank 0 finished)
  int pad;
};

// Per-worker device scratch: operand copies and the resolved arguments.
struct WorkerBufs {
  double* Lneg;
  double* Wg;
  int* phys;
  SchurDyn* dyn;
};

cudaError_t launch_dist_signal(DistShared* sh, unsigned long long seq, int curA, int desc_idx, cudaStream_t st);
cudaError_t launch_dist_wait_done(DistShared* sh, int world, unsigned long long seq, cudaStream_t st);
cudaError_t launch_dist_finish(DistShared* sh, cudaStream_t st);
// Worker side (sh, A0/A1, desc, Lneg/Wg/phys are rank 0's buffers as mapped in this process).
cudaError_t launch_worker_panel(DistShared* sh, int rank, int world, unsigned long long seq, double* A0,
                                double* A1, const PanelDesc* desc, const double* Lneg0, const double* Wg0,
                                const int* phys0, int64_t n, int tpad, const WorkerBufs& wb, cudaStream_t st);

}  // namespace rcp
