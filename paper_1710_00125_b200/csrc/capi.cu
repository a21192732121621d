// C ABI + host-side driver of the RCP factorization (include/rcp_b200.h).
//
// The driver is the native counterpart of the reference engine loop
// (_Engine.run / _run_panel, factor.py:508-568): per panel it launches the
// cooperative panel kernel, reads back the panel outcome (k_end, guard status,
// numerical error) with one small D2H copy, then launches the gather, the
// trailing Schur update and the sketch correction.  All matrix data stays on the
// device; the host never touches a matrix element.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/rcp_b200.h"
#include "misc.cuh"
#include "panel.cuh"
#include "rcp_common.cuh"
#include "solve.cuh"
#include "layout.cuh"
#include "dist.cuh"

using namespace rcp;

namespace {

struct Scal {  // scalar results block (device)
  double amax, beta, dmax, maxmult;
  int vflags[2];
};

struct HostCache {
  int dev = -1;
  bool ok = false;
  PanelState* hstate = nullptr;
  PanelState* hsnap = nullptr;  // 2 slots
  Scal* hscal = nullptr;
  PanelDesc* hdesc = nullptr;   // 2 slots x 2 descriptors
  cudaEvent_t bev[2] = {nullptr, nullptr};
  cudaStream_t cst = nullptr;  // copy stream of the host L sink (created on first use)
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  void reset() { used = 0; }
  cudaEvent_t event() {
    if (used == pool.size()) {
      cudaEvent_t e = nullptr;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void release() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
    pool.clear();
    used = 0;
    for (int i = 0; i < 2; ++i)
      if (bev[i]) cudaEventDestroy(bev[i]);
    if (cst) cudaStreamDestroy(cst);
    cst = nullptr;
    if (hstate) cudaFreeHost(hstate);
    if (hsnap) cudaFreeHost(hsnap);
    if (hscal) cudaFreeHost(hscal);
    if (hdesc) cudaFreeHost(hdesc);
    hstate = hsnap = nullptr;
    hscal = nullptr;
    hdesc = nullptr;
    bev[0] = bev[1] = nullptr;
    ok = false;
  }
  ~HostCache() {}  // process teardown: leave the driver to reclaim (the context may be gone)
};

HostCache& host_cache(int dev) {
  thread_local HostCache hc;
  if (hc.ok && hc.dev == dev) return hc;
  if (hc.ok) hc.release();
  hc.dev = dev;
  hc.ok = cudaMallocHost(&hc.hstate, sizeof(PanelState)) == cudaSuccess &&
          cudaMallocHost(&hc.hsnap, 2 * sizeof(PanelState)) == cudaSuccess &&
          cudaMallocHost(&hc.hscal, sizeof(Scal)) == cudaSuccess &&
          cudaMallocHost(&hc.hdesc, 4 * sizeof(PanelDesc)) == cudaSuccess &&
          cudaEventCreateWithFlags(&hc.bev[0], cudaEventDisableTiming) == cudaSuccess &&
          cudaEventCreateWithFlags(&hc.bev[1], cudaEventDisableTiming) == cudaSuccess;
  return hc;
}

WorkerBufs carve_worker(unsigned char* b, int64_t n, const Layout& L) {
  WorkerBufs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* p = b + off;
    off += align_up(bytes);
    return p;
  };
  w.Lneg = reinterpret_cast<double*>(take((size_t)L.rows_pad * L.tpad * 8));
  w.Wg = reinterpret_cast<double*>(take((size_t)L.rows_pad * L.tpad * 8));
  w.phys = reinterpret_cast<int*>(take((size_t)n * 4));
  w.dyn = reinterpret_cast<SchurDyn*>(take(sizeof(SchurDyn)));
  return w;
}

#ifndef RCP_FUSED_SKETCH
#define RCP_FUSED_SKETCH 1  // single GPU: the sketch correction runs as extra Schur tiles
#endif

int validate_cfg(const rcp_config* c, int64_t n) {
  if (!c || n < 1) return RCP_ERR_INVALID_ARG;
  if (c->p < 1 || c->b < 1 || c->robust_r < 0) return RCP_ERR_INVALID_ARG;
  if (c->strategy < RCP_STRATEGY_RCP || c->strategy > RCP_STRATEGY_BBK) return RCP_ERR_INVALID_ARG;
  if (!(c->q == 1 || c->q == c->b)) return RCP_ERR_INVALID_ARG;
  if (c->p < c->q) return RCP_ERR_INVALID_ARG;
  if (n > (int64_t)INT_MAX / 2) return RCP_ERR_INVALID_ARG;
  return RCP_OK;
}


#define RCP_CHECK(expr)                                                                           \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess) {                                                                      \
      if (stats) snprintf(stats->message, sizeof(stats->message), "%s at %s:%d", cudaGetErrorString(e_), \
                          __FILE__, __LINE__);                                                    \
      return RCP_ERR_CUDA;                                                                        \
    }                                                                                             \
  } while (0)

#define RCP_LAUNCH(expr) \
  do {                   \
    RCP_CHECK(expr);     \
    ++launches;          \
  } while (0)

struct PanelRecord {
  int k0, k_end;
  int64_t snap_off;
};

struct EventPair {
  cudaEvent_t a, b;
};

}  // namespace

extern "C" {

const char* rcp_version(void) { return "rcp_b200 0.1.0 sm_100a"; }

size_t rcp_workspace_bytes(int64_t n, const rcp_config* cfg) {
  if (validate_cfg(cfg, n) != RCP_OK) return 0;
  return make_layout(n, *cfg).total;
}

size_t rcp_worker_workspace_bytes(int64_t n, const rcp_config* cfg) {
  if (validate_cfg(cfg, n) != RCP_OK) return 0;
  const Layout L = make_layout(n, *cfg);
  return align_up((size_t)L.rows_pad * L.tpad * 8) * 2 + align_up((size_t)n * 4) + align_up(sizeof(SchurDyn)) + kAlign;
}

// Host sink for L (pinned, dense row-major n x n): 256-row block rows of L's lower trapezoid go
// over PCIe on a copy stream as soon as their rows are final, overlapping the rest of the
// factorization; host threads zero the strictly-upper part the copies do not cover meanwhile.
// The destructor joins the threads and drains the copy stream on every exit path.
struct HostLSink {
  static constexpr int64_t kBlk = 256;
  double* h = nullptr;
  const double* d = nullptr;
  int64_t n = 0, sent = 0;
  cudaStream_t cs = nullptr;
  std::vector<std::thread> th;
  bool failed = false;
  void start(double* host, const double* dev, int64_t n_, cudaStream_t copy_stream) {
    h = host;
    d = dev;
    n = n_;
    cs = copy_stream;
    const int64_t nb = (n + kBlk - 1) / kBlk;
    unsigned hw = std::thread::hardware_concurrency();
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)(hw ? hw : 1) / 2, 8, nb}));
    for (int tt = 0; tt < nt; ++tt)
      th.emplace_back([this, tt, nt, nb]() {
        for (int64_t b = tt; b < nb; b += nt) {
          const int64_t i0 = b * kBlk, i1 = std::min(n, i0 + kBlk);
          if (i1 < n)
            for (int64_t i = i0; i < i1; ++i) memset(h + i * n + i1, 0, (size_t)(n - i1) * sizeof(double));
        }
      });
  }
  // copy the complete block rows below row `upto` (all rows when upto == n) once `ready` is done
  void flush(int64_t upto, cudaEvent_t ready) {
    if (!h || failed) return;
    const int64_t lim = (upto >= n) ? n : (upto / kBlk) * kBlk;
    if (lim <= sent) return;
    if (cudaStreamWaitEvent(cs, ready, 0) != cudaSuccess) failed = true;
    const size_t pitch = (size_t)n * sizeof(double);
    while (!failed && sent < lim) {
      const int64_t i0 = sent, i1 = std::min(n, i0 + kBlk);
      if (cudaMemcpy2DAsync(h + i0 * n, pitch, d + i0 * n, pitch, (size_t)i1 * sizeof(double), (size_t)(i1 - i0),
                            cudaMemcpyDeviceToHost, cs) != cudaSuccess)
        failed = true;
      sent = i1;
    }
  }
  bool finish() {  // true when every block row arrived
    for (auto& x : th) x.join();
    th.clear();
    if (!h) return true;
    const bool ok = cudaStreamSynchronize(cs) == cudaSuccess && !failed && sent >= n;
    h = nullptr;
    return ok;
  }
  ~HostLSink() { finish(); }
};

int rcp_factor(const rcp_config* cfg, int64_t n, const double* a, int64_t lda, const double* omega_dev,
               rcp_draw_fn draw, void* draw_ctx, void* workspace, size_t workspace_bytes, int64_t* perm,
               double* Lout, double* d_diag, double* d_off, int8_t* pattern, int8_t* trace_kind, int32_t* trace_r,
               rcp_stats* stats, void* cuda_stream) {
  return rcp_factor_dist(cfg, n, a, lda, omega_dev, draw, draw_ctx, workspace, workspace_bytes, perm, Lout, d_diag,
                         d_off, pattern, trace_kind, trace_r, stats, 1, 0, nullptr, 0, cuda_stream);
}

static int factor_core(const rcp_config* cfg, int64_t n, const double* a, int64_t lda, const double* omega_dev,
                       rcp_draw_fn draw, void* draw_ctx, void* workspace, size_t workspace_bytes, int64_t* perm,
                       double* Lout, double* d_diag, double* d_off, int8_t* pattern, int8_t* trace_kind,
                       int32_t* trace_r, rcp_stats* stats, int world, int emulate, void* worker_ws,
                       size_t worker_ws_bytes, void* cuda_stream, double* L_host, const double* a_host,
                       rcp_diag* diag = nullptr);

int rcp_factor_dist(const rcp_config* cfg, int64_t n, const double* a, int64_t lda, const double* omega_dev,
                    rcp_draw_fn draw, void* draw_ctx, void* workspace, size_t workspace_bytes, int64_t* perm,
                    double* Lout, double* d_diag, double* d_off, int8_t* pattern, int8_t* trace_kind,
                    int32_t* trace_r, rcp_stats* stats, int world, int emulate, void* worker_ws,
                    size_t worker_ws_bytes, void* cuda_stream) {
  return factor_core(cfg, n, a, lda, omega_dev, draw, draw_ctx, workspace, workspace_bytes, perm, Lout, d_diag, d_off,
                     pattern, trace_kind, trace_r, stats, world, emulate, worker_ws, worker_ws_bytes, cuda_stream,
                     nullptr, nullptr);
}

int rcp_factor_host_l(const rcp_config* cfg, int64_t n, const double* a, int64_t lda, const double* omega_dev,
                      rcp_draw_fn draw, void* draw_ctx, void* workspace, size_t workspace_bytes, int64_t* perm,
                      double* Lout, double* d_diag, double* d_off, int8_t* pattern, int8_t* trace_kind,
                      int32_t* trace_r, rcp_stats* stats, double* L_host, void* cuda_stream) {
  if (!L_host) return RCP_ERR_INVALID_ARG;
  return factor_core(cfg, n, a, lda, omega_dev, draw, draw_ctx, workspace, workspace_bytes, perm, Lout, d_diag, d_off,
                     pattern, trace_kind, trace_r, stats, 1, 0, nullptr, 0, cuda_stream, L_host, nullptr);
}

int rcp_factor_diag(const rcp_config* cfg, int64_t n, const double* a, int64_t lda, const double* omega_dev,
                    rcp_draw_fn draw, void* draw_ctx, void* workspace, size_t workspace_bytes, int64_t* perm,
                    double* Lout, double* d_diag, double* d_off, int8_t* pattern, int8_t* trace_kind,
                    int32_t* trace_r, rcp_stats* stats, rcp_diag* diag, void* cuda_stream) {
  if (!diag || diag->cap < n + 1 || (diag->track_full && !diag->snapshots) ||
      (diag->audit && (!diag->drift || !diag->omega_orig)))
    return RCP_ERR_INVALID_ARG;
  return factor_core(cfg, n, a, lda, omega_dev, draw, draw_ctx, workspace, workspace_bytes, perm, Lout, d_diag, d_off,
                     pattern, trace_kind, trace_r, stats, 1, 0, nullptr, 0, cuda_stream, nullptr, nullptr, diag);
}

// Exact symmetry of a row-major host matrix (core.py:48-53: A == A.T elementwise, so a NaN
// anywhere fails), checked on host threads while the device works; 64 x 64 tile pairs.
struct HostSymCheck {
  std::vector<std::thread> th;
  std::atomic<int> asym{0};
  void start(const double* a, int64_t n, int64_t lda) {
    const int64_t T = 64, nti = (n + T - 1) / T;
    unsigned hw = std::thread::hardware_concurrency();
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)(hw ? hw : 1) / 2, 8, nti}));
    for (int tt = 0; tt < nt; ++tt)
      th.emplace_back([this, a, n, lda, nti, nt, tt]() {
        for (int64_t I = tt; I < nti; I += nt) {  // tile row I: pairs (I, J <= I)
          if (asym.load(std::memory_order_relaxed)) return;
          const int64_t i0 = I * T, i1 = std::min(n, i0 + T);
          int bad = 0;
          for (int64_t J = 0; J <= I; ++J) {
            const int64_t j0 = J * T, j1 = std::min(n, j0 + T);
            for (int64_t i = i0; i < i1; ++i) {
              const double* ri = a + i * lda;
              const int64_t je = (I == J) ? i + 1 : j1;
              for (int64_t j = j0; j < je; ++j) bad |= !(ri[j] == a[j * lda + i]);
            }
          }
          if (bad) {
            asym.store(1);
            return;
          }
        }
      });
  }
  bool join() {
    for (auto& x : th) x.join();
    th.clear();
    return asym.load() != 0;
  }
  ~HostSymCheck() { join(); }
};

int rcp_factor_host(const rcp_config* cfg, int64_t n, const double* a_host, int64_t lda, const double* omega_dev,
                    rcp_draw_fn draw, void* draw_ctx, void* workspace, size_t workspace_bytes, int64_t* perm,
                    double* Lout, double* d_diag, double* d_off, int8_t* pattern, int8_t* trace_kind,
                    int32_t* trace_r, rcp_stats* stats, double* L_host, void* cuda_stream) {
  if (!a_host || n < 1 || lda < n) return RCP_ERR_INVALID_ARG;
  HostSymCheck chk;
  chk.start(a_host, n, lda);
  const int rc = factor_core(cfg, n, nullptr, lda, omega_dev, draw, draw_ctx, workspace, workspace_bytes, perm, Lout,
                             d_diag, d_off, pattern, trace_kind, trace_r, stats, 1, 0, nullptr, 0, cuda_stream,
                             L_host, a_host);
  if (rc != RCP_ERR_INVALID_ARG && rc != RCP_ERR_WORKSPACE && chk.join()) {
    if (stats) snprintf(stats->message, sizeof(stats->message), "A must be symmetric");
    return RCP_ERR_NOT_SYMMETRIC;  // the reference checks symmetry first (core.py:48-53)
  }
  return rc;
}

static int factor_core(const rcp_config* cfg, int64_t n, const double* a, int64_t lda, const double* omega_dev,
                       rcp_draw_fn draw, void* draw_ctx, void* workspace, size_t workspace_bytes, int64_t* perm,
                       double* Lout, double* d_diag, double* d_off, int8_t* pattern, int8_t* trace_kind,
                       int32_t* trace_r, rcp_stats* stats, int world, int emulate, void* worker_ws,
                       size_t worker_ws_bytes, void* cuda_stream, double* L_host, const double* a_host,
                       rcp_diag* diag) {
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->deficient_from = -1;
  }
  int vc = validate_cfg(cfg, n);
  if (vc != RCP_OK) return vc;
  const bool rcp_strat = cfg->strategy == RCP_STRATEGY_RCP;  // bkpp / bbk: no sketch (factor.py:306)
  if (lda < n || (!a && !a_host) || (rcp_strat && !omega_dev && !(a_host && draw)) || !perm || !Lout || !d_diag ||
      !d_off || !pattern)
    return RCP_ERR_INVALID_ARG;
  const rcp_config c = *cfg;
  const Layout Lay = make_layout(n, c);
  if (!workspace || workspace_bytes < Lay.total) return RCP_ERR_WORKSPACE;
  if (world < 1 || world > kMaxWorld) return RCP_ERR_INVALID_ARG;
  const size_t wslot = rcp_worker_workspace_bytes(n, cfg);
  if (world > 1 && emulate && (!worker_ws || worker_ws_bytes < wslot * (size_t)(world - 1))) return RCP_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  DistShared* dsh = reinterpret_cast<DistShared*>(ws + Lay.dist);
  unsigned long long dseq = 0;  // multi-GPU signal sequence
  std::vector<WorkerBufs> vworkers;  // emulation: the other ranks' scratch on this device
  if (world > 1 && emulate) {
    for (int r = 1; r < world; ++r) {
      unsigned char* b = reinterpret_cast<unsigned char*>(worker_ws) + wslot * (size_t)(r - 1);
      vworkers.push_back(carve_worker(b, n, Lay));
    }
  }
  // the workers must be released whatever happens (errors included)
  struct DistFinish {
    DistShared* sh;
    cudaStream_t st;
    int world;
    ~DistFinish() {
      if (world > 1) {
        launch_dist_finish(sh, st);
        cudaStreamSynchronize(st);
      }
    }
  } dist_finish{dsh, st, world};
  auto dptr = [&](size_t off) { return reinterpret_cast<double*>(ws + off); };
  auto iptr = [&](size_t off) { return reinterpret_cast<int*>(ws + off); };

  double* A[2] = {dptr(Lay.A0), dptr(Lay.A1)};
  double* B[2] = {dptr(Lay.B0), dptr(Lay.B1)};
  int* permb[2] = {iptr(Lay.perm0), iptr(Lay.perm1)};
  double* Lbuf = dptr(Lay.Lbuf);
  double* W = dptr(Lay.W);
  double* Lneg = dptr(Lay.Lneg);
  double* Wg = dptr(Lay.Wg);
  double* Y = dptr(Lay.Y);
  double* L11c = dptr(Lay.L11);
  double* omg = dptr(Lay.omega);
  int* phys = iptr(Lay.phys);
  int* lop = iptr(Lay.lop);
  int* pol = iptr(Lay.pol);
  int* poso = iptr(Lay.poso);
  int* snap = iptr(Lay.snap);
  PanelState* dstate = reinterpret_cast<PanelState*>(ws + Lay.state);
  unsigned long long* tstamp = reinterpret_cast<unsigned long long*>(ws + Lay.tstamp);
  Scal* dscal = reinterpret_cast<Scal*>(ws + Lay.scal);
  const int P = c.p;
  const int tpad = Lay.tpad;

  int dev = 0;
  RCP_CHECK(cudaGetDevice(&dev));
  int num_sms = 0, max_optin = 0;
  // device attributes and kernel smem limits once per device and thread (driver calls here can
  // queue behind an NVML client such as a running nvidia-smi)
  static thread_local int attr_dev = -1, attr_sms = 0, attr_optin = 0, attr_static = 0;
  if (attr_dev != dev) {
    RCP_CHECK(cudaDeviceGetAttribute(&attr_sms, cudaDevAttrMultiProcessorCount, dev));
    RCP_CHECK(cudaDeviceGetAttribute(&attr_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    attr_static = panel_static_smem_bytes();
    RCP_CHECK(panel_init_attributes(attr_optin - attr_static));
    RCP_CHECK(gemm_init_attributes());
    attr_dev = dev;
  }
  num_sms = attr_sms;
  max_optin = attr_optin;
  const int smem_budget = max_optin - attr_static - 1024;

  // pinned snapshots and CUDA events come from a per-thread cache (cudaMallocHost /
  // cudaFreeHost and event creation per call cost milliseconds of GPU idle time)
  HostCache& hc = host_cache(dev);
  if (!hc.ok) {
    if (stats) snprintf(stats->message, sizeof(stats->message), "pinned host cache allocation failed");
    return RCP_ERR_CUDA;
  }
  hc.reset();
  PanelState* hstate = hc.hstate;
  Scal* hscal = hc.hscal;
  cudaEvent_t ev_start = hc.event(), ev_stop = hc.event();

  int64_t launches = 0;
  double schur_flops = 0.0;
  RCP_CHECK(cudaEventRecord(ev_start, st));

  // ---- init state
  PanelState init{};
  init.seq = 0;
  init.err = LLONG_MAX;
  RCP_CHECK(cudaMemcpyAsync(dstate, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  RCP_CHECK(cudaMemsetAsync(ws + Lay.xrec, 0, Lay.state - Lay.xrec, st));  // LL exchange buffers: no stale tags
  RCP_CHECK(cudaMemsetAsync(ws + Lay.tstamp, 0, 8 * 4 * (size_t)(n + 2), st));
  RCP_LAUNCH(launch_tstamp_init(reinterpret_cast<unsigned long long*>(ws + Lay.tstamp), 2 * (n + 2), st));
  RCP_CHECK(cudaMemsetAsync(dscal, 0, sizeof(Scal), st));
  if (world > 1 && emulate) RCP_CHECK(cudaMemsetAsync(dsh, 0, sizeof(DistShared), st));
  RCP_CHECK(cudaMemsetAsync(d_off, 0, sizeof(double) * n, st));
  if (trace_kind) RCP_CHECK(cudaMemsetAsync(trace_kind, -1, n, st));
  if (trace_r) RCP_CHECK(cudaMemsetAsync(trace_r, 0xff, sizeof(int32_t) * n, st));

  // ---- input validation + copy (factor.py:277-286)
  const double* a_in = a;
  int64_t lda_in = lda;
  std::vector<double> omega_buf;
  if (a_host) {  // host input: only its lower trapezoid crosses PCIe (256-row block rows), staged
    double* stage = A[1];  // in A1 (free until the first trailing update), mirrored by the kernel
    for (int64_t i0 = 0; i0 < n; i0 += 256) {
      const int64_t i1 = std::min<int64_t>(n, i0 + 256);
      RCP_CHECK(cudaMemcpy2DAsync(stage + i0 * n, (size_t)n * sizeof(double), a_host + i0 * lda,
                                  (size_t)lda * sizeof(double), (size_t)i1 * sizeof(double), (size_t)(i1 - i0),
                                  cudaMemcpyHostToDevice, st));
    }
    a_in = stage;
    lda_in = n;
  }
  RCP_LAUNCH(launch_validate_copy(a_in, lda_in, n, A[0], dscal->vflags, &dscal->amax, st, a_host ? 1 : 0));
  if (a_host && rcp_strat && !omega_dev) {  // Omega = the stream's first draw, drawn while the copies run
    omega_buf.resize((size_t)P * n);
    if (draw(draw_ctx, P, n, omega_buf.data()) != 0) return RCP_ERR_NEED_NORMALS;
    RCP_CHECK(cudaMemcpyAsync(omg, omega_buf.data(), sizeof(double) * (size_t)P * n, cudaMemcpyHostToDevice, st));
    omega_dev = omg;
  }
  RCP_CHECK(cudaMemcpyAsync(hscal, dscal, sizeof(Scal), cudaMemcpyDeviceToHost, st));
  RCP_CHECK(cudaStreamSynchronize(st));
  if (hscal->vflags[0]) return RCP_ERR_NOT_SYMMETRIC;
  if (hscal->vflags[1]) return RCP_ERR_NONFINITE_INPUT;
  const double amax = hscal->amax;

  const bool dsnap = diag && diag->track_full, daudit = diag && diag->audit && rcp_strat;
  if (diag) {
    diag->n_snapshots = diag->n_drift = 0;
    if (dsnap) RCP_CHECK(cudaMemsetAsync(diag->snapshots, 0, sizeof(double) * 2 * (size_t)diag->cap, st));
    if (diag->audit && diag->drift) RCP_CHECK(cudaMemsetAsync(diag->drift, 0, sizeof(double) * (size_t)diag->cap, st));
    if (daudit)  // Omega in original column order (the permutation is the identity here)
      RCP_CHECK(cudaMemcpyAsync(diag->omega_orig, omega_dev, sizeof(double) * (size_t)P * n, cudaMemcpyDeviceToDevice, st));
  }
  // ---- sketch B = Omega A (factor.py:307-309) and guard setup (factor.py:314-317)
  if (rcp_strat) RCP_LAUNCH(launch_sketch_gemm(P, n, omega_dev, n, A[0], n, B[0], 0, st));
  const bool armed = rcp_strat && c.robust_r >= 1;  // factor.py:314
  double delta = armed ? 1.0 / c.robust_r : 0.0;
  double thr = armed ? std::pow(DBL_EPSILON, delta) : 0.0;
  double beta = 0.0;
  if (armed) {
    RCP_LAUNCH(launch_sketch_norm_max(B[0], P, n, &dscal->beta, st));
    RCP_CHECK(cudaMemcpyAsync(hscal, dscal, sizeof(Scal), cudaMemcpyDeviceToHost, st));
    RCP_CHECK(cudaStreamSynchronize(st));
    beta = hscal->beta;
  }
  RCP_LAUNCH(launch_iota(n, permb[0], st));

  int curA = 0, curB = 0;  // ping-pong buffers holding the current trailing block / sketch
  int pcur = 0;      // perm buffer for the current order
  int64_t k = 0;
  int64_t recomputes = 0;
  // panel-level op counters (factor.py:377-378, 564-565, 577-599); step-level ones come from the kernel
  long long h_mul = 0, h_add = 0, h_div = 0, h_cmp = 0;
  int64_t deficient_from = -1;
  std::vector<PanelRecord> panels;
  std::vector<double> draw_buf;

  if (armed && beta == 0.0) {  // factor.py:510-511
    RCP_LAUNCH(launch_deficient_fill(n, 0, permb[0], perm, d_diag, d_off, pattern, st));
    deficient_from = 0;
    k = n;
  }

  // ---- panel loop, device driven (see PanelDesc): the host enqueues panels back to back
  // and reads their outcome only once per batch; guard events and errors stop the device
  // chain, the host rolls back to that panel and handles them.
  const bool q1 = rcp_strat && (c.q == 1);
  const int q_eff = rcp_strat ? c.q : 0;  // no sketch selection outside rcp (factor.py:548, 608)
  int sms_cap = std::min(num_sms, kMaxSMs);
  // Experiment knob (SM-partition model): RCP_PANEL_SMS caps the panel grid as if
  // only that many SMs were reserved for the panel.  Unset in production.
  if (const char* e = std::getenv("RCP_PANEL_SMS")) {
    const int v = std::atoi(e);
    if (v >= 1 && v < sms_cap) sms_cap = v;
  }
  // launch grid: the largest G any panel can ask for (G(m0) is not monotone in m0); CTAs
  // beyond a panel's own G return at once
  const int gmax = sms_cap;
  PanelDesc* ddesc = reinterpret_cast<PanelDesc*>(ws + Lay.desc);
  PanelLog* dplog = reinterpret_cast<PanelLog*>(ws + Lay.plog);
  PanelDesc* hdesc = hc.hdesc;  // [slot][2]: double-buffered chain snapshots
  PanelState* hsnap = hc.hsnap;  // [slot]
  struct Hist {
    int curA, curB, pcur;
  };
  std::vector<Hist> hist;
  int guard_req = armed ? 1 : 0;
  int pidx = 0;
  bool chain_done = (k >= n);
  int stop_k0 = -1;
  if (!chain_done) {
    hdesc[0] = PanelDesc{(int)k, 1, 0, 0, 0, 0, 0};
    RCP_CHECK(cudaMemcpyAsync(ddesc, hdesc, sizeof(PanelDesc), cudaMemcpyHostToDevice, st));
    int neg1 = -1;
    RCP_CHECK(cudaMemcpyAsync(&dstate->stop_pidx, &neg1, sizeof(int), cudaMemcpyHostToDevice, st));
  }
  int batch = 2;
  constexpr int kBatchMax = 16;
  int nbatch = 0;                // batches enqueued since the last fix-up
  int batch_end[2] = {0, 0};     // pidx after each snapshot slot's batch
  PanelParams base{};
  base.n = n;
  base.P = P;
  base.alpha = rcp_strat ? std::sqrt(2.0) / 2.0 : (1.0 + std::sqrt(17.0)) / 8.0;  // factor.py:299
  base.strategy = c.strategy;
  base.bkscr = Lneg;
  base.tstamp = tstamp;  // free while a panel runs (the gather fills it afterwards)
  base.q1 = q1 ? 1 : 0;
  base.qscr = dptr(Lay.qscr);
  base.Lbuf = Lbuf;
  base.W = W;
  base.log_of_phys = lop;
  base.phys_of_log = pol;
  base.perm_out = perm;
  base.d_diag = d_diag;
  base.d_off = d_off;
  base.pattern = pattern;
  base.trace_kind = trace_kind;
  base.trace_r = trace_r;
  base.xll = reinterpret_cast<unsigned long long*>(ws + Lay.xrec);
  base.qll = reinterpret_cast<unsigned long long*>(ws + Lay.qrec);
  base.qcll = reinterpret_cast<unsigned long long*>(ws + Lay.qcol);
  base.sdll = reinterpret_cast<unsigned long long*>(ws + Lay.sdec);
  base.qdll = reinterpret_cast<unsigned long long*>(ws + Lay.qdec);
  base.st = dstate;
  base.b = c.b;
  base.q = q_eff;
  base.num_sms = sms_cap;
  base.smem_budget = smem_budget;

  // L in final order is written row block by row block as panels commit (finalize_rows after
  // each gather); its strictly-upper part stays zero
  double* lorig = dptr(Lay.lorig);
  RCP_CHECK(cudaMemsetAsync(Lout, 0, sizeof(double) * (size_t)n * n, st));
  RCP_LAUNCH(launch_unit_diag(n, Lout, st));
  HostLSink hsink;
  if (L_host) {
    if (!hc.cst) RCP_CHECK(cudaStreamCreateWithFlags(&hc.cst, cudaStreamNonBlocking));
    hsink.start(L_host, Lout, n, hc.cst);
  }

  while (!chain_done) {
    for (int bi = 0; bi < batch; ++bi) {
      hist.push_back(Hist{curA, curB, pcur});
      PanelDesc* din = ddesc + (pidx & 1);
      PanelDesc* dout = ddesc + ((pidx + 1) & 1);
      PanelParams prm = base;
      prm.desc = din;
      prm.guard_mode = guard_req;
      prm.guard_limit = thr * beta;
      prm.A = A[curA];
      prm.B = B[curB];
      prm.Bout = B[curB ^ 1];
      prm.perm_cur = permb[pcur];
      if (dsnap) RCP_LAUNCH(launch_snapshot(n, A[curA], din, diag->snapshots + 2 * (size_t)pidx, st));
      RCP_LAUNCH(launch_panel(prm, gmax, (size_t)smem_budget, st));
      RCP_LAUNCH(launch_panel_commit(din, dout, dplog, dstate, n, c.b, q_eff, P, (long long)Lay.snap_cap, st));
      RCP_LAUNCH(launch_gather(n, 0, 0, 0, tpad, 0, pol, Lbuf, W, permb[pcur], permb[pcur ^ 1], snap, phys, Lneg, Wg,
                               L11c, st, din, lorig));
      RCP_LAUNCH(launch_finalize_rows(n, 0, 0, 0, 0, perm, lorig, L11c, Lout, &dscal->maxmult, c.b + 2, st, din));
      // sketch correction once per panel (factor.py:554-565): Y = B1 L11^-T, then B2 -= Y L21^T as
      // extra tiles of the Schur kernel (single GPU) or as its own GEMM (multi-GPU)
      const bool sketch_corr = rcp_strat && !q1;
      const bool fused_sk = sketch_corr && world == 1 && RCP_FUSED_SKETCH;
      if (fused_sk) RCP_LAUNCH(launch_ysolve(n, P, 0, c.b, tpad, pol, B[curB], L11c, Y, st, din));
      if (world > 1) {  // hand the panel to the other devices (dist.cuh)
        ++dseq;
        RCP_LAUNCH(launch_dist_signal(dsh, dseq, curA, pidx & 1, st));
        for (int r = 1; r < (int)vworkers.size() + 1; ++r)
          RCP_LAUNCH(launch_worker_panel(dsh, r, world, dseq, A[0], A[1], ddesc, Lneg, Wg, phys, n, tpad,
                                         vworkers[r - 1], st));
      }
      RCP_LAUNCH(launch_schur_update(n, 0, 0, Lneg, Wg, tpad, 0, A[curA], phys, A[curA ^ 1], st, din, 0, world,
                                     fused_sk ? Y : nullptr, B[curB], B[curB ^ 1], P, tstamp));
      if (world > 1) RCP_LAUNCH(launch_dist_wait_done(dsh, world, dseq, st));
      if (sketch_corr && !fused_sk) {
        RCP_LAUNCH(launch_ysolve(n, P, 0, c.b, tpad, pol, B[curB], L11c, Y, st, din));
        RCP_LAUNCH(launch_sketch_correction(P, n, 0, Y, tpad, c.b, Lneg, B[curB], phys, B[curB ^ 1], st, din, n));
      }
      // q = 1: the panel kernel itself wrote the per-step-updated sketch into B[curB ^ 1]
      if (daudit)
        RCP_LAUNCH(launch_drift(n, P, A[curA ^ 1], B[curB ^ 1], diag->omega_orig, permb[pcur ^ 1], din,
                                diag->drift + pidx, st));
      curA ^= 1;
      curB ^= 1;
      pcur ^= 1;
      ++pidx;
      guard_req = armed ? 1 : 0;  // a stop check (2) applies to a relaunched panel only
    }
    // snapshot the chain after this batch, then inspect the PREVIOUS batch's snapshot: the
    // device always has one batch queued while the host waits
    {
      const int slot = nbatch & 1;
      RCP_CHECK(cudaMemcpyAsync(hsnap + slot, dstate, sizeof(PanelState), cudaMemcpyDeviceToHost, st));
      RCP_CHECK(cudaMemcpyAsync(hdesc + 2 * slot, ddesc, 2 * sizeof(PanelDesc), cudaMemcpyDeviceToHost, st));
      RCP_CHECK(cudaEventRecord(hc.bev[slot], st));
      batch_end[slot] = pidx;
      ++nbatch;
    }
    batch = std::min(batch * 2, kBatchMax);
    int chk;  // snapshot slot to inspect
    if (nbatch == 1) {  // first batch: nothing older to look at yet
      continue;
    }
    chk = (nbatch - 2) & 1;
    RCP_CHECK(cudaEventSynchronize(hc.bev[chk]));
    *hstate = hsnap[chk];
    if (hstate->status == 0 && hstate->err == LLONG_MAX) {
      hsink.flush(hstate->k_end, hc.bev[chk]);  // rows before k_end are final in Lout
      // the descriptor after that batch's last panel decides whether the chain went on
      if (!hdesc[2 * chk + (batch_end[chk] & 1)].run) {
        chain_done = true;  // k == n; the newer batch is all no-ops
        RCP_CHECK(cudaStreamSynchronize(st));
      }
      continue;
    }
    RCP_CHECK(cudaStreamSynchronize(st));  // drain the newer (no-op) batch before any fix-up
    hdesc[0] = hdesc[2 * chk];
    hdesc[1] = hdesc[2 * chk + 1];
    // a guard event or an error at panel tp: later panels were no-ops; roll back to tp
    const int tp = hstate->stop_pidx;
    if (tp < 0 || tp >= (int)hist.size()) {
      if (stats) snprintf(stats->message, sizeof(stats->message), "panel chain lost its stop index");
      return RCP_ERR_CUDA;
    }
    curA = hist[tp].curA;
    curB = hist[tp].curB;
    pcur = hist[tp].pcur;
    hist.resize(tp);
    pidx = tp;
    const int k0 = hdesc[0].k0;  // no-op panels carry the stopped panel's k0 / snap_off forward
    const long long so = hdesc[0].snap_off;
    const int m0 = (int)(n - k0);
    if (hstate->err != LLONG_MAX) {
      if (stats) {
        stats->num_kind = (int)(hstate->err & 0xff);
        stats->num_step = (int)(hstate->err >> 8);
        stats->n_steps = hstate->n_steps;
        stats->n_2x2 = hstate->n_2x2;
      }
      return RCP_ERR_NUMERICAL;
    }
    if (hstate->status == 99 || hstate->status == 97) {
      if (stats)
        snprintf(stats->message, sizeof(stats->message), "panel %s at k=%d",
                 hstate->status == 99 ? "exchange watchdog fired" : "snapshot capacity exceeded", k0);
      return RCP_ERR_CUDA;
    }
    if (m0 > 1) {  // the stopped / tripped panel's sketch norms (factor.py:576-577, 608-610)
      h_mul += (long long)P * (m0 - 1);
      h_add += (long long)P * (m0 - 1);
      h_cmp += m0 - 1;
    }
    if (hstate->status == 2) {  // confirmed collapse: deficient tail (factor.py:405-410, 381-385)
      stop_k0 = k0;
      break;
    }
    // guard trip: fresh projection of the active block (factor.py:392-404), relaunch panel tp
    if (!q1 && m0 > 1) {  // charged again by the relaunch's commit -> undo the extra charge
      h_mul -= (long long)P * (m0 - 1);
      h_add -= (long long)P * (m0 - 1);
      h_cmp -= m0 - 1;
    }
    if (q1 && m0 > 1) {  // q = 1: the relaunch charges the same step's norms itself
      h_mul -= (long long)P * (m0 - 1);
      h_add -= (long long)P * (m0 - 1);
      h_cmp -= m0 - 1;
    }
    if (!draw) {
      if (stats) snprintf(stats->message, sizeof(stats->message), "guard recompute needs normals at k=%d", k0);
      return RCP_ERR_NEED_NORMALS;
    }
    draw_buf.resize((size_t)P * m0);
    if (draw(draw_ctx, P, m0, draw_buf.data()) != 0) return RCP_ERR_NEED_NORMALS;
    RCP_CHECK(cudaMemcpyAsync(omg, draw_buf.data(), sizeof(double) * (size_t)P * m0, cudaMemcpyHostToDevice, st));
    if (daudit) RCP_LAUNCH(launch_omega_scatter(n, P, k0, omg, m0, permb[pcur], diag->omega_orig, st));
#if !RCP_FULL_STORAGE
    RCP_LAUNCH(launch_mirror_lower(n, k0, A[curA], st));  // the projection reads full columns
#endif
    RCP_LAUNCH(launch_sketch_gemm(P, m0, omg, m0, A[curA] + k0 + (int64_t)k0 * n, n, B[curB], k0, st));
    recomputes += 1;
    delta += 1.0 / c.robust_r;
    thr = std::pow(DBL_EPSILON, delta);
    guard_req = 2;
    hdesc[0] = PanelDesc{k0, 1, tp, 0, 0, 0, so};
    RCP_CHECK(cudaMemcpyAsync(ddesc + (tp & 1), hdesc, sizeof(PanelDesc), cudaMemcpyHostToDevice, st));
    RCP_CHECK(cudaMemsetAsync(&dstate->status, 0, sizeof(int), st));
    int neg1 = -1;
    RCP_CHECK(cudaMemcpyAsync(&dstate->stop_pidx, &neg1, sizeof(int), cudaMemcpyHostToDevice, st));
    RCP_CHECK(cudaStreamSynchronize(st));  // neg1 / hdesc are host stack / pinned values
    batch = 1;
    nbatch = 0;
  }
  if (world > 1) {
    int derr = 0;
    RCP_CHECK(cudaMemcpyAsync(&derr, &dsh->error, sizeof(int), cudaMemcpyDeviceToHost, st));
    RCP_CHECK(cudaStreamSynchronize(st));
    if (derr) {
      if (stats) snprintf(stats->message, sizeof(stats->message), "multi-GPU peer watchdog fired");
      return RCP_ERR_CUDA;
    }
  }
  if (stop_k0 >= 0) {
    RCP_LAUNCH(launch_deficient_fill(n, stop_k0, permb[pcur], perm, d_diag, d_off, pattern, st));
    deficient_from = stop_k0;
  }
  // committed panels: records for the assembly, flop and op-counter bookkeeping
  {
    int np = 0;
    RCP_CHECK(cudaMemcpyAsync(hstate, dstate, sizeof(PanelState), cudaMemcpyDeviceToHost, st));
    RCP_CHECK(cudaStreamSynchronize(st));
    np = hstate->panels_done;
    std::vector<PanelLog> logs((size_t)np);
    if (np > 0) {
      RCP_CHECK(cudaMemcpyAsync(logs.data(), dplog, sizeof(PanelLog) * (size_t)np, cudaMemcpyDeviceToHost, st));
      RCP_CHECK(cudaStreamSynchronize(st));
    }
    if (diag) {  // snapshots: one per step run (the stopping one included); drift: panels with k < n
      diag->n_snapshots = dsnap ? (int64_t)np + (stop_k0 >= 0 ? 1 : 0) : 0;
      int64_t nd = 0;
      for (const PanelLog& lg : logs) nd += (lg.k_end < n) ? 1 : 0;
      diag->n_drift = daudit ? nd : 0;
    }
    for (const PanelLog& lg : logs) {
      panels.push_back(PanelRecord{lg.k0, lg.k_end, (int64_t)lg.snap_off});
      const int t = lg.k_end - lg.k0;
      const long long mp = n - lg.k_end;
      const int m0 = lg.m0;
      if (rcp_strat && !q1 && m0 > 1) {  // preselect norms (factor.py:576-577)
        h_mul += (long long)P * (m0 - 1);
        h_add += (long long)P * (m0 - 1);
        h_cmp += m0 - 1;
      }
      for (int j = 0; j < lg.qn; ++j) {  // QRCP slots (sketch.py:135-169 via factor.py:586-599)
        h_cmp += m0 - 1 - j;
        h_mul += 2LL * P * (m0 - j);
        h_add += 2LL * P * (m0 - j);
      }
      if (mp > 0 && t > 0) {
        schur_flops += (double)t * (double)mp * (double)(mp + 1);
        if (rcp_strat && !q1 && world == 1 && RCP_FUSED_SKETCH)  // sketch tiles in the same kernel
          schur_flops += 2.0 * (double)P * (double)t * (double)mp;
        h_mul += (long long)t * (mp * (mp + 1) / 2);  // _apply_trailing (factor.py:377-378)
        h_add += (long long)t * (mp * (mp + 1) / 2);
        if (rcp_strat && !q1) {
          h_mul += (long long)t * P * mp + (long long)(t * (t - 1) / 2) * mp;
          h_add += (long long)t * P * mp + (long long)(t * (t - 1) / 2) * mp;
        }
      }
    }
  }

  // ---- assemble L in final order + statistics (factor.py:514-538)
  if (stop_k0 > 0) {  // rows of a deficient tail: the committed columns (factor.py:405-410)
    RCP_LAUNCH(launch_finalize_rows(n, stop_k0, n, stop_k0, 0, perm, lorig, nullptr, Lout, &dscal->maxmult, 0, st));
  }
  RCP_LAUNCH(launch_dmax(n, d_diag, d_off, &dscal->dmax, st));
  RCP_CHECK(cudaEventRecord(ev_stop, st));
  hsink.flush(n, ev_stop);  // the remaining block rows (tail included)
  RCP_CHECK(cudaMemcpyAsync(hscal, dscal, sizeof(Scal), cudaMemcpyDeviceToHost, st));
  RCP_CHECK(cudaMemcpyAsync(hstate, dstate, sizeof(PanelState), cudaMemcpyDeviceToHost, st));
  RCP_CHECK(cudaStreamSynchronize(st));
  if (!hsink.finish()) {
    if (stats) snprintf(stats->message, sizeof(stats->message), "host L copy failed");
    return RCP_ERR_CUDA;
  }

  if (stats) {
    stats->amax = amax;
    stats->dmax = hscal->dmax;
    stats->max_multiplier = n > 1 ? hscal->maxmult : 0.0;
    if (amax == 0.0) {
      stats->rho_cheap = hscal->dmax == 0.0 ? 1.0 : INFINITY;
    } else {
      stats->rho_cheap = hscal->dmax / amax;
    }
    stats->recompute_count = recomputes;
    stats->n_panels = (int64_t)panels.size();
    stats->n_steps = hstate->n_steps;
    stats->n_2x2 = hstate->n_2x2;
    stats->deficient_from = deficient_from;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev_start, ev_stop);
    stats->t_factor_ms = ms;
    double tp = 0, ts = 0;  // kernel durations from the device timestamps (one copy)
    {
      const int np = hstate->panels_done + 2 < (int)n + 2 ? hstate->panels_done + 2 : (int)n + 2;
      std::vector<unsigned long long> h(4 * (size_t)np);
      if (cudaMemcpy(h.data(), tstamp, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost) == cudaSuccess) {
        for (int i = 0; i < np; ++i) {
          const unsigned long long* q = &h[4 * (size_t)i];
          if (q[0] != ~0ULL && q[1] > q[0]) tp += (double)(q[1] - q[0]) * 1e-6;
          if (q[2] != ~0ULL && q[3] > q[2]) ts += (double)(q[3] - q[2]) * 1e-6;
        }
      }
    }
    stats->t_panel_ms = tp;
    stats->t_schur_ms = ts;
    stats->schur_flops = schur_flops;
    static thread_local int clk_khz = 0, clk_dev = -1;
    if (clk_dev != dev) {
      cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
      clk_dev = dev;
    }
    for (int i = 0; i < 16; ++i) stats->panel_prof_ms[i] = clk_khz > 0 ? (double)hstate->cyc[i] / clk_khz : 0.0;
    stats->n_launches = launches;
    stats->mults = h_mul + hstate->cnt[0];
    stats->adds = h_add + hstate->cnt[1];
    stats->divs = h_div + hstate->cnt[2];
    stats->comps = h_cmp + hstate->cnt[3];
  }
  return RCP_OK;
}


int rcp_dist_prepare(int64_t n, const rcp_config* cfg, void* workspace, void* cuda_stream) {
  if (validate_cfg(cfg, n) != RCP_OK || !workspace) return RCP_ERR_INVALID_ARG;
  const Layout Lay = make_layout(n, *cfg);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  if (cudaMemsetAsync(reinterpret_cast<unsigned char*>(workspace) + Lay.dist, 0, sizeof(DistShared), st) != cudaSuccess)
    return RCP_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? RCP_OK : RCP_ERR_CUDA;
}

int rcp_schur_worker(const rcp_config* cfg, int64_t n, int rank, int world, void* rank0_workspace, void* worker_ws,
                     size_t worker_ws_bytes, void* cuda_stream) {
  if (validate_cfg(cfg, n) != RCP_OK || !rank0_workspace || rank < 1 || rank >= world || world > kMaxWorld)
    return RCP_ERR_INVALID_ARG;
  if (!worker_ws || worker_ws_bytes < rcp_worker_workspace_bytes(n, cfg)) return RCP_ERR_WORKSPACE;
  const Layout Lay = make_layout(n, *cfg);
  unsigned char* b0 = reinterpret_cast<unsigned char*>(rank0_workspace);
  DistShared* sh = reinterpret_cast<DistShared*>(b0 + Lay.dist);
  double* A0 = reinterpret_cast<double*>(b0 + Lay.A0);
  double* A1 = reinterpret_cast<double*>(b0 + Lay.A1);
  const PanelDesc* desc = reinterpret_cast<const PanelDesc*>(b0 + Lay.desc);
  const double* Lneg0 = reinterpret_cast<const double*>(b0 + Lay.Lneg);
  const double* Wg0 = reinterpret_cast<const double*>(b0 + Lay.Wg);
  const int* phys0 = reinterpret_cast<const int*>(b0 + Lay.phys);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  const WorkerBufs wb = carve_worker(reinterpret_cast<unsigned char*>(worker_ws), n, Lay);
  if (gemm_init_attributes() != cudaSuccess) return RCP_ERR_CUDA;
  unsigned long long seq = 0;
  SchurDyn hd{};
  int hflags[2] = {0, 0};
  for (int batch = 2;; batch = std::min(batch * 2, 16)) {
    for (int i = 0; i < batch; ++i)
      if (launch_worker_panel(sh, rank, world, ++seq, A0, A1, desc, Lneg0, Wg0, phys0, n, Lay.tpad, wb, st) !=
          cudaSuccess)
        return RCP_ERR_CUDA;
    if (cudaMemcpyAsync(&hd, wb.dyn, sizeof(SchurDyn), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(hflags, &sh->finished, 2 * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return RCP_ERR_CUDA;
    if (hflags[1]) return RCP_ERR_CUDA;  // watchdog
    if (!hd.go) return RCP_OK;            // rank 0 finished
  }
}

int rcp_lower_to_host(int64_t n, const double* dL, double* hL, void* cuda_stream) {
  // The unit-lower L (row-major n x n on the device) into a dense host array: block rows of the
  // lower trapezoid go over PCIe as 2D copies (half the bytes of the dense matrix) while host
  // threads zero the strictly upper part the copies do not cover (disjoint regions).
  if (n < 0 || (n > 0 && (dL == nullptr || hL == nullptr))) return RCP_ERR_INVALID_ARG;
  if (n == 0) return RCP_OK;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const int64_t blk = 256;
  const size_t pitch = static_cast<size_t>(n) * sizeof(double);
  for (int64_t i0 = 0; i0 < n; i0 += blk) {
    const int64_t i1 = std::min(n, i0 + blk);
    if (cudaMemcpy2DAsync(hL + i0 * n, pitch, dL + i0 * n, pitch, static_cast<size_t>(i1) * sizeof(double),
                          static_cast<size_t>(i1 - i0), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return RCP_ERR_CUDA;
  }
  const int64_t nb = (n + blk - 1) / blk;
  unsigned hw = std::thread::hardware_concurrency();
  const int nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({(int64_t)(hw ? hw : 1), 16, nb})));
  auto zero = [&](int tt) {
    for (int64_t b = tt; b < nb; b += nt) {
      const int64_t i0 = b * blk, i1 = std::min(n, i0 + blk);
      if (i1 < n)
        for (int64_t i = i0; i < i1; ++i) memset(hL + i * n + i1, 0, static_cast<size_t>(n - i1) * sizeof(double));
    }
  };
  std::vector<std::thread> th;
  for (int tt = 1; tt < nt; ++tt) th.emplace_back(zero, tt);
  zero(0);
  for (auto& x : th) x.join();
  return cudaStreamSynchronize(st) == cudaSuccess ? RCP_OK : RCP_ERR_CUDA;
}

int rcp_device_alloc(size_t bytes, void** ptr) {
  return cudaMalloc(ptr, bytes) == cudaSuccess ? RCP_OK : RCP_ERR_CUDA;
}

int rcp_device_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? RCP_OK : RCP_ERR_CUDA; }

int rcp_ipc_export(const void* base, void* handle_out) {
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(base)) != cudaSuccess) return RCP_ERR_CUDA;
  memcpy(handle_out, &h, sizeof(h));
  return RCP_OK;
}

int rcp_ipc_import(const void* handle, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? RCP_OK : RCP_ERR_CUDA;
}

int rcp_ipc_close(void* ptr) { return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? RCP_OK : RCP_ERR_CUDA; }

size_t rcp_solve_workspace_bytes(int64_t n, int64_t nrhs) {
  if (n < 1 || nrhs < 1) return 0;
  return solve_workspace_bytes(n, nrhs) + 256;
}

int rcp_solve(int64_t n, const int64_t* perm, const double* L, const double* d_diag, const double* d_off,
              const int8_t* pattern, int64_t nrhs, const double* b, double* x, void* workspace,
              size_t workspace_bytes, int32_t* singular, void* cuda_stream) {
  rcp_stats* stats = nullptr;
  if (n < 1 || nrhs < 1 || !perm || !L || !d_diag || !d_off || !pattern || !b || !x) return RCP_ERR_INVALID_ARG;
  const size_t need = rcp_solve_workspace_bytes(n, nrhs);
  if (!workspace || workspace_bytes < need) return RCP_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  int* dflag = reinterpret_cast<int*>(ws + solve_workspace_bytes(n, nrhs));
  int dev = 0, num_sms = 0;
  RCP_CHECK(cudaGetDevice(&dev));
  RCP_CHECK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  RCP_CHECK(cudaMemsetAsync(dflag, 0, sizeof(int), st));
  RCP_CHECK(solve_device(n, perm, L, d_diag, d_off, pattern, nrhs, b, x, ws, dflag, st, num_sms));
  int h = 0;
  RCP_CHECK(cudaMemcpyAsync(&h, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RCP_CHECK(cudaStreamSynchronize(st));
  if (singular) *singular = h;
  return RCP_OK;
}

int rcp_reconstruct(int64_t n, const double* L, const double* d_diag, const double* d_off, const int8_t* pattern,
                    double* out, void* cuda_stream) {
  rcp_stats* stats = nullptr;
  if (n < 1 || !L || !d_diag || !d_off || !pattern || !out) return RCP_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  void* scratch = nullptr;
  RCP_CHECK(cudaMallocAsync(&scratch, sizeof(double) * (size_t)n * n, st));
  cudaError_t e = reconstruct_device(n, L, d_diag, d_off, pattern, out, reinterpret_cast<double*>(scratch), st);
  cudaFreeAsync(scratch, st);
  RCP_CHECK(e);
  RCP_CHECK(cudaStreamSynchronize(st));
  return RCP_OK;
}

}  // extern "C"
