// Microbenchmark: latency of one grid-wide argmax exchange (+ broadcast of the winner's
// 144-double vector) on B200 for the panel kernel's per-step decisions.
//   reducer : every CTA writes an 11-word LL record, CTA 0 reduces, writes a decision, all read it
//   hier<CS>: thread-block clusters of CS CTAs; members deposit (key, idx) in the leader's smem
//             through DSMEM + a remote mbarrier arrive; each leader publishes one 3-word LL
//             record; every CTA reads all leader records (one L2 hop) and reduces them itself.
// Each step then fetches the winner's LL vector (written before the exchange).
// Checks that all CTAs agree on every winner (checksum).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
constexpr int P = 144;
__device__ __forceinline__ void put(u64* p, unsigned tag, unsigned d) {
  u64 v = ((u64)tag << 32) | d;
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 get(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned hsh(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ unsigned cluster_rank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned cluster_nrank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
  unsigned r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r;
}

// vector publish: words [0, 2P) of this CTA's buffer
__device__ void publish_vec(u64* buf, unsigned tag, int cta) {
  for (int w = threadIdx.x; w < 2 * P; w += blockDim.x) put(buf + w, tag, cta * 1000 + w);
}
__device__ unsigned fetch_vec(const u64* buf, unsigned tag) {
  unsigned acc = 0;
  for (int w = threadIdx.x; w < 2 * P; w += blockDim.x) {
    u64 v;
    do { v = get(buf + w); } while ((unsigned)(v >> 32) != tag);
    acc += (unsigned)v;
  }
  return acc;
}

__global__ void k_reducer(u64* rec, u64* dec, u64* vec, int steps, long long* out, unsigned* chk) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  __shared__ unsigned s_best, s_win;
  __shared__ unsigned s_acc;
  unsigned checksum = 0;
  long long t0 = clock64();
  for (int s = 1; s <= steps; ++s) {
    const unsigned tag = s;
    const int pb = s & 1;
    const unsigned key = hsh(cta * 977 + s * 131);
    publish_vec(vec + ((size_t)pb * G + cta) * 2 * P, tag, cta);
    if (tid == 0) {
      u64* q = rec + ((size_t)pb * G + cta) * 16;
      for (int w = 0; w < 11; ++w) put(q + w, tag, w == 0 ? key : cta);
    }
    if (cta == 0) {
      if (tid == 0) s_best = 0;
      __syncthreads();
      for (int c = tid; c < G; c += blockDim.x) {
        const u64* q = rec + ((size_t)pb * G + c) * 16;
        unsigned w0 = 0;
        while (true) {
          bool ok = true;
          for (int w = 0; w < 11; ++w) { u64 v = get(q + w); ok &= (unsigned)(v >> 32) == tag; if (w == 0) w0 = (unsigned)v; }
          if (ok) break;
        }
        atomicMax(&s_best, (u64)0 + ((w0 & 0xffffff00u) | (unsigned)c) );
      }
      __syncthreads();
      if (tid < 12) put(dec + pb * 16 + tid, tag, s_best & 0xffu);
      if (tid == 0) s_win = s_best & 0xffu;
    } else {
      if (tid < 12) {
        u64 v;
        do { v = get(dec + pb * 16 + tid); } while ((unsigned)(v >> 32) != tag);
        if (tid == 0) s_win = (unsigned)v;
      }
    }
    __syncthreads();
    const unsigned w = s_win;
    if (tid == 0) s_acc = 0;
    __syncthreads();
    atomicAdd(&s_acc, fetch_vec(vec + ((size_t)pb * G + w) * 2 * P, tag));
    __syncthreads();
    checksum = checksum * 31 + w + s_acc;
    __syncthreads();
  }
  if (tid == 0) { chk[cta] = checksum; if (cta == 0) out[0] = clock64() - t0; }
}

// hierarchical: leader publishes (key|slot, cta) ; every CTA polls all leader records
template <int CS, bool MB>
__global__ void k_hier(u64* lrec, u64* vec, int steps, long long* out, unsigned* chk) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int NC = G / CS;
  const unsigned crank = cluster_rank();
  const int cid = cta / CS;
  __shared__ __align__(8) u64 slots[CS];
  __shared__ __align__(8) u64 mbar;
  __shared__ u64 s_red[8];
  __shared__ unsigned s_win, s_acc;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(CS));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  unsigned checksum = 0;
  long long t0 = clock64();
  for (int s = 1; s <= steps; ++s) {
    const unsigned tag = s;
    const int pb = s & 1;
    const unsigned key = hsh(cta * 977 + s * 131);
    publish_vec(vec + ((size_t)pb * G + cta) * 2 * P, tag, cta);
    const u64 packed = ((u64)(key & 0xffffff00u) << 32) | (unsigned)cta;
    if (MB) {
      if (tid == 0) {
        const unsigned la = smem_u32(&slots[crank]);
        const unsigned ra = mapa(la, 0);
        const unsigned rb = mapa(smem_u32(&mbar), 0);
        asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(packed) : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
      }
      if (crank == 0 && tid == 0) {
        const unsigned par = (s - 1) & 1;
        unsigned done = 0;
        while (!done) {
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                       : "=r"(done) : "r"(smem_u32(&mbar)), "r"(par) : "memory");
        }
        u64 best = 0;
        for (int i = 0; i < CS; ++i) { u64 v = *(volatile u64*)&slots[i]; best = v > best ? v : best; }
        u64* q = lrec + ((size_t)pb * NC + cid) * 4;
        put(q, tag, (unsigned)(best >> 32));
        put(q + 1, tag, (unsigned)best);
      }
    } else {  // cluster barrier variant
      if (tid == 0) {
        const unsigned ra = mapa(smem_u32(&slots[crank]), 0);
        asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(packed) : "memory");
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      if (crank == 0 && tid == 0) {
        u64 best = 0;
        for (int i = 0; i < CS; ++i) { u64 v = slots[i]; best = v > best ? v : best; }
        u64* q = lrec + ((size_t)pb * NC + cid) * 4;
        put(q, tag, (unsigned)(best >> 32));
        put(q + 1, tag, (unsigned)best);
      }
    }
    // every CTA: poll all NC leader records
    u64 mine = 0;
    for (int c = tid; c < NC; c += blockDim.x) {
      const u64* q = lrec + ((size_t)pb * NC + c) * 4;
      u64 a, b;
      do { a = get(q); b = get(q + 1); } while ((unsigned)(a >> 32) != tag || (unsigned)(b >> 32) != tag);
      mine = ((u64)(unsigned)a << 32) | (unsigned)b;
    }
    if (tid < 32 * ((NC + 31) / 32)) {
      for (int off = 16; off > 0; off >>= 1) { u64 o = __shfl_xor_sync(0xffffffffu, mine, off); mine = o > mine ? o : mine; }
      if ((tid & 31) == 0) s_red[tid >> 5] = mine;
    }
    __syncthreads();
    if (tid == 0) {
      u64 b = 0;
      for (int w = 0; w < (NC + 31) / 32; ++w) b = s_red[w] > b ? s_red[w] : b;
      s_win = (unsigned)b;
      s_acc = 0;
    }
    __syncthreads();
    const unsigned w = s_win;
    atomicAdd(&s_acc, fetch_vec(vec + ((size_t)pb * G + w) * 2 * P, tag));
    __syncthreads();
    checksum = checksum * 31 + w + s_acc;
  }
  if (tid == 0) { chk[cta] = checksum; if (cta == 0) out[0] = clock64() - t0; }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}


// push reducer: CTA c writes its record to slot c (reducer thread c polls it); the reducer pushes
// the 4-word decision into every CTA's private mailbox line (one poller per CTA, no hot line).
template <bool VEC, bool WARPRED>
__global__ void k_push(u64* rec, u64* mbox, u64* vec, int steps, long long* out, unsigned* chk) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  __shared__ unsigned s_win, s_acc;
  __shared__ u64 s_red[8];
  unsigned checksum = 0;
  long long t0 = clock64();
  for (int s = 1; s <= steps; ++s) {
    const unsigned tag = s;
    const int pb = s & 1;
    const unsigned key = hsh(cta * 977 + s * 131);
    if (VEC) publish_vec(vec + ((size_t)pb * G + cta) * 2 * P, tag, cta);
    if (tid == 0) {
      u64* q = rec + ((size_t)pb * G + cta) * 16;
      put(q, tag, key);
      put(q + 1, tag, cta);
    }
    if (cta == 0) {
      u64 mine = 0;
      if (tid < G) {
        const u64* q = rec + ((size_t)pb * G + tid) * 16;
        u64 a, b;
        do { a = get(q); b = get(q + 1); } while ((unsigned)(a >> 32) != tag || (unsigned)(b >> 32) != tag);
        mine = ((u64)((unsigned)a & 0xffffff00u) << 32) | (unsigned)b;
      }
      for (int off = 16; off > 0; off >>= 1) { u64 o = __shfl_xor_sync(0xffffffffu, mine, off); mine = o > mine ? o : mine; }
      if ((tid & 31) == 0) s_red[tid >> 5] = mine;
      __syncthreads();
      u64 b = 0;
      for (int w = 0; w < 8; ++w) b = s_red[w] > b ? s_red[w] : b;
      for (int c = tid; c < G; c += blockDim.x) {
        u64* m = mbox + ((size_t)pb * G + c) * 16;
        put(m, tag, (unsigned)b);
        put(m + 1, tag, (unsigned)(b >> 32));
      }
      if (tid == 0) s_win = (unsigned)b;
    } else {
      if (tid == 0) {
        const u64* m = mbox + ((size_t)pb * G + cta) * 16;
        u64 a, b2;
        do { a = get(m); b2 = get(m + 1); } while ((unsigned)(a >> 32) != tag || (unsigned)(b2 >> 32) != tag);
        s_win = (unsigned)a;
      }
    }
    __syncthreads();
    const unsigned w = s_win;
    unsigned acc = 0;
    if (VEC) {
      if (tid == 0) s_acc = 0;
      __syncthreads();
      atomicAdd(&s_acc, fetch_vec(vec + ((size_t)pb * G + w) * 2 * P, tag));
      __syncthreads();
      acc = s_acc;
    }
    checksum = checksum * 31 + w + acc;
  }
  if (tid == 0) { chk[cta] = checksum; if (cta == 0) out[0] = clock64() - t0; }
}

__global__ void k_pingpong(u64* rec, u64* mbox, u64* vec, int steps, long long* out, unsigned* chk) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  for (int s = 1; s <= steps; ++s) {
    const unsigned tag = s; const int pb = s & 1;
    if (tid == 0) {
      if (cta == 0) { put(mbox + pb * 16, tag, s); while ((unsigned)(get(mbox + 64 + pb * 16) >> 32) != tag) {} }
      else if (cta == G - 1) { while ((unsigned)(get(mbox + pb * 16) >> 32) != tag) {} put(mbox + 64 + pb * 16, tag, s); }
    }
  }
  if (tid == 0) chk[cta] = 0;
}


// minimal: one warp per CTA, 1-word records, no __syncthreads (G <= 32)
template <int MODE>
__global__ void k_min(u64* rec, u64* mbox, u64* vec, int steps, long long* out, unsigned* chk) {
  const int G = gridDim.x, cta = blockIdx.x, lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  unsigned checksum = 0;
  for (int s = 1; s <= steps; ++s) {
    const unsigned tag = s; const int pb = s & 1;
    const unsigned key = hsh(cta * 977 + s * 131) & 0xffffff00u;
    if (lane == 0) put(rec + ((size_t)pb * G + cta) * 16, tag, key | cta);
    unsigned win;
    if (cta == 0) {
      unsigned mine = 0;
      if (lane < G) {
        u64 a;
        do { a = get(rec + ((size_t)pb * G + lane) * 16); } while ((unsigned)(a >> 32) != tag);
        mine = (unsigned)a;
      }
      for (int off = 16; off > 0; off >>= 1) mine = max(mine, __shfl_xor_sync(0xffffffffu, mine, off));
      win = mine;
      if (lane < G) put(mbox + ((size_t)pb * G + lane) * 16, tag, win);
    } else {
      u64 a = 0;
      if (lane == 0) { do { a = get(mbox + ((size_t)pb * G + cta) * 16); } while ((unsigned)(a >> 32) != tag); }
      win = __shfl_sync(0xffffffffu, (unsigned)a, 0);
    }
    checksum = checksum * 31 + win;
  }
  if (lane == 0) chk[cta] = checksum;
}


// variants of the minimal protocol with 256-thread CTAs (G <= 32):
//  MODE 0: workers: thread 0 polls mailbox, then __syncthreads; reducer warp 0 only (no barrier)
//  MODE 1: MODE 0 + __syncthreads right after the record put (workers and reducer)
//  MODE 2: MODE 0 + reducer uses a __syncthreads between reduce and push
template <int MODE>
__global__ void k_var(u64* rec, u64* mbox, u64* vec, int steps, long long* out, unsigned* chk) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  __shared__ unsigned s_win;
  unsigned checksum = 0;
  for (int s = 1; s <= steps; ++s) {
    const unsigned tag = s; const int pb = s & 1;
    const unsigned key = hsh(cta * 977 + s * 131) & 0xffffff00u;
    if (tid == 0) put(rec + ((size_t)pb * G + cta) * 16, tag, key | cta);
    if (MODE == 1) __syncthreads();
    if (cta == 0) {
      if (tid < 32) {
        unsigned mine = 0;
        if (lane < G) {
          u64 a;
          do { a = get(rec + ((size_t)pb * G + lane) * 16); } while ((unsigned)(a >> 32) != tag);
          mine = (unsigned)a;
        }
        for (int off = 16; off > 0; off >>= 1) mine = max(mine, __shfl_xor_sync(0xffffffffu, mine, off));
        if (lane == 0) s_win = mine;
        if (MODE != 2 && lane < G) put(mbox + ((size_t)pb * G + lane) * 16, tag, mine);
      }
      if (MODE == 2) {
        __syncthreads();
        if (tid < G) put(mbox + ((size_t)pb * G + tid) * 16, tag, s_win);
      }
    } else {
      if (tid == 0) {
        u64 a;
        do { a = get(mbox + ((size_t)pb * G + cta) * 16); } while ((unsigned)(a >> 32) != tag);
        s_win = (unsigned)a;
      }
    }
    __syncthreads();
    checksum = checksum * 31 + s_win;
    __syncthreads();
  }
  if (tid == 0) chk[cta] = checksum;
}


// generalized var1 (barrier after the record put), G <= 256, optional winner-vector fetch;
// FENCE: use __threadfence() after the put instead of the barrier
template <bool VEC, int POST>
__global__ void k_gen(u64* rec, u64* mbox, u64* vec, int steps, long long* out, unsigned* chk) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  __shared__ unsigned s_win, s_best, s_acc;
  unsigned checksum = 0;
  if (tid == 0) s_best = 0;
  for (int s = 1; s <= steps; ++s) {
    const unsigned tag = s; const int pb = s & 1;
    const unsigned key = hsh(cta * 977 + s * 131) & 0xffffff00u;
    if (VEC) publish_vec(vec + ((size_t)pb * G + cta) * 2 * P, tag, cta);
    if (tid == 0) put(rec + ((size_t)pb * G + cta) * 16, tag, key | cta);
    if (POST == 0) __syncthreads();
    if (POST == 1 && tid == 0) __threadfence();
    if (cta == 0) {
      unsigned mine = 0;
      if (tid < G) {
        u64 a;
        do { a = get(rec + ((size_t)pb * G + tid) * 16); } while ((unsigned)(a >> 32) != tag);
        mine = (unsigned)a;
      }
      for (int off = 16; off > 0; off >>= 1) mine = max(mine, __shfl_xor_sync(0xffffffffu, mine, off));
      if (lane == 0 && tid < G) atomicMax(&s_best, mine);
      __syncthreads();
      const unsigned w = s_best;
      if (tid < G) put(mbox + ((size_t)pb * G + tid) * 16, tag, w);
      if (tid == 0) s_win = w;
    } else {
      if (tid == 0) {
        u64 a;
        do { a = get(mbox + ((size_t)pb * G + cta) * 16); } while ((unsigned)(a >> 32) != tag);
        s_win = (unsigned)a;
      }
    }
    __syncthreads();
    const unsigned w = s_win & 0xffu;
    if (tid == 0) { s_best = 0; s_acc = 0; }
    unsigned acc = 0;
    if (VEC) {
      __syncthreads();
      atomicAdd(&s_acc, fetch_vec(vec + ((size_t)pb * G + w) * 2 * P, tag));
      __syncthreads();
      acc = s_acc;
    }
    checksum = checksum * 31 + s_win + acc;
    __syncthreads();
  }
  if (tid == 0) chk[cta] = checksum;
}

static void coop(const char* name, void* fn, int G, u64* a, u64* b, u64* c, int steps, long long* out, unsigned* chk) {
  cudaMemset(a, 0, 1 << 20); cudaMemset(b, 0, 1 << 20); cudaMemset(c, 0, 8 << 20);
  int st = steps;
  void* args[] = {&a, &b, &c, &st, &out, &chk};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t e = cudaLaunchCooperativeKernel(fn, G, 256, args, 0, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned h[256]; cudaMemcpy(h, chk, sizeof(unsigned) * G, cudaMemcpyDeviceToHost);
  bool agree = true; for (int i = 1; i < G; ++i) agree &= h[i] == h[0];
  printf("%-12s G=%3d %s agree=%d %.3f us/step\n", name, G, cudaGetErrorString(e), agree, ms * 1e3 / steps);
}

template <class K>
static void run(const char* name, K kern, int G, int CS, bool coop, u64* a, u64* b, u64* c, int steps, long long* out,
                unsigned* chk) {
  cudaMemset(a, 0, 1 << 20); cudaMemset(b, 0, 1 << 20); cudaMemset(c, 0, 8 << 20);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 0; cfg.stream = 0;
  cudaLaunchAttribute at[2]; int na = 0;
  if (CS > 1) { at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim.x = CS; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1; ++na; }
  if (coop) { at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na; }
  cfg.attrs = at; cfg.numAttrs = na;
  int ncl = -1;
  if (CS > 1) cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg);
  if (CS > 1 && ncl * CS < G) { printf("%-12s G=%3d CS=%2d: only %d clusters fit, skipped\n", name, G, CS, ncl); return; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t e;
  if (CS > 1 || coop) e = cudaLaunchKernelEx(&cfg, kern, a, c, steps, out, chk);
  else e = cudaErrorInvalidValue;
  cudaEventRecord(e1);
  cudaError_t e2 = cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  unsigned h[256]; cudaMemcpy(h, chk, sizeof(unsigned) * G, cudaMemcpyDeviceToHost);
  bool agree = true; for (int i = 1; i < G; ++i) agree &= h[i] == h[0];
  printf("%-12s G=%3d CS=%2d coop=%d maxClusters=%3d launch=%s sync=%s agree=%d  %.3f us/step\n", name, G, CS, coop, ncl,
         cudaGetErrorString(e), cudaGetErrorString(e2), agree, ms * 1e3 / steps);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  u64 *a, *b, *c; long long* out; unsigned* chk;
  cudaMalloc(&a, 1 << 20); cudaMalloc(&b, 1 << 20); cudaMalloc(&c, 8 << 20); cudaMalloc(&out, 64); cudaMalloc(&chk, 4096);
  const int steps = 20000;
  for (int G : {sms, 128}) {
    // reducer with cooperative launch
    {
      cudaMemset(a, 0, 1 << 20); cudaMemset(b, 0, 1 << 20); cudaMemset(c, 0, 8 << 20);
      void* args[] = {&a, &b, &c, (void*)&steps, &out, &chk};
      int st = steps; args[3] = &st;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchCooperativeKernel((void*)k_reducer, G, 256, args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      unsigned h[256]; cudaMemcpy(h, chk, sizeof(unsigned) * G, cudaMemcpyDeviceToHost);
      bool agree = true; for (int i = 1; i < G; ++i) agree &= h[i] == h[0];
      printf("%-12s G=%3d %s agree=%d %.3f us/step\n", "reducer", G, cudaGetErrorString(e), agree, ms * 1e3 / steps);
    }
  }
  coop("pingpong", (void*)k_pingpong, 148, a, b, c, steps, out, chk);
  for (int g : {2, 32}) coop("min", (void*)k_min<0>, g, a, b, c, steps, out, chk);
  for (int g : {2, 32}) coop("var0", (void*)k_var<0>, g, a, b, c, steps, out, chk);
  for (int g : {2, 32, 148}) coop("gen-bar", (void*)k_gen<false, 0>, g, a, b, c, steps, out, chk);
  for (int g : {2, 32, 148}) coop("gen-fence", (void*)k_gen<false, 1>, g, a, b, c, steps, out, chk);
  for (int g : {2, 32, 148}) coop("gen-none", (void*)k_gen<false, 2>, g, a, b, c, steps, out, chk);
  for (int g : {32, 148}) coop("gen-bar+vec", (void*)k_gen<true, 0>, g, a, b, c, steps, out, chk);
  for (int g : {2, 32}) coop("var1-barafterput", (void*)k_var<1>, g, a, b, c, steps, out, chk);
  for (int g : {2, 32}) coop("var2-redbar", (void*)k_var<2>, g, a, b, c, steps, out, chk);
  coop("push+vec", (void*)k_push<true, true>, 148, a, b, c, steps, out, chk);
  coop("push", (void*)k_push<false, true>, 148, a, b, c, steps, out, chk);
  coop("push+vec", (void*)k_push<true, true>, 128, a, b, c, steps, out, chk);
  if (0) { bool coop = true;
    run("hier2-mb", k_hier<2, true>, 148, 2, coop, a, b, c, steps, out, chk);
    run("hier4-mb", k_hier<4, true>, 128, 4, coop, a, b, c, steps, out, chk);
    run("hier4-mb", k_hier<4, true>, 144, 4, coop, a, b, c, steps, out, chk);
    run("hier8-mb", k_hier<8, true>, 128, 8, coop, a, b, c, steps, out, chk);
    run("hier8-bar", k_hier<8, false>, 128, 8, coop, a, b, c, steps, out, chk);
    run("hier4-bar", k_hier<4, false>, 128, 4, coop, a, b, c, steps, out, chk);
  }
  cudaError_t e = cudaGetLastError();
  printf("last error: %s\n", cudaGetErrorString(e));
  return 0;
}
