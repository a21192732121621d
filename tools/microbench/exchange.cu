// Microbenchmark of grid-wide exchange patterns on B200 (one CTA per SM, cooperative launch):
//  a2a   : every CTA writes a 12-word LL record, every CTA reads all G records (current panel scheme)
//  a2a1  : same, but readers spin on one word before loading the rest
//  red   : every CTA writes its record; CTA 0 reads all, reduces, writes one decision; all read it
//  pp    : ping-pong latency between CTA 0 and CTA G-1
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ void put(u64* p, unsigned tag, unsigned d) {
  u64 v = ((u64)tag << 32) | d;
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 get(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <int MODE>
__global__ void kern(u64* rec, u64* dec, int steps, long long* out) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  __shared__ unsigned s_best;
  long long t0 = clock64();
  for (int s = 1; s <= steps; ++s) {
    const unsigned tag = s;
    const int pb = s & 1;
    if (MODE == 3) {  // ping-pong CTA 0 <-> CTA G-1
      if (tid == 0) {
        if (cta == 0) {
          put(dec + pb * 16, tag, s);
          while ((unsigned)(get(dec + 64 + pb * 16) >> 32) != tag) {}
        } else if (cta == G - 1) {
          while ((unsigned)(get(dec + pb * 16) >> 32) != tag) {}
          put(dec + 64 + pb * 16, tag, s);
        }
      }
      continue;
    }
    if (tid == 0) {
      u64* q = rec + ((size_t)pb * G + cta) * 16;
      for (int w = 0; w < 12; ++w) put(q + w, tag, cta * 7 + s + w);
    }
    if (MODE == 0 || MODE == 1) {
      unsigned best = 0;
      for (int c = tid; c < G; c += blockDim.x) {
        const u64* q = rec + ((size_t)pb * G + c) * 16;
        if (MODE == 1) while ((unsigned)(get(q) >> 32) != tag) {}
        while (true) {
          bool ok = true;
          unsigned acc = 0;
          for (int w = 0; w < 12; ++w) { u64 v = get(q + w); ok &= (unsigned)(v >> 32) == tag; acc += (unsigned)v; }
          if (ok) { best = max(best, acc); break; }
        }
      }
      if (tid == 0) s_best = 0;
      __syncthreads();
      atomicMax(&s_best, best);
      __syncthreads();
    } else {  // MODE 2: reducer
      if (cta == 0) {
        unsigned best = 0;
        for (int c = tid; c < G; c += blockDim.x) {
          const u64* q = rec + ((size_t)pb * G + c) * 16;
          while ((unsigned)(get(q) >> 32) != tag) {}
          while (true) {
            bool ok = true;
            unsigned acc = 0;
            for (int w = 0; w < 12; ++w) { u64 v = get(q + w); ok &= (unsigned)(v >> 32) == tag; acc += (unsigned)v; }
            if (ok) { best = max(best, acc); break; }
          }
        }
        if (tid == 0) s_best = 0;
        __syncthreads();
        atomicMax(&s_best, best);
        __syncthreads();
        if (tid < 12) put(dec + pb * 16 + tid, tag, s_best + tid);
      } else {
        if (tid < 12) {
          while ((unsigned)(get(dec + pb * 16 + tid) >> 32) != tag) {}
        }
        __syncthreads();
      }
    }
  }
  if (cta == 0 && tid == 0) out[MODE] = clock64() - t0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  u64 *rec, *dec; long long* out;
  cudaMalloc(&rec, 2 * 160 * 16 * 8); cudaMalloc(&dec, 256 * 8); cudaMalloc(&out, 64);
  int steps = 4000;
  void* fns[4] = {(void*)kern<0>, (void*)kern<1>, (void*)kern<2>, (void*)kern<3>};
  const char* names[4] = {"a2a", "a2a-poll1", "reducer", "pingpong"};
  for (int G : {sms, 74, 32}) {
    for (int m = 0; m < 4; ++m) {
      cudaMemset(rec, 0, 2 * 160 * 16 * 8); cudaMemset(dec, 0, 256 * 8);
      void* args[] = {&rec, &dec, &steps, &out};
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(fns[m], G, 256, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("G=%3d %-10s %s  %.3f us/step\n", G, names[m], cudaGetErrorString(e), ms * 1e3 / steps);
    }
  }
  return 0;
}
