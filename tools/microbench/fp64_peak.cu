// FP64 microbenchmarks for B200 (sm_100a): DFMA peak, DMMA (mma.sync m8n8k4 f64) peak,
// and a software grid-barrier round trip.  Used to pick the Schur-update inner loop
// and to put a measured FP64 denominator next to MEASURED_PEAKS.json (which has none).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;

__device__ __forceinline__ void grid_barrier(unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int gen = g_gen;
    __threadfence();
    unsigned int arrived = atomicAdd(&g_count, 1);
    if (arrived == nblocks - 1) {
      g_count = 0;
      __threadfence();
      g_gen = gen + 1;
    } else {
      while (g_gen == gen) { }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void barrier_kernel(int iters, unsigned long long* cycles) {
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) grid_barrier(gridDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) cycles[0] = clock64() - t0;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d clock(kHz) %d\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  double* d; CK(cudaMalloc(&d, 8));
  unsigned long long* cyc; CK(cudaMalloc(&cyc, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = prop.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 20000, threads = 256, blocks = sms * 8;
    dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0)); dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 16 * iters * (double)threads * blocks;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flop / ms / 1e9, ms);
    int it2 = 20000;
    dmma_kernel<<<blocks, threads>>>(d, it2);
    CK(cudaEventRecord(e0)); dmma_kernel<<<blocks, threads>>>(d, it2); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flop2 = 2.0 * 256 * 8 * (double)it2 * (threads / 32) * blocks;
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flop2 / ms / 1e9, ms);
  }
  for (int bthreads : {256, 512}) {
    int iters = 10000;
    void* args[] = {&iters, &cyc};
    CK(cudaLaunchCooperativeKernel((void*)barrier_kernel, sms, bthreads, args, 0, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    CK(cudaLaunchCooperativeKernel((void*)barrier_kernel, sms, bthreads, args, 0, 0));
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("grid barrier (%d CTAs x %d thr): %.3f us per barrier\n", sms, bthreads, ms * 1e3 / iters);
  }
  return 0;
}
