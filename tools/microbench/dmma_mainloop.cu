// DMMA mainloop throughput vs warps/SM and fragment-load pattern (B200, sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// MODE 0: LDS fragments (8 A + 4 B per k-step) + 32 DMMA; MODE 1: registers only (no LDS)
template <int MODE, int MF, int NF>
__global__ void mainloop(double* out, int iters) {
  __shared__ double a[64][20], b[64][20];
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) { (&a[0][0])[i] = i * 1e-3; (&b[0][0])[i] = 1.0 - i * 1e-4; }
  __syncthreads();
  double acc[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  double af[MF], bf[NF];
#pragma unroll
  for (int i = 0; i < MF; ++i) af[i] = a[8 * i + g][q];
#pragma unroll
  for (int j = 0; j < NF; ++j) bf[j] = b[8 * j + g][q];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < MF; ++i) af[i] = a[8 * i + g][kk + q];
#pragma unroll
        for (int j = 0; j < NF; ++j) bf[j] = b[8 * j + g][kk + q];
      }
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1.2345) out[0] = s;
}
template <int MODE, int MF, int NF>
void run(const char* name, int threads, int blocks_per_sm, int sms, double* d) {
  int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  mainloop<MODE, MF, NF><<<sms * blocks_per_sm, threads>>>(d, 10);
  cudaEventRecord(e0);
  mainloop<MODE, MF, NF><<<sms * blocks_per_sm, threads>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flop = 2.0 * 256 * MF * NF * 4 * (double)iters * (threads / 32) * sms * blocks_per_sm;
  printf("%-34s thr=%3d cta/SM=%d warps/SM=%2d : %6.2f TFLOP/s  (%s)\n", name, threads, blocks_per_sm,
         threads / 32 * blocks_per_sm, flop / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  run<0, 8, 4>("LDS+DMMA 64x32 warp tile", 128, 2, sms, d);
  run<1, 8, 4>("regs-only DMMA 64x32", 128, 2, sms, d);
  run<0, 8, 4>("LDS+DMMA 64x32 warp tile", 256, 1, sms, d);
  run<0, 8, 4>("LDS+DMMA 64x32 warp tile", 128, 1, sms, d);
  run<1, 8, 4>("regs-only DMMA 64x32", 128, 1, sms, d);
  run<0, 8, 4>("LDS+DMMA 64x32 warp tile", 256, 2, sms, d);
  run<0, 4, 4>("LDS+DMMA 32x32 warp tile", 128, 4, sms, d);
  run<0, 4, 8>("LDS+DMMA 32x64 warp tile", 256, 2, sms, d);
  return 0;
}
