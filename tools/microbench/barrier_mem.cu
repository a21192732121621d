// Does __syncthreads wait for outstanding global stores / loads?  Cycles per iteration of
// {memory op by every thread; __syncthreads} on one CTA of 256 threads (B200).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* g, long long* out, int iters) {
  const int tid = threadIdx.x;
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1) g[(size_t)it * 256 + tid] = (double)it;            // store, then barrier
    if (MODE == 2) acc += __ldcg(g + (size_t)((it * 7919) % 4096) * 256 + tid);  // load (result used late), then barrier
    if (MODE == 3) { g[(size_t)it * 256 + tid] = (double)it; __threadfence_block(); }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[MODE] = (t1 - t0) / iters;
  if (acc == 1.2345) g[0] = acc;
}
int main() {
  double* g; long long* out; cudaMalloc(&g, 8ull << 20 << 4); cudaMalloc(&out, 64);
  cudaMemset(g, 0, 8ull << 20 << 4);
  long long h[4];
  k<0><<<1, 256>>>(g, out, 4096); k<1><<<1, 256>>>(g, out, 4096); k<2><<<1, 256>>>(g, out, 4096); k<3><<<1, 256>>>(g, out, 4096);
  cudaDeviceSynchronize();
  k<0><<<1, 256>>>(g, out, 4096); k<1><<<1, 256>>>(g, out, 4096); k<2><<<1, 256>>>(g, out, 4096); k<3><<<1, 256>>>(g, out, 4096);
  cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
  printf("cycles/iter: barrier only %lld, store+barrier %lld, load(unused)+barrier %lld, store+fence.cta+barrier %lld\n", h[0], h[1], h[2], h[3]);
  return 0;
}
