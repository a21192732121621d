// Does cuTensorMapEncodeTiled accept the 3-D "chunk-major" view of a K-contiguous fp64 operand
// panel (dims {4, rows, tpad/4}, strides {tpad*8, 32} bytes: the third stride is smaller than the second)?
// And does a 3-D TMA box {4,128,4} land in shared memory as [chunk][row][4]?
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int row0, int kc0) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* s = reinterpret_cast<double*>(raw);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(raw + 16384);
  unsigned sb = (unsigned)__cvta_generic_to_shared(bar), sd = (unsigned)__cvta_generic_to_shared(s);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(16384) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(sd), "l"(&tm), "r"(0), "r"(row0), "r"(kc0), "r"(sb) : "memory");
  }
  unsigned ok = 0;
  while (!ok) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(sb) : "memory");
  }
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = s[i];
}
int main() {
  const int rows = 256, tpad = 144;
  double* d; cudaMalloc(&d, rows * tpad * 8);
  double* h = new double[rows * tpad];
  for (int r = 0; r < rows; ++r) for (int c = 0; c < tpad; ++c) h[r * tpad + c] = r * 1000 + c;
  cudaMemcpy(d, h, rows * tpad * 8, cudaMemcpyHostToDevice);
  EncodeTiled enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no entry point\n"); return 1; }
  CUtensorMap tm;
  cuuint64_t dims[3] = {4, (cuuint64_t)rows, (cuuint64_t)tpad / 4};
  cuuint64_t str[2] = {(cuuint64_t)tpad * 8, 32};
  cuuint32_t box[3] = {4, 128, 4}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode 3D chunk-major: CUresult %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 2;
  double* o; cudaMalloc(&o, 2048 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 64);
  k<<<1, 128, 16384 + 64>>>(tm, o, 128, 4);  // rows 128..255 (row 255 valid), k = 16..31
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double ho[2048]; cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int c = 0; c < 4; ++c) for (int rr = 0; rr < 128; ++rr) for (int x = 0; x < 4; ++x) {
    double want = (128 + rr) * 1000 + 16 + 4 * c + x;
    if (ho[c * 512 + rr * 4 + x] != want) { if (bad < 5) printf("mismatch c%d r%d x%d got %g want %g\n", c, rr, x, ho[c * 512 + rr * 4 + x], want); ++bad; }
  }
  printf("layout [chunk][row][4]: %s (%d mismatches)\n", bad ? "NO" : "yes", bad);
  return 0;
}
