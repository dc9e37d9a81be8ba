// Do the fp64 tensor path (DMMA, mma.sync m8n8k4) and the fp64 FMA pipe (DFMA) run concurrently
// on sm_100a?  Three kernels, same grid (148 x 4 CTAs x 256 threads), CUDA-event timed (warm run):
//   dmma  : every warp issues 8 independent DMMA chains
//   dfma  : every warp issues 16 independent DFMA chains
//   mixed : even warps DMMA, odd warps DFMA (the same per-warp loops)
// If the mixed aggregate TFLOP/s is near dmma + dfma, a kernel could split its contractions
// across the two pipes; if it is near either alone, they share the fp64 datapath.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma_loop(double* out, int iters) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 1.2345) out[0] = s;
}
__device__ __forceinline__ void dfma_loop(double* out, int iters) {
  double c[16];
  for (int k = 0; k < 16; ++k) c[k] = threadIdx.x * 1e-3 + k;
  const double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 16; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;\n" : "+d"(c[k]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 16; ++k) s += c[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dmma(double* o, int it) { dmma_loop(o, it); }
__global__ void k_dfma(double* o, int it) { dfma_loop(o, it); }
__global__ void k_mixed(double* o, int it_mma, int it_fma) {
  if ((threadIdx.x >> 5) & 1) dfma_loop(o, it_fma);
  else dmma_loop(o, it_mma);
}

int main() {
  double* od;
  cudaMalloc(&od, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 4, threads = 256, warps = blocks * threads / 32;
  const int it_mma = 500, it_fma = 200;
  const double f_mma = 2.0 * 8 * 8 * 4 * 8.0 * it_mma;  // per warp
  const double f_fma = 2.0 * 32 * 16 * 16.0 * it_fma;   // per warp
  float ms;
  for (int r = 0; r < 2; ++r) {
    k_dmma<<<blocks, threads>>>(od, 5);
    cudaEventRecord(e0); k_dmma<<<blocks, threads>>>(od, it_mma); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double t_mma = ms;
    printf("dmma  : %.1f TFLOP/s (%.3f ms)\n", f_mma * warps / ms / 1e9, ms);
    k_dfma<<<blocks, threads>>>(od, 5);
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(od, it_fma); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double t_fma = ms;
    printf("dfma  : %.1f TFLOP/s (%.3f ms)\n", f_fma * warps / ms / 1e9, ms);
    // mixed: size the two halves so that each alone would take about the same time
    const int it_f = (int)(it_fma * t_mma / t_fma);
    k_mixed<<<blocks, threads>>>(od, 5, 5);
    cudaEventRecord(e0); k_mixed<<<blocks, threads>>>(od, it_mma, it_f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (f_mma + 2.0 * 32 * 16 * 16.0 * it_f) * (warps / 2);
    printf("mixed : %.1f TFLOP/s (%.3f ms; half the warps each; alone each half ~%.3f ms)\n", fl / ms / 1e9, ms,
           0.5 * t_mma);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
