// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// FP32 FFMA, FP64 DFMA (register and constant-bank operand forms) and a
// plain streaming copy / read bandwidth with this repo's own kernels.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__constant__ float cF[64];
__constant__ double cD[64];

template <typename T, int ACC>
__global__ void fma_reg(T* out, T a, T b, int iters) {
  T acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = acc[i] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += acc[i];
  if (s == (T)-1.2345) out[threadIdx.x] = s;
}

// constant-bank operand: acc[i] = acc[i]*x[i] + c[k]; the multiplier comes from c[]
template <typename T, int ACC>
__global__ void fma_const(T* out, int iters) {
  const T* C;
  if (sizeof(T) == 4) C = (const T*)cF; else C = (const T*)cD;
  T acc[ACC], x[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { acc[i] = (T)(threadIdx.x + i); x[i] = (T)1.0001 + (T)i * (T)1e-6; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
#pragma unroll
      for (int i = 0; i < ACC; ++i) acc[i] = fma(x[i], C[k], acc[i]);
    }
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += acc[i];
  if (s == (T)-1.2345) out[threadIdx.x] = s;
}

__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void read4(const float4* __restrict__ a, float* out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  float s = 0;
  for (; i < n; i += st) { float4 v = a[i]; s += v.x + v.y + v.z + v.w; }
  if (s == -1.f) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d", p.name, p.multiProcessorCount, clk);
  float hf[64]; double hd[64];
  for (int i = 0; i < 64; ++i) { hf[i] = 0.999f + i * 1e-6f; hd[i] = 0.999 + i * 1e-9; }
  CK(cudaMemcpyToSymbol(cF, hf, sizeof(hf))); CK(cudaMemcpyToSymbol(cD, hd, sizeof(hd)));
  float* of; double* od; CK(cudaMalloc(&of, 4096)); CK(cudaMalloc(&od, 8192));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256;
  auto run = [&](const char* name, auto launch, double flops) {
    for (int w = 0; w < 3; ++w) launch();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf(",\"%s_tflops\":%.2f", name, flops / (best * 1e-3) / 1e12);
  };
  int it = 4096;
  double nthr = (double)blocks * threads;
  run("ffma_reg", [&] { fma_reg<float, 16><<<blocks, threads>>>(of, 0.9999f, 1e-7f, it); }, 2.0 * 16 * it * nthr);
  run("dfma_reg", [&] { fma_reg<double, 16><<<blocks, threads>>>(od, 0.9999, 1e-7, it / 4); }, 2.0 * 16 * (it / 4) * nthr);
  run("ffma_const", [&] { fma_const<float, 16><<<blocks, threads>>>(of, it / 32); }, 2.0 * 16 * 32 * (it / 32) * nthr);
  run("dfma_const", [&] { fma_const<double, 16><<<blocks, threads>>>(od, it / 128); }, 2.0 * 16 * 32 * (it / 128) * nthr);
  size_t bytes = (size_t)2 << 30; size_t n4 = bytes / 16;
  float4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  cudaMemset(a, 0, bytes); cudaMemset(b, 0, bytes);
  auto runbw = [&](const char* name, auto launch, double by) {
    for (int w = 0; w < 3; ++w) launch();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf(",\"%s_gbs\":%.1f", name, by / (best * 1e-3) / 1e9);
  };
  runbw("copy", [&] { copy4<<<p.multiProcessorCount * 16, 512>>>(a, b, n4); }, 2.0 * bytes);
  runbw("read", [&] { read4<<<p.multiProcessorCount * 16, 512>>>(a, of, n4); }, 1.0 * bytes);
  CK(cudaDeviceSynchronize());
  printf("}\n");
  return 0;
}
