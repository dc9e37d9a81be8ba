// fp64 pipe throughput vs warps per SM sub-partition (SMSP): DFMA (ACC independent chains per thread,
// register operands, and a broadcast shared-memory operand like the stage kernels' operator rows) and
// DMMA m8n8k4 (8 independent accumulators per warp).  One CTA per SM (grid = #SMs, forced by shared
// memory), W warps per CTA.  Reports TFLOP/s and the fraction of the fp64 datapath (64 FMA/clk/SM).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_occ.cu -o tools/fp64_occ && tools/fp64_occ
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

constexpr int SMEM_FORCE = 150 * 1024;  // one CTA per SM

template <int ACC>
__global__ void dfma_reg(double* out, double a, double b, int iters) {
  extern __shared__ double sm[];
  double acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += acc[i];
  if (s == -1.2345) out[threadIdx.x] = s + sm[0];
}

// the stage kernels' volume pattern: per column j, a field value x_j per lane (LDS, lane-varying) and
// R operator rows broadcast (LDS.128 {Dr, Ds}); 4 FMAs per (row, column) into u, v, w accumulators
template <int R>
__global__ void dfma_smem(double* out, int iters) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  double* f = sm;                         // [64][32] field values
  double2* op = reinterpret_cast<double2*>(sm + 64 * 32);  // [64][R] operator pairs
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) f[i] = 1.0 + 1e-3 * i;
  for (int i = threadIdx.x; i < 64 * R; i += blockDim.x) op[i] = make_double2(0.5 + 1e-4 * i, 0.25 - 1e-4 * i);
  __syncthreads();
  double u[R], v[R], w[R];
#pragma unroll
  for (int r = 0; r < R; ++r) u[r] = v[r] = w[r] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int j = 0; j < 64; ++j) {
      const double ez = f[j * 32 + lane], w1 = f[((j + 7) & 63) * 32 + lane];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double2 d = op[j * R + r];
        u[r] = fma(d.x, ez, u[r]);
        v[r] = fma(d.y, ez, v[r]);
        w[r] = fma(d.x, w1, w[r]);
        w[r] = fma(d.y, ez, w[r]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) s += u[r] + v[r] + w[r];
  if (s == -1.2345) out[threadIdx.x] = s;
}

__global__ void dmma_k(double* out, int iters) {
  extern __shared__ double sm[];
  double c[8][2];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[threadIdx.x] = s + sm[0];
}

// mma.sync m16n8k8 tf32 (the fp32 3xTF32 path's instruction): CH independent accumulators per warp
template <int CH>
__global__ void tf32_k(float* out, int iters) {
  extern __shared__ double sm[];
  float c[CH][4];
  const uint32_t a0 = 0x3f800000u + threadIdx.x, b0 = 0x3f000000u + threadIdx.x;
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a0), "r"(a0 + 1), "r"(a0 + 2), "r"(a0 + 3), "r"(b0), "r"(b0 + 1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345f) out[threadIdx.x] = s + (float)sm[0];
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount;
  double* od;
  CK(cudaMalloc(&od, 1 << 16));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(dfma_reg<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_FORCE));
  CK(cudaFuncSetAttribute(dfma_reg<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_FORCE));
  CK(cudaFuncSetAttribute(dfma_smem<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_FORCE));
  CK(cudaFuncSetAttribute(dmma_k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_FORCE));
  CK(cudaFuncSetAttribute(tf32_k<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_FORCE));
  CK(cudaFuncSetAttribute(tf32_k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_FORCE));
  auto run = [&](const char* name, int warps, auto launch, double flop) {
    for (int w = 0; w < 2; ++w) launch();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double tf = flop / (best * 1e-3) / 1e12;
    const double peak = 2.0 * 64 * sms * clk * 1e3 / 1e12;  // fp64 datapath (tf32 lines: the ratio is vs this too)
    printf("%-22s warps/SM %2d (per SMSP %.1f): %6.2f TFLOP/s  %.2f of 64 FMA/clk/SM at %d MHz\n", name, warps,
           warps / 4.0, tf, tf / peak, clk / 1000);
  };
  for (int w : {4, 8, 12, 16, 24}) {
    const int th = 32 * w, it = 2048;
    run("dfma reg ACC=16", w, [&] { dfma_reg<16><<<sms, th, SMEM_FORCE>>>(od, 0.9999, 1e-7, it); },
        2.0 * 16 * it * (double)th * sms);
    run("dfma reg ACC=8", w, [&] { dfma_reg<8><<<sms, th, SMEM_FORCE>>>(od, 0.9999, 1e-7, it); },
        2.0 * 8 * it * (double)th * sms);
    run("dfma smem R=6", w, [&] { dfma_smem<6><<<sms, th, SMEM_FORCE>>>(od, 64); },
        2.0 * 64 * 6 * 4 * 64 * (double)th * sms);
    run("dmma x8 chains", w, [&] { dmma_k<<<sms, th, SMEM_FORCE>>>(od, 512); },
        2.0 * 256 * 8 * 512 * (double)(th / 32) * sms);
    run("tf32 mma x9 chains", w, [&] { tf32_k<9><<<sms, th, SMEM_FORCE>>>((float*)od, 1024); },
        2.0 * 1024 * 9 * 1024 * (double)(th / 32) * sms);
    run("tf32 mma x3 chains", w, [&] { tf32_k<3><<<sms, th, SMEM_FORCE>>>((float*)od, 1024); },
        2.0 * 1024 * 3 * 1024 * (double)(th / 32) * sms);
  }
  CK(cudaGetLastError());
  printf("ok\n");
  return 0;
}
