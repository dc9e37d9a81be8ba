// Probe of the tcgen05 encodings the fp32 tensor-core stage kernel relies on (sm_100a):
//   * A operand in TMEM (tcgen05.st.32x32b: warp w, thread t -> lane 32w + t = MMA row),
//   * B operand in shared memory, K-major, no swizzle: 8-row x 16-byte core matrices,
//     SBO = stride between 8-row groups along N, LBO = stride between the two 16-byte K chunks,
//   * tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = 24 / 48, K = 8 per instruction,
//     accumulate flag, D at a column offset, tcgen05.commit -> mbarrier,
//   * D read back with tcgen05.ld.32x32b.
// Checks against a host fp64 product of the tf32-truncated operands, then times back-to-back MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe tools/umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (bits 61-63 = 0)
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4)        // D fp32
       | (2u << 7)        // A tf32
       | (2u << 10)       // B tf32
       | (0u << 15)       // A K-major
       | (0u << 16)       // B K-major
       | ((uint32_t)(N >> 3) << 17)
       | ((uint32_t)(M >> 4) << 24);
}

template <int NCOL>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&v)[NCOL]);
template <>
__device__ __forceinline__ void tmem_st<8>(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr) : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
               ::"r"(smem_u32(bar)), "r"(par) : "memory");
}

constexpr int M = 128, K = 24, NMAX = 256;

// B (N x K, element (n, k)) in smem, K-major no-swizzle core matrices:
// offset(n, k) = (k / 8) * KSTEP + ((k % 8) / 4) * LBO + (n / 8) * SBO + (n % 8) * 16 + (k % 4) * 4
template <int N>
__global__ void probe(const float* A, const float* B, float* D, long long* clk, int reps, int nacc) {
  __shared__ __align__(1024) float sB[K * NMAX];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  constexpr uint32_t SBO = 128, LBO = (N / 8) * 128, KSTEP = 2 * LBO;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const uint32_t off = (k / 8) * KSTEP + ((k % 8) / 4) * LBO + (n / 8) * SBO + (n % 8) * 16 + (k % 4) * 4;
    sB[off / 4] = B[n * K + k];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic smem writes -> async proxy (MMA reads)
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tb = tbase;
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  // A row `tid` (K values) -> TMEM columns [128, 128 + K)
  for (int c = 0; c < K; c += 8) {
    uint32_t v[8];
    for (int j = 0; j < 8; ++j) v[j] = __float_as_uint(A[tid * K + c + j]);
    tmem_st<8>(tb + lane_base + 384 + c, v);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  constexpr uint32_t idesc = make_idesc(M, N);
  const uint32_t sb = smem_u32(sB);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    // D at column 8 (an offset, to check D addressing); 3 k-steps, the first overwrites
    for (int ks = 0; ks < K / 8; ++ks)
      mma_tf32(tb + 8, tb + 384 + 8 * ks, make_desc(sb + ks * KSTEP, LBO, SBO), idesc, ks > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    tmem_ld8(tb + lane_base + 8 + c, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int j = 0; j < 8; ++j) D[tid * N + c + j] = __uint_as_float(v[j]);
  }
  // timing: reps x (K/8) back-to-back MMAs into one accumulator
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (tid == 0) {
    t0 = clock64();
    const uint64_t d0 = make_desc(sb, LBO, SBO), d1 = make_desc(sb + KSTEP, LBO, SBO), d2 = make_desc(sb + 2 * KSTEP, LBO, SBO);
    const uint32_t a0 = tb + 384;
    if (nacc == 1) {
      for (int r = 0; r < reps; ++r) {
        mma_tf32(tb + 8, a0, d0, idesc, 1);
        mma_tf32(tb + 8, a0 + 8, d1, idesc, 1);
        mma_tf32(tb + 8, a0 + 16, d2, idesc, 1);
      }
    } else if (N <= 48) {
      for (int r = 0; r < reps; ++r) {
        mma_tf32(tb + 8, a0, d0, idesc, 1);
        mma_tf32(tb + 56, a0 + 8, d1, idesc, 1);
        mma_tf32(tb + 104, a0 + 16, d2, idesc, 1);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 1);
  if (tid == 0) {
    t1 = clock64();
    clk[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tb), "r"(512));
}

static float tf32_trunc(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

template <int N>
int run() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX - 0.5f;
  for (auto& x : B) x = (float)rand() / RAND_MAX - 0.5f;
  float *dA, *dB, *dD;
  long long* dclk;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMalloc(&dclk, 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  const int reps = 1000;
  long long clks[4];
  for (int nacc = (N <= 48 ? 3 : 1); nacc >= 1; --nacc) {
    probe<N><<<1, 128>>>(dA, dB, dD, dclk, reps, nacc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&clks[nacc], dclk, 8, cudaMemcpyDeviceToHost));
  }
  printf("  rotating over 3 / 2 accumulators: %.2f / %.2f clk/MMA\n", (double)clks[3] / (reps * K / 8),
         (double)clks[2] / (reps * K / 8));
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long long clk;
  CK(cudaMemcpy(&clk, dclk, 8, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)tf32_trunc(A[m * K + k]) * tf32_trunc(B[n * K + k]);
      const double e = fabs(ref - D[m * N + n]);
      maxerr = fmax(maxerr, e);
      maxref = fmax(maxref, fabs(ref));
      if (e > 1e-4 && bad++ < 5) printf("  mismatch m=%d n=%d got %g want %g\n", m, n, D[m * N + n], ref);
    }
  printf("N=%d: max|D - ref| = %.3e (max|ref| %.3f) %s; %d MMAs (M=128,N=%d,K=8 tf32) in %lld clk = %.2f clk/MMA\n", N,
         maxerr, maxref, maxerr < 1e-5 ? "OK" : "FAIL", reps * K / 8, N, clk, (double)clk / (reps * K / 8));
  return maxerr < 1e-5 ? 0 : 1;
}

int main() {
  int f = run<24>();
  f |= run<48>();
  f |= run<32>();
  f |= run<64>();
  f |= run<128>();
  f |= run<256>();
  printf(f ? "PROBE FAILED\n" : "PROBE OK\n");
  return f;
}
