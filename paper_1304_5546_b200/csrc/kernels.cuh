// Stage kernels of the nodal-DG TM Maxwell operator for one (N, precision).
//
// Included once per translation unit (inst/k_N<N>_<prec>.cu) with
//   DG_N   polynomial degree,  DG_T  float | double,  DG_TAG  e.g. N5_f32
// so that every (N, T) is a separate CUDA module with its OWN __constant__
// bank holding Dr, Ds (Np x Np) and LIFT (Np x 3Nfp).  Uniform (warp-wide
// identical) operator entries are then fed to FFMA/DFMA straight from the
// constant bank -- no shared-memory traffic for the operator at all.
//
// Work decomposition:
//   * one warp lane per element, one warp per 32-element tile ("tile-blocked"
//     layout, kernel_api.h) -- every field access of a warp is one contiguous
//     128 B / 256 B line;
//   * a tile's rows n are split over P "row-group" warps when the per-thread
//     accumulators 3R (R rows) would exceed the register budget;
//   * TPC tiles per CTA; the CTA first stages its tiles' Hx, Hy, Ez
//     (cp.async 16 B, coalesced) and the neighbour traces q[vmapP]
//     (cp.async 4/8 B gathers, mostly L2 hits) into shared memory, then each
//     thread streams its element's column out of shared memory (conflict-free:
//     lane = element).
//
// Arithmetic per element (eq. 9, readings A1/A2; eq. 6 for the
// chain rule; 1/2 eq. 5 flux, reading A3; A12 for materials):
//   u = Dr Ez, v = Ds Ez                          -> rhsHx = -(ry u + sy v), rhsHy = rx u + sx v
//   w = Dr (rx Hy - ry Hx) + Ds (sx Hy - sy Hx)   -> rhsEz = w   (= Dx Hy - Dy Hx, affine elements)
//   rhs += LIFT (Fsc-scaled flux)
//   res = a res + dt rhs;  q_out = q_in + b res   (LSERK4; A10)
#include <cstdint>
#include <cuda_runtime.h>

#include "kernel_api.h"

#ifndef DG_N
#error "DG_N must be defined"
#endif

#define DG_CAT2(a, b) a##b
#define DG_CAT(a, b) DG_CAT2(a, b)

namespace {

using T = DG_T;
constexpr int N = DG_N;
constexpr int NP = (N + 1) * (N + 2) / 2;
constexpr int NFP = N + 1;
constexpr int NF = 3 * NFP;
constexpr int TL = dg::TILE;

// register budget for the 3R row accumulators
constexpr int RMAX = (sizeof(T) == 4) ? 28 : 16;
constexpr int P = (NP + RMAX - 1) / RMAX;   // row-group warps per tile
constexpr int R = (NP + P - 1) / P;         // rows per group

constexpr size_t smem_per_tile(bool surf) {
  return (size_t)(3 * NP + (surf ? 3 * NF : 0)) * TL * sizeof(T);
}
constexpr int choose_tpc() {
  int t = 4 / P;
  if (t < 1) t = 1;
  while (t > 1 && smem_per_tile(true) * t > 96 * 1024) --t;
  return t;
}
constexpr int TPC = choose_tpc();
constexpr int THREADS = TPC * P * 32;

__constant__ T cDr[NP * NP];
__constant__ T cDs[NP * NP];
__constant__ T cLIFT[NP * NF];

// Face node ids, increasing node index (closed form of the node ordering: row j
// of the triangle starts at j(N+1) - j(j-1)/2).  Checked against the setup's
// coordinate-derived Fmask by the runtime at context creation.
__host__ __device__ constexpr int row_start(int j) { return j * (N + 1) - j * (j - 1) / 2; }
__host__ __device__ constexpr int fmask(int f, int i) {
  return f == 0 ? i : (f == 1 ? row_start(i) + N - i : row_start(i));
}

__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* s, const void* g) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(sa), "l"(g), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

template <int MODE>
struct ModeTraits {
  static constexpr bool vol = (MODE == dg::MODE_FUSED_RK || MODE == dg::MODE_VOLUME || MODE == dg::MODE_RHS);
  static constexpr bool surf = (MODE != dg::MODE_VOLUME);
  static constexpr bool rk = (MODE == dg::MODE_FUSED_RK || MODE == dg::MODE_SURFACE_RK);
};

// One row group G of one tile: rows [G R, G R + RR).
template <int MODE, bool MAT, int G>
__device__ __forceinline__ void tile_body(const dg::StageArgs& p, const T* __restrict__ sq,
                                          const T* __restrict__ sp, int tile, int lane) {
  using MT = ModeTraits<MODE>;
  constexpr int NGEO = MAT ? dg::NGEO_MAT : dg::NGEO_CONST;
  constexpr int n0 = G * R;
  constexpr int RR = (NP - n0 < R) ? (NP - n0) : R;
  const T* __restrict__ gg = static_cast<const T*>(p.geo) + (int64_t)tile * NGEO * TL + lane;

  T rhx[RR], rhy[RR], rez[RR];
  if constexpr (MT::vol) {
    const T rx = gg[0 * TL], sx = gg[1 * TL], ry = gg[2 * TL], sy = gg[3 * TL];
    T u[RR], v[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) { u[r] = T(0); v[r] = T(0); rez[r] = T(0); }
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const T hx = sq[(0 * NP + j) * TL + lane];
      const T hy = sq[(1 * NP + j) * TL + lane];
      const T ez = sq[(2 * NP + j) * TL + lane];
      const T w1 = rx * hy - ry * hx;
      const T w2 = sx * hy - sy * hx;
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const T dr = cDr[(n0 + r) * NP + j];
        const T ds = cDs[(n0 + r) * NP + j];
        u[r] = fma(dr, ez, u[r]);
        v[r] = fma(ds, ez, v[r]);
        rez[r] = fma(dr, w1, rez[r]);
        rez[r] = fma(ds, w2, rez[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      rhx[r] = -(ry * u[r] + sy * v[r]);
      rhy[r] = rx * u[r] + sx * v[r];
    }
  } else if constexpr (MODE == dg::MODE_SURFACE_RK) {
    const T* __restrict__ rv = static_cast<const T*>(p.rhsv);
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      const int64_t off = ((int64_t)tile * NP + n0 + r) * TL + lane;
      rhx[r] = rv[off];
      rhy[r] = rv[p.vstride + off];
      rez[r] = rv[2 * p.vstride + off];
    }
  } else {
#pragma unroll
    for (int r = 0; r < RR; ++r) { rhx[r] = T(0); rhy[r] = T(0); rez[r] = T(0); }
  }

  if constexpr (MT::surf) {
    const T alpha = static_cast<T>(p.alpha);
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const T nx = gg[(4 + 3 * f) * TL], ny = gg[(5 + 3 * f) * TL], hF = gg[(6 + 3 * f) * TL];
      const T bsc = gg[(13 + f) * TL];
      T wEH = T(0), wHH = T(0), wHE = T(0), wEE = T(0);
      if constexpr (MAT) {
        wEH = gg[(18 + 4 * f) * TL];
        wHH = gg[(19 + 4 * f) * TL];
        wHE = gg[(20 + 4 * f) * TL];
        wEE = gg[(21 + 4 * f) * TL];
      }
#pragma unroll
      for (int i = 0; i < NFP; ++i) {
        const int m = f * NFP + i;
        const int fm = fmask(f, i);
        const T hxm = sq[(0 * NP + fm) * TL + lane];
        const T hym = sq[(1 * NP + fm) * TL + lane];
        const T ezm = sq[(2 * NP + fm) * TL + lane];
        const T hxp = sp[(0 * NF + m) * TL + lane];
        const T hyp = sp[(1 * NF + m) * TL + lane];
        const T ezp = sp[(2 * NF + m) * TL + lane];
        const T dHx = hxm - hxp;
        const T dHy = hym - hyp;
        const T dEz = ezm - bsc * ezp;
        T fHx, fHy, fEz;
        if constexpr (!MAT) {
          const T ndotdH = nx * dHx + ny * dHy;
          fHx = hF * (ny * dEz + alpha * (nx * ndotdH - dHx));
          fHy = hF * (-nx * dEz + alpha * (ny * ndotdH - dHy));
          fEz = hF * (ny * dHx - nx * dHy - alpha * dEz);
        } else {
          const T dHt = nx * dHy - ny * dHx;
          const T gH = wEH * dEz + wHH * dHt;
          fHx = hF * (ny * gH);
          fHy = -hF * (nx * gH);
          fEz = -hF * (wHE * dHt + wEE * dEz);
        }
#pragma unroll
        for (int r = 0; r < RR; ++r) {
          const T L = cLIFT[(n0 + r) * NF + m];
          rhx[r] = fma(L, fHx, rhx[r]);
          rhy[r] = fma(L, fHy, rhy[r]);
          rez[r] = fma(L, fEz, rez[r]);
        }
      }
    }
  }

  // material factors 1/mu, 1/eps (reading A12).  In split mode the volume kernel
  // writes the UNSCALED rhsV and the surface kernel scales the sum.
  if constexpr (MAT) {
    if (MODE != dg::MODE_VOLUME || p.scale_volume) {
      const T imu = gg[16 * TL], ieps = gg[17 * TL];
#pragma unroll
      for (int r = 0; r < RR; ++r) { rhx[r] *= imu; rhy[r] *= imu; rez[r] *= ieps; }
    }
  }

  if constexpr (MT::rk) {
    T* __restrict__ res = static_cast<T*>(p.res);
    T* __restrict__ qo = static_cast<T*>(p.q_out);
    const T a = static_cast<T>(p.a), b = static_cast<T>(p.b), dt = static_cast<T>(p.dt);
    const bool read_res = p.a != 0.0;
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      const int n = n0 + r;
      const int64_t off = ((int64_t)tile * NP + n) * TL + lane;
      const T rhs[3] = {rhx[r], rhy[r], rez[r]};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        T rs = dt * rhs[c];
        if (read_res) rs = fma(a, res[c * p.vstride + off], rs);
        if (p.write_res) res[c * p.vstride + off] = rs;
        qo[c * p.fstride + off] = fma(b, rs, sq[(c * NP + n) * TL + lane]);
      }
    }
  } else {
    T* __restrict__ out = static_cast<T*>(p.out);
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      const int64_t off = ((int64_t)tile * NP + n0 + r) * TL + lane;
      out[off] = rhx[r];
      out[p.vstride + off] = rhy[r];
      out[2 * p.vstride + off] = rez[r];
    }
  }
}

template <int MODE, bool MAT, int G>
__device__ __forceinline__ void dispatch_group(int g, const dg::StageArgs& p, const T* sq, const T* sp,
                                               int tile, int lane) {
  if constexpr (G < P) {
    if (g == G) tile_body<MODE, MAT, G>(p, sq, sp, tile, lane);
    else dispatch_group<MODE, MAT, G + 1>(g, p, sq, sp, tile, lane);
  }
}

template <int MODE, bool MAT>
__global__ void __launch_bounds__(THREADS) stage_kernel(const dg::StageArgs p) {
  using MT = ModeTraits<MODE>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sq = reinterpret_cast<T*>(smem_raw);          // [TPC][3][NP][32]
  T* sp = sq + (size_t)TPC * 3 * NP * TL;          // [TPC][3][NF][32]
  const T* __restrict__ q = static_cast<const T*>(p.q_in);
  const int slot0 = blockIdx.x * TPC;

  // ---- stage this CTA's tiles and their neighbour traces into shared memory
  constexpr int CH = 16 / (int)sizeof(T);
  constexpr int CHUNKS = NP * TL / CH;  // 16 B chunks per field tile
  for (int i = threadIdx.x; i < TPC * 3 * CHUNKS; i += THREADS) {
    const int tl = i / (3 * CHUNKS);
    const int rem = i - tl * 3 * CHUNKS;
    const int c = rem / CHUNKS;
    const int ch = rem - c * CHUNKS;
    const int slot = slot0 + tl;
    if (slot >= p.ntiles) continue;
    const int tile = p.tiles ? p.tiles[slot] : slot;
    cp_async16(sq + ((size_t)tl * 3 + c) * NP * TL + ch * CH, q + c * p.fstride + (int64_t)tile * NP * TL + ch * CH);
  }
  if constexpr (MT::surf) {
    for (int i = threadIdx.x; i < TPC * NF * TL; i += THREADS) {
      const int tl = i / (NF * TL);
      const int rem = i - tl * NF * TL;  // m*32 + lane
      const int slot = slot0 + tl;
      if (slot >= p.ntiles) continue;
      const int tile = p.tiles ? p.tiles[slot] : slot;
      const int idx = __ldg(p.vmapP + (int64_t)tile * NF * TL + rem);
#pragma unroll
      for (int c = 0; c < 3; ++c)
        cp_async_small<sizeof(T)>(sp + ((size_t)tl * 3 + c) * NF * TL + rem, q + c * p.fstride + idx);
    }
  }
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tl = warp / P, g = warp - (warp / P) * P;
  const int slot = slot0 + tl;
  if (slot >= p.ntiles) return;
  const int tile = p.tiles ? p.tiles[slot] : slot;
  dispatch_group<MODE, MAT, 0>(g, p, sq + (size_t)tl * 3 * NP * TL, sp + (size_t)tl * 3 * NF * TL, tile, lane);
}

template <int MODE, bool MAT>
cudaError_t launch_one(const dg::StageArgs& a, cudaStream_t s) {
  constexpr size_t smem = TPC * smem_per_tile(ModeTraits<MODE>::surf);
  static bool configured = false;  // per process; attribute is per device-function (set once)
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(stage_kernel<MODE, MAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = (a.ntiles + TPC - 1) / TPC;
  if (grid == 0) return cudaSuccess;
  stage_kernel<MODE, MAT><<<grid, THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch(int mode, bool mat, const dg::StageArgs& a, cudaStream_t s) {
  switch (mode * 2 + (mat ? 1 : 0)) {
    case dg::MODE_FUSED_RK * 2 + 0: return launch_one<dg::MODE_FUSED_RK, false>(a, s);
    case dg::MODE_FUSED_RK * 2 + 1: return launch_one<dg::MODE_FUSED_RK, true>(a, s);
    case dg::MODE_VOLUME * 2 + 0: return launch_one<dg::MODE_VOLUME, false>(a, s);
    case dg::MODE_VOLUME * 2 + 1: return launch_one<dg::MODE_VOLUME, true>(a, s);
    case dg::MODE_SURFACE_RK * 2 + 0: return launch_one<dg::MODE_SURFACE_RK, false>(a, s);
    case dg::MODE_SURFACE_RK * 2 + 1: return launch_one<dg::MODE_SURFACE_RK, true>(a, s);
    case dg::MODE_RHS * 2 + 0: return launch_one<dg::MODE_RHS, false>(a, s);
    case dg::MODE_RHS * 2 + 1: return launch_one<dg::MODE_RHS, true>(a, s);
    case dg::MODE_SURFACE * 2 + 0: return launch_one<dg::MODE_SURFACE, false>(a, s);
    case dg::MODE_SURFACE * 2 + 1: return launch_one<dg::MODE_SURFACE, true>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t upload(const double* Dr, const double* Ds, const double* LIFT) {
  T h[NP * (NP > NF ? NP : NF)];
  for (int i = 0; i < NP * NP; ++i) h[i] = static_cast<T>(Dr[i]);
  cudaError_t e = cudaMemcpyToSymbol(cDr, h, sizeof(T) * NP * NP);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < NP * NP; ++i) h[i] = static_cast<T>(Ds[i]);
  e = cudaMemcpyToSymbol(cDs, h, sizeof(T) * NP * NP);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < NP * NF; ++i) h[i] = static_cast<T>(LIFT[i]);
  e = cudaMemcpyToSymbol(cLIFT, h, sizeof(T) * NP * NF);
  return e;
}

// the closed-form face masks compiled into the kernels must match the setup's node set
bool check_fmask(const int* Fmask) {
  for (int f = 0; f < 3; ++f)
    for (int i = 0; i < NFP; ++i)
      if (Fmask[f * NFP + i] != fmask(f, i)) return false;
  return true;
}

dg::KernelInfo info() {
  dg::KernelInfo k;
  k.N = N;
  k.prec = (int)sizeof(T);
  k.threads = THREADS;
  k.tiles_per_cta = TPC;
  k.row_groups = P;
  k.rows_per_group = R;
  k.smem_bytes = TPC * smem_per_tile(true);
  return k;
}

}  // namespace

namespace dg {
KernelModule DG_CAT(dg_module_, DG_TAG)() {
  KernelModule m;
  m.N = N;
  m.prec = (int)sizeof(T);
  m.upload = &upload;
  m.launch = &launch;
  m.info = &info;
  m.check_fmask = &check_fmask;
  return m;
}
}  // namespace dg
