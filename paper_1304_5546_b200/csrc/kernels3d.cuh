// Stage kernels of the 3D tetrahedral Maxwell operator for one (N, precision) (SURVEY.md §8(f)
// row 4; the paper's hedge workload).
//
// Included once per translation unit (inst/k3_N<N>_<prec>.cu) with DG_N, DG_T, DG_TAG.
// Fields (Hx, Hy, Hz, Ex, Ey, Ez), eps = mu = 1, PEC walls; the paper's two-kernel structure:
//   K1 volume:  per 32-element tile (TMA-staged fields + geometry), dH/dt = -curl E, dE/dt = curl H
//               by the chain rule d/dx = rx Dr + sx Ds + tx Dt regrouped so that each curl component
//               is three mat-vecs: (curl E)_x = Dr(ry Ez - rz Ey) + Ds(sy Ez - sz Ey) + Dt(ty Ez - tz Ey)
//               (18 mat-vecs per element); the operators broadcast from shared memory, one lane per
//               element, warp g computing output rows [gR, gR + R)  -> rhsV
//   K2 surface: per face point (split over the team) the traces q- (own node) and q+ (vmapP code;
//               PEC mirror E+ = -E-, H+ = H-), the upwind flux 1/2 (n x [E] + a(n(n.[H]) - [H])) and
//               1/2 (-n x [H] + a(n(n.[E]) - [E])) scaled by Fsc into shared memory; LIFT; + rhsV;
//               the LSERK4 update (res = a res + dt rhs; q_out = q_in + b res) with coalesced stores.
// Tile-blocked layout of kernel_api.h (6 fields, identity column swizzle).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "kernel_api.h"
#include "kernel3_api.h"

#ifndef DG_N
#error "DG_N must be defined"
#endif
#define DG_CAT2(a, b) a##b
#define DG_CAT(a, b) DG_CAT2(a, b)

namespace {

using T = DG_T;
constexpr bool F32 = sizeof(T) == 4;
constexpr int N = DG_N;
constexpr int NP = (N + 1) * (N + 2) * (N + 3) / 6;
constexpr int NFP = (N + 1) * (N + 2) / 2;
constexpr int NF = 4 * NFP;
constexpr int TL = dg::TILE;
constexpr int NG = dg::NGEO3;
#ifndef DG_R
#define DG_R (sizeof(DG_T) == 4 ? 8 : 4)
#endif
constexpr int R = DG_R;                    // output rows per warp
constexpr int P = (NP + R - 1) / R;        // warps per tile
constexpr int RP = P * R;                  // padded rows (zero operator rows)
constexpr int TEAM = 32 * P;
// surface kernel: its own rows per warp (smaller: more warps to hide the trace-load latency)
#ifndef DG_RS
#define DG_RS (sizeof(DG_T) == 4 ? 4 : 2)
#endif
constexpr int RS = DG_RS * 32 >= NP ? DG_RS : (NP + 31) / 32;  // at most 32 warps per CTA
constexpr int PS = (NP + RS - 1) / RS;
constexpr int RPS = PS * RS;
constexpr int TEAMS = 32 * PS;
constexpr int KPT = (NF + PS - 1) / PS;    // face points per warp (surface kernel)
// fused stage kernel: its own rows per warp (volume + LIFT accumulators and the residual in registers)
#ifndef DG_RF
#define DG_RF 4
#endif
constexpr int RF = DG_RF * 32 >= NP ? DG_RF : (NP + 31) / 32;
constexpr int PF = (NP + RF - 1) / RF;
constexpr int RPF = PF * RF;
constexpr int TEAMF = 32 * PF;
// DG_VS (fused kernel): the volume term by the 18 derivative sums D_d F_c of each output row (18 FMAs per
// operator entry, the chain rule applied once per row) instead of the regrouped W form, whose 36
// geometry products per node column every warp repeats
#ifndef DG_VS
#define DG_VS 1
#endif
constexpr bool VSUM = DG_VS;
#ifndef DG_VSV
#define DG_VSV 0  // the same for the volume kernel (split stages, dg3_eval_rhs); off: at fp64 N = 5,
                  // the one tuned case that runs it, its 18 R sums spill
#endif
constexpr bool VSUMV = DG_VSV;
// DG_G3 (fused kernel), the neighbour traces of the flux:
//   0  codes and traces loaded inside the flux loop (code -> trace: two dependent L2 round trips)
//   1  codes loaded at the top of the tile into registers, the cross-tile traces gathered by cp.async
//      into the flux buffer there too (each thread its own face points); measured slower
//   2  codes loaded at the top of the tile into registers (their latency hides behind the volume),
//      traces from L2 in the (fully unrolled) flux loop
#ifndef DG_G3
#define DG_G3 0
#endif
constexpr bool G3 = DG_G3 == 1;
constexpr bool PRECODE = DG_G3 != 0;
constexpr int RPD = RP > RPF ? RP : RPF;  // operator-row padding of DV (volume and fused kernels)
// operator block: DV[j][n] = {Dr, Ds, Dt, 0} [NP][RP], LV[m][n] [NF][RP], fmask [NF] int32
struct alignas(4 * sizeof(T)) T4 { T x, y, z, w; };
constexpr size_t DVB = (size_t)NP * RPD * sizeof(T4);
constexpr int RPM = (RP > RPS ? RP : RPS) > RPF ? (RP > RPS ? RP : RPS) : RPF;  // LIFT row padding (all kernels)
constexpr size_t LVB = (size_t)NF * RPM * sizeof(T);
constexpr size_t FMB = ((size_t)NF * 4 + 15) / 16 * 16;
constexpr size_t OPS = DVB + LVB + FMB;
constexpr size_t QB = (size_t)6 * NP * TL * sizeof(T);
constexpr size_t GB = (size_t)NG * TL * sizeof(T);
constexpr size_t SPB = (size_t)6 * NF * TL * sizeof(T);
constexpr size_t BARB = 64;
constexpr size_t SMEM_VOL = BARB + DVB + QB + GB;
// the surface kernel stages the tile's fields and geometry by TMA (own and same-tile neighbour traces
// and q_in from shared memory) whenever that fits; else traces straight from global memory (L2)
constexpr size_t SMEM_SURF_Q = BARB + LVB + FMB + SPB + QB + GB;
#ifndef DG_SQ
#define DG_SQ 1
#endif
constexpr bool STAGEQ = DG_SQ && SMEM_SURF_Q <= 227 * 1024;
// DG_PF3: the surface kernel loads rhsV and the residual of its rows at the top of the tile (registers)
#ifndef DG_PF3
#define DG_PF3 1
#endif
constexpr bool PF3 = DG_PF3;
constexpr size_t SMEM_SURF = STAGEQ ? SMEM_SURF_Q : LVB + FMB + SPB;
static_assert(SMEM_VOL <= 227 * 1024 && SMEM_SURF <= 227 * 1024, "3D kernel shared memory");
// fused stage kernel (volume + flux + LIFT + LSERK4, one launch per stage) when its tile fits
// DG_D3: the fused kernel double-buffers the tile's {fields, geometry} (the next tile's TMA is issued at
// the top of the current one) where the second buffer fits
#ifndef DG_D3
#define DG_D3 0
#endif
constexpr bool D3 = DG_D3 && BARB + DVB + LVB + FMB + 2 * (QB + GB) + SPB <= 227 * 1024;
constexpr size_t SMEM_FUSED = BARB + DVB + LVB + FMB + (D3 ? 2 : 1) * (QB + GB) + SPB;
#ifndef DG_F3
#define DG_F3 1
#endif
constexpr bool FUSED3 = DG_F3 && SMEM_FUSED <= 227 * 1024;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile("{\n.reg .pred P1;\nW3_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W3_%=;\n}\n" ::"r"(
                   smem_u32(bar)),
               "r"(parity)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

template <int MODE>
__host__ __device__ constexpr bool is_rk() { return MODE == dg::MODE_FUSED_RK || MODE == dg::MODE_SURFACE_RK; }

// Volume term by derivative sums (DG_VS): for each of the RR output rows n0 + r, S[d][c] = (D_d F_c)(n)
// over the tile's staged fields (18 FMAs per operator entry), then the chain rule once per row:
// acc = (-curl E, curl H) = (dH/dt, dE/dt), fields Hx Hy Hz Ex Ey Ez = 0..5
template <int RR>
__device__ __forceinline__ void volume_sums(const T* __restrict__ sq, const T4* __restrict__ DV, const T* __restrict__ gg,
                                          int n0, int lane, T (&acc)[6][RR]) {
  T S[3][6][RR];
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int c = 0; c < 6; ++c)
#pragma unroll
      for (int r = 0; r < RR; ++r) S[d][c][r] = T(0);
#pragma unroll 2
  for (int j = 0; j < NP; ++j) {
    const T* col = sq + j * TL + lane;
    T F[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) F[c] = col[c * NP * TL];
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      const T4 dd = DV[j * RPD + n0 + r];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        S[0][c][r] = fma(dd.x, F[c], S[0][c][r]);
        S[1][c][r] = fma(dd.y, F[c], S[1][c][r]);
        S[2][c][r] = fma(dd.z, F[c], S[2][c][r]);
      }
    }
  }
  const T dxv[3] = {gg[0 * TL], gg[3 * TL], gg[6 * TL]}, dyv[3] = {gg[1 * TL], gg[4 * TL], gg[7 * TL]},
          dzv[3] = {gg[2 * TL], gg[5 * TL], gg[8 * TL]};
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    // d/dx F_c = sum_d dx_d S[d][c] (eq. 6's chain rule, 3D); fields Hx Hy Hz Ex Ey Ez = 0..5
    auto Dx = [&](int c) { return dxv[0] * S[0][c][r] + dxv[1] * S[1][c][r] + dxv[2] * S[2][c][r]; };
    auto Dy = [&](int c) { return dyv[0] * S[0][c][r] + dyv[1] * S[1][c][r] + dyv[2] * S[2][c][r]; };
    auto Dz = [&](int c) { return dzv[0] * S[0][c][r] + dzv[1] * S[1][c][r] + dzv[2] * S[2][c][r]; };
    acc[0][r] = Dz(4) - Dy(5);  // dHx/dt = -(curl E)_x
    acc[1][r] = Dx(5) - Dz(3);
    acc[2][r] = Dy(3) - Dx(4);
    acc[3][r] = Dy(2) - Dz(1);  // dEx/dt = (curl H)_x
    acc[4][r] = Dz(0) - Dx(2);
    acc[5][r] = Dx(1) - Dy(0);
  }
}

// ---------------------------------------------------------------- K1: volume (curl) kernel
__global__ void __launch_bounds__(TEAM, 1) volume3d(const dg::StageArgs3 p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  const T4* DV = reinterpret_cast<const T4*>(smem_raw + BARB);
  T* sq = reinterpret_cast<T*>(smem_raw + BARB + DVB);
  T* sg = reinterpret_cast<T*>(smem_raw + BARB + DVB + QB);
  const T* __restrict__ q = static_cast<const T*>(p.q_in);
  const T* __restrict__ geo = static_cast<const T*>(p.geo);
  const int tid = threadIdx.x, g = tid >> 5, lane = tid & 31, n0 = g * R;
  const int first = blockIdx.x, stride = gridDim.x;
  const int n_it = first < p.ntiles ? (p.ntiles - first + stride - 1) / stride : 0;
  if (n_it == 0) return;
  auto issue = [&](int it) {
    if (tid == 0) {
      const int64_t t = first + (int64_t)it * stride;
      mbar_expect_tx(bar, (unsigned)(QB + GB));
#pragma unroll
      for (int c = 0; c < 6; ++c)
        tma_load_1d(sq + c * NP * TL, q + c * p.fstride + t * NP * TL, (unsigned)(NP * TL * sizeof(T)), bar);
      tma_load_1d(sg, geo + t * NG * TL, (unsigned)GB, bar);
    }
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const int4* src = reinterpret_cast<const int4*>(p.ops);
    int4* dst = reinterpret_cast<int4*>(smem_raw + BARB);
    for (int i = tid; i < (int)(DVB / 16); i += TEAM) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  issue(0);
  for (int it = 0; it < n_it; ++it) {
    mbar_wait(bar, (unsigned)(it & 1));
    __syncthreads();
    if (it + 1 < n_it && tid == 0) {
      const int64_t t1 = first + (int64_t)(it + 1) * stride;
#pragma unroll
      for (int c = 0; c < 6; ++c) prefetch_l2(q + c * p.fstride + t1 * NP * TL, (unsigned)(NP * TL * sizeof(T)));
      prefetch_l2(geo + t1 * NG * TL, (unsigned)GB);
    }
    const int64_t t = first + (int64_t)it * stride;
    const T* gg = sg + lane;
    if constexpr (VSUMV) {  // derivative sums (volume_sums): acc = (dH/dt, dE/dt) directly
      T acc[6][R];
      volume_sums<R>(sq, DV, gg, n0, lane, acc);
      __syncthreads();  // every warp is done with the tile's fields: the next TMA may overwrite them
      if (it + 1 < n_it) issue(it + 1);
      T* __restrict__ out = static_cast<T*>(p.out);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int n = n0 + r;
        if (RP != NP && n >= NP) break;
        const int64_t o = (t * NP + n) * TL + lane;
#pragma unroll
        for (int c = 0; c < 6; ++c) out[c * p.vstride + o] = acc[c][r];
      }
      continue;
    }
    const T rx = gg[0 * TL], ry = gg[1 * TL], rz = gg[2 * TL], sx = gg[3 * TL], sy = gg[4 * TL], sz = gg[5 * TL],
            tx = gg[6 * TL], ty = gg[7 * TL], tz = gg[8 * TL];
    T acc[6][R];
#pragma unroll
    for (int c = 0; c < 6; ++c)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[c][r] = T(0);
#pragma unroll 2
    for (int j = 0; j < NP; ++j) {
      const T* col = sq + j * TL + lane;
      const T Hx = col[0 * NP * TL], Hy = col[1 * NP * TL], Hz = col[2 * NP * TL];
      const T Ex = col[3 * NP * TL], Ey = col[4 * NP * TL], Ez = col[5 * NP * TL];
      // (curl F)_x = sum_d D_d (dy_d Fz - dz_d Fy), _y = D_d(dz_d Fx - dx_d Fz), _z = D_d(dx_d Fy - dy_d Fx)
      // with (dx_d, dy_d, dz_d) = (rx, ry, rz), (sx, sy, sz), (tx, ty, tz) for d = r, s, t
      T W[6][3];
      const T dxv[3] = {rx, sx, tx}, dyv[3] = {ry, sy, ty}, dzv[3] = {rz, sz, tz};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        W[0][d] = dyv[d] * Ez - dzv[d] * Ey;  // curl E -> accumulated, negated for dH/dt
        W[1][d] = dzv[d] * Ex - dxv[d] * Ez;
        W[2][d] = dxv[d] * Ey - dyv[d] * Ex;
        W[3][d] = dyv[d] * Hz - dzv[d] * Hy;  // curl H -> dE/dt
        W[4][d] = dzv[d] * Hx - dxv[d] * Hz;
        W[5][d] = dxv[d] * Hy - dyv[d] * Hx;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const T4 d = DV[j * RPD + n0 + r];
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[c][r] = fma(d.x, W[c][0], fma(d.y, W[c][1], fma(d.z, W[c][2], acc[c][r])));
      }
    }
    __syncthreads();  // every warp is done with the tile's fields: the next TMA may overwrite them
    if (it + 1 < n_it) issue(it + 1);
    T* __restrict__ out = static_cast<T*>(p.out);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int n = n0 + r;
      if (RP != NP && n >= NP) break;
      const int64_t o = (t * NP + n) * TL + lane;
#pragma unroll
      for (int c = 0; c < 6; ++c) out[c * p.vstride + o] = c < 3 ? -acc[c][r] : acc[c][r];
    }
  }
}

// ---------------------------------------------------------------- K2: surface + LIFT (+ LSERK4)
template <int MODE>
__global__ void __launch_bounds__(TEAMS, 1) surface3d(const dg::StageArgs3 p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr size_t OFF = STAGEQ ? BARB : 0;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  const T* LV = reinterpret_cast<const T*>(smem_raw + OFF);
  const int32_t* fmask = reinterpret_cast<const int32_t*>(smem_raw + OFF + LVB);
  T* sp = reinterpret_cast<T*>(smem_raw + OFF + LVB + FMB);
  T* sq = reinterpret_cast<T*>(smem_raw + OFF + LVB + FMB + SPB);       // STAGEQ: the tile's fields
  T* sgeo = reinterpret_cast<T*>(smem_raw + OFF + LVB + FMB + SPB + QB);  // STAGEQ: its geometry
  const T* __restrict__ q = static_cast<const T*>(p.q_in);
  const T* __restrict__ geo = static_cast<const T*>(p.geo);
  const int tid = threadIdx.x, g = tid >> 5, lane = tid & 31, n0 = g * RS;
  const int first = blockIdx.x, stride = gridDim.x;
  const int n_it = first < p.ntiles ? (p.ntiles - first + stride - 1) / stride : 0;
  if (n_it == 0) return;
  auto issue = [&](int it) {
    if (STAGEQ && tid == 0) {
      const int64_t t = first + (int64_t)it * stride;
      mbar_expect_tx(bar, (unsigned)(QB + GB));
#pragma unroll
      for (int c = 0; c < 6; ++c)
        tma_load_1d(sq + c * NP * TL, q + c * p.fstride + t * NP * TL, (unsigned)(NP * TL * sizeof(T)), bar);
      tma_load_1d(sgeo, geo + t * NG * TL, (unsigned)GB, bar);
    }
  };
  if (STAGEQ && tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const int4* src = reinterpret_cast<const int4*>(static_cast<const unsigned char*>(p.ops) + DVB);
    int4* dst = reinterpret_cast<int4*>(smem_raw + OFF);
    for (int i = tid; i < (int)((LVB + FMB) / 16); i += TEAMS) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  issue(0);
  const T alpha = static_cast<T>(p.alpha);
  const bool read_res = is_rk<MODE>() && p.a != 0.0;
  for (int it = 0; it < n_it; ++it) {
    const int64_t t = first + (int64_t)it * stride;
    if constexpr (STAGEQ) {
      mbar_wait(bar, (unsigned)(it & 1));
      __syncthreads();
      if (it + 1 < n_it && tid == 0) {
        const int64_t t1 = t + stride;
#pragma unroll
        for (int c = 0; c < 6; ++c) prefetch_l2(q + c * p.fstride + t1 * NP * TL, (unsigned)(NP * TL * sizeof(T)));
        prefetch_l2(geo + t1 * NG * TL, (unsigned)GB);
      }
    }
    // geometry and own traces: shared memory (STAGEQ) or global; field stride FSQ of that source
    const T* gg = STAGEQ ? sgeo + lane : geo + t * NG * TL + lane;
    const T* qt = STAGEQ ? sq + lane : q + t * NP * TL + lane;
    const int64_t FSQ = STAGEQ ? (int64_t)NP * TL : p.fstride;
    const int32_t* codes = p.vmapP + t * NF * TL + lane;
    // rhsV (the volume kernel's output) and the LSERK4 residual of this warp's rows: issued before the
    // flux, so their latency hides behind the flux and the LIFT (DG_PF3; the LIFT accumulates onto rhsV)
    T acc[6][RS], rr[6][RS];
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const int n = n0 + r < NP ? n0 + r : NP - 1;
      const int64_t o = (t * NP + n) * TL + lane;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        acc[c][r] = (PF3 && MODE != dg::MODE_SURFACE) ? static_cast<const T*>(p.rhsv)[c * p.vstride + o] : T(0);
        if constexpr (PF3 && is_rk<MODE>()) rr[c][r] = read_res ? __ldcs(static_cast<const T*>(p.res) + c * p.vstride + o) : T(0);
      }
    }
    // flux at this warp's face points m = g + kP (compile-time trip count: the trace loads of
    // several points are in flight together)
#pragma unroll 4
    for (int k = 0; k < KPT; ++k) {
      const int m = g + k * PS;
      if (m >= NF) break;
      const int f = m / NFP;
      const int fm = fmask[m];
      const int32_t code = __ldg(codes + m * TL);
      // code >= 0: offset in a global field; code < 0 (STAGEQ): same tile, shared offset -(1 + code)
      const T* pn = code >= 0 ? q + code : sq + (-1 - code);
      const int64_t fsn = code >= 0 ? p.fstride : (int64_t)NP * TL;
      T own[6], nb[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        own[c] = qt[c * FSQ + fm * TL];
        nb[c] = pn[c * fsn];
      }
      const T nx = gg[(9 + 4 * f) * TL], ny = gg[(10 + 4 * f) * TL], nz = gg[(11 + 4 * f) * TL];
      const T hF = gg[(12 + 4 * f) * TL], bsc = gg[(25 + f) * TL];
      T d[6];
#pragma unroll
      for (int c = 0; c < 6; ++c)  // PEC (bsc = -1, code = own node): [H] = 0, [E] = 2 E-
        d[c] = c < 3 ? (bsc < T(0) ? T(0) : own[c] - nb[c]) : own[c] - bsc * nb[c];
      const T ndH = nx * d[0] + ny * d[1] + nz * d[2];
      const T ndE = nx * d[3] + ny * d[4] + nz * d[5];
      T* s = sp + m * TL + lane;
      s[0 * NF * TL] = hF * ((ny * d[5] - nz * d[4]) + alpha * (nx * ndH - d[0]));
      s[1 * NF * TL] = hF * ((nz * d[3] - nx * d[5]) + alpha * (ny * ndH - d[1]));
      s[2 * NF * TL] = hF * ((nx * d[4] - ny * d[3]) + alpha * (nz * ndH - d[2]));
      s[3 * NF * TL] = hF * (-(ny * d[2] - nz * d[1]) + alpha * (nx * ndE - d[3]));
      s[4 * NF * TL] = hF * (-(nz * d[0] - nx * d[2]) + alpha * (ny * ndE - d[4]));
      s[5 * NF * TL] = hF * (-(nx * d[1] - ny * d[0]) + alpha * (nz * ndE - d[5]));
    }
    __syncthreads();
#pragma unroll 2
    for (int m = 0; m < NF; ++m) {
      T fv[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) fv[c] = sp[(c * NF + m) * TL + lane];
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const T l = LV[m * RPM + n0 + r];
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[c][r] = fma(l, fv[c], acc[c][r]);
      }
    }
    __syncthreads();  // sp is rewritten by the next tile
    const T a = static_cast<T>(p.a), b = static_cast<T>(p.b), dt = static_cast<T>(p.dt);
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const int n = n0 + r;
      if (RPS != NP && n >= NP) break;
      const int64_t o = (t * NP + n) * TL + lane;
      T rhs[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        rhs[c] = acc[c][r];
        if (!PF3 && MODE != dg::MODE_SURFACE) rhs[c] += static_cast<const T*>(p.rhsv)[c * p.vstride + o];
      }
      if constexpr (is_rk<MODE>()) {
        T* __restrict__ res = static_cast<T*>(p.res);
        T* __restrict__ qo = static_cast<T*>(p.q_out);
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          T rs = dt * rhs[c];
          if (read_res) rs = fma(a, PF3 ? rr[c][r] : __ldcs(res + c * p.vstride + o), rs);
          if (p.write_res) __stcs(res + c * p.vstride + o, rs);
          __stcs(qo + c * p.fstride + o, fma(b, rs, qt[c * FSQ + n * TL]));
        }
      } else {
        T* __restrict__ out = static_cast<T*>(p.out);
#pragma unroll
        for (int c = 0; c < 6; ++c) out[c * p.vstride + o] = rhs[c];
      }
    }
    if constexpr (STAGEQ) {
      if (it + 1 < n_it) {
        __syncthreads();  // every thread is done with the tile's staged fields
        issue(it + 1);
      }
    }
  }
}


// ---------------------------------------------------------------- fused stage: K1 + K2 + LSERK4
// One launch per LSERK4 stage: per tile the fields and geometry arrive by
// TMA; the volume curl (as volume3d) and the LIFT of the flux (as surface3d) accumulate into the same
// registers (warp g: rows [gR, gR + R)); the flux of this warp's face points m = g + kP reads own and
// same-tile neighbour traces from shared memory, other neighbours from global memory / L2; the
// LSERK4 residual of the warp's rows is loaded at the top of the tile.  No rhsV round trip.
#ifndef DG_F3C
#define DG_F3C 1  // resident fused CTAs per SM the register budget is sized for
#endif
__global__ void __launch_bounds__(TEAMF, DG_F3C) fused3d(const dg::StageArgs3 p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  const T4* DV = reinterpret_cast<const T4*>(smem_raw + BARB);
  const T* LV = reinterpret_cast<const T*>(smem_raw + BARB + DVB);
  const int32_t* fmask = reinterpret_cast<const int32_t*>(smem_raw + BARB + DVB + LVB);
  T* const sq0 = reinterpret_cast<T*>(smem_raw + BARB + DVB + LVB + FMB);
  T* const sg0 = reinterpret_cast<T*>(smem_raw + BARB + DVB + LVB + FMB + QB);
  T* sp = reinterpret_cast<T*>(smem_raw + BARB + DVB + LVB + FMB + QB + GB);
  T* const sq1 = D3 ? reinterpret_cast<T*>(smem_raw + BARB + DVB + LVB + FMB + QB + GB + SPB) : sq0;  // DG_D3
  T* const sg1 = D3 ? sq1 + (size_t)6 * NP * TL : sg0;
  const T* __restrict__ q = static_cast<const T*>(p.q_in);
  const T* __restrict__ geo = static_cast<const T*>(p.geo);
  const int tid = threadIdx.x, g = tid >> 5, lane = tid & 31, n0 = g * RF;
  const int first = blockIdx.x, stride = gridDim.x;
  const int n_it = first < p.ntiles ? (p.ntiles - first + stride - 1) / stride : 0;
  if (n_it == 0) return;
  constexpr int KPF = (NF + PF - 1) / PF;  // face points per warp
  auto issue = [&](int it) {
    if (tid == 0) {
      const int64_t t = first + (int64_t)it * stride;
      uint64_t* bb = bar + (D3 ? (it & 1) : 0);
      T* dq = D3 && (it & 1) ? sq1 : sq0;
      T* dg = D3 && (it & 1) ? sg1 : sg0;
      mbar_expect_tx(bb, (unsigned)(QB + GB));
#pragma unroll
      for (int c = 0; c < 6; ++c)
        tma_load_1d(dq + c * NP * TL, q + c * p.fstride + t * NP * TL, (unsigned)(NP * TL * sizeof(T)), bb);
      tma_load_1d(dg, geo + t * NG * TL, (unsigned)GB, bb);
    }
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    if (D3) mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const int4* src = reinterpret_cast<const int4*>(p.ops);
    int4* dst = reinterpret_cast<int4*>(smem_raw + BARB);
    for (int i = tid; i < (int)((DVB + LVB + FMB) / 16); i += TEAMF) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  issue(0);
  const T alpha = static_cast<T>(p.alpha);
  const bool read_res = p.a != 0.0;
  const T a = static_cast<T>(p.a), b = static_cast<T>(p.b), dt = static_cast<T>(p.dt);
  for (int it = 0; it < n_it; ++it) {
    const int64_t t = first + (int64_t)it * stride;
    T* const sq = D3 && (it & 1) ? sq1 : sq0;
    T* const sg = D3 && (it & 1) ? sg1 : sg0;
    mbar_wait(bar + (D3 ? (it & 1) : 0), (unsigned)(D3 ? ((it >> 1) & 1) : (it & 1)));
    __syncthreads();
    if (D3 && it + 1 < n_it) issue(it + 1);  // the other buffer: tile it-1 is done with it
    if (it + 1 < n_it && tid == 0) {
      const int64_t t1 = t + stride;
#pragma unroll
      for (int c = 0; c < 6; ++c) prefetch_l2(q + c * p.fstride + t1 * NP * TL, (unsigned)(NP * TL * sizeof(T)));
      prefetch_l2(geo + t1 * NG * TL, (unsigned)GB);
    }
    const int32_t* codes = p.vmapP + t * NF * TL + lane;
    int32_t cc[(NF + PF - 1) / PF];  // neighbour codes of this thread's face points m = g + k PF (PRECODE)
    if constexpr (PRECODE) {
#pragma unroll
      for (int k = 0; k < (NF + PF - 1) / PF; ++k) {
        const int m = g + k * PF;
        cc[k] = m < NF ? __ldg(codes + m * TL) : -1;
      }
    }
    if constexpr (G3) {  // cross-tile neighbour traces -> sp (the previous tile's LIFT is done with it)
#pragma unroll
      for (int k = 0; k < (NF + PF - 1) / PF; ++k) {
        const int m = g + k * PF;
        if (m < NF && cc[k] >= 0) {
#pragma unroll
          for (int c = 0; c < 6; ++c)
            cp_async_small<sizeof(T)>(sp + (c * NF + m) * TL + lane, q + cc[k] + c * p.fstride);
        }
      }
      cp_async_commit();
    }
    // the LSERK4 residual of this warp's rows (in flight during the volume and surface phases)
    T rr[6][RF];
#pragma unroll
    for (int r = 0; r < RF; ++r) {
      const int n = n0 + r < NP ? n0 + r : NP - 1;
      const int64_t o = (t * NP + n) * TL + lane;
#pragma unroll
      for (int c = 0; c < 6; ++c) rr[c][r] = read_res ? __ldcs(static_cast<const T*>(p.res) + c * p.vstride + o) : T(0);
    }
    const T* gg = sg + lane;
    T acc[6][RF];
    if constexpr (VSUM) {  // volume by derivative sums (volume_sums)
      volume_sums<RF>(sq, DV, gg, n0, lane, acc);
    } else {  // volume: acc = (-curl E, curl H) of rows n0 .. n0 + R - 1 (volume3d's regrouped chain rule)
      const T rx = gg[0 * TL], ry = gg[1 * TL], rz = gg[2 * TL], sx = gg[3 * TL], sy = gg[4 * TL], sz = gg[5 * TL],
              tx = gg[6 * TL], ty = gg[7 * TL], tz = gg[8 * TL];
#pragma unroll
      for (int c = 0; c < 6; ++c)
#pragma unroll
        for (int r = 0; r < RF; ++r) acc[c][r] = T(0);
#pragma unroll 2
      for (int j = 0; j < NP; ++j) {
        const T* col = sq + j * TL + lane;
        const T Hx = col[0 * NP * TL], Hy = col[1 * NP * TL], Hz = col[2 * NP * TL];
        const T Ex = col[3 * NP * TL], Ey = col[4 * NP * TL], Ez = col[5 * NP * TL];
        T W[6][3];
        const T dxv[3] = {rx, sx, tx}, dyv[3] = {ry, sy, ty}, dzv[3] = {rz, sz, tz};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          W[0][d] = dzv[d] * Ey - dyv[d] * Ez;  // -(curl E)  -> dH/dt
          W[1][d] = dxv[d] * Ez - dzv[d] * Ex;
          W[2][d] = dyv[d] * Ex - dxv[d] * Ey;
          W[3][d] = dyv[d] * Hz - dzv[d] * Hy;  // curl H -> dE/dt
          W[4][d] = dzv[d] * Hx - dxv[d] * Hz;
          W[5][d] = dxv[d] * Hy - dyv[d] * Hx;
        }
#pragma unroll
        for (int r = 0; r < RF; ++r) {
          const T4 d = DV[j * RPD + n0 + r];
#pragma unroll
          for (int c = 0; c < 6; ++c) acc[c][r] = fma(d.x, W[c][0], fma(d.y, W[c][1], fma(d.z, W[c][2], acc[c][r])));
        }
      }
    }
    // flux of this warp's face points into sp (surface3d's upwind flux, 1/2 of the jump form)
    if constexpr (G3) cp_async_wait_all();  // this thread's own gathers
#pragma unroll (PRECODE ? KPF : 4)
    for (int k = 0; k < KPF; ++k) {
      const int m = g + k * PF;
      if (m >= NF) break;
      const int f = m / NFP;
      const int fm = fmask[m];
      int32_t code;
      if constexpr (PRECODE) code = cc[k];
      else code = __ldg(codes + m * TL);
      const T* pn = code >= 0 ? (G3 ? sp + m * TL + lane : q + code) : sq + (-1 - code);
      const int64_t fsn = code >= 0 ? (G3 ? (int64_t)NF * TL : p.fstride) : (int64_t)NP * TL;
      T own[6], nb[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        own[c] = sq[c * NP * TL + fm * TL + lane];
        nb[c] = pn[c * fsn];
      }
      const T nx = gg[(9 + 4 * f) * TL], ny = gg[(10 + 4 * f) * TL], nz = gg[(11 + 4 * f) * TL];
      const T hF = gg[(12 + 4 * f) * TL], bsc = gg[(25 + f) * TL];
      T d[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) d[c] = c < 3 ? (bsc < T(0) ? T(0) : own[c] - nb[c]) : own[c] - bsc * nb[c];
      const T ndH = nx * d[0] + ny * d[1] + nz * d[2];
      const T ndE = nx * d[3] + ny * d[4] + nz * d[5];
      T* s = sp + m * TL + lane;
      s[0 * NF * TL] = hF * ((ny * d[5] - nz * d[4]) + alpha * (nx * ndH - d[0]));
      s[1 * NF * TL] = hF * ((nz * d[3] - nx * d[5]) + alpha * (ny * ndH - d[1]));
      s[2 * NF * TL] = hF * ((nx * d[4] - ny * d[3]) + alpha * (nz * ndH - d[2]));
      s[3 * NF * TL] = hF * (-(ny * d[2] - nz * d[1]) + alpha * (nx * ndE - d[3]));
      s[4 * NF * TL] = hF * (-(nz * d[0] - nx * d[2]) + alpha * (ny * ndE - d[4]));
      s[5 * NF * TL] = hF * (-(nx * d[1] - ny * d[0]) + alpha * (nz * ndE - d[5]));
    }
    __syncthreads();
#pragma unroll 2
    for (int m = 0; m < NF; ++m) {  // LIFT onto the volume term
      T fv[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) fv[c] = sp[(c * NF + m) * TL + lane];
#pragma unroll
      for (int r = 0; r < RF; ++r) {
        const T l = LV[m * RPM + n0 + r];
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[c][r] = fma(l, fv[c], acc[c][r]);
      }
    }
    // LSERK4 update (q_in from shared memory), streaming stores
    T* __restrict__ res = static_cast<T*>(p.res);
    T* __restrict__ qo = static_cast<T*>(p.q_out);
#pragma unroll
    for (int r = 0; r < RF; ++r) {
      const int n = n0 + r;
      if (RPF != NP && n >= NP) break;
      const int64_t o = (t * NP + n) * TL + lane;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        T rs = dt * acc[c][r];
        if (read_res) rs = fma(a, rr[c][r], rs);
        if (p.write_res) __stcs(res + c * p.vstride + o, rs);
        __stcs(qo + c * p.fstride + o, fma(b, rs, sq[(c * NP + n) * TL + lane]));
      }
    }
    if (!D3 && it + 1 < n_it) {
      __syncthreads();  // every thread is done with the tile's fields and flux
      issue(it + 1);
    }
  }
}

template <typename KER>
cudaError_t launch_k(KER kernel, size_t smem, int team, const dg::StageArgs3& a, cudaStream_t s, int* cap) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64) return cudaErrorInvalidDevice;
  if (cap[dev] == 0) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cudaGetLastError(), e;
    int per_sm = 0, sms = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, team, smem)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    cap[dev] = (per_sm > 0 ? per_sm : 1) * sms;
  }
  int grid = a.ntiles < cap[dev] ? a.ntiles : cap[dev];
  if (a.max_ctas > 0 && grid > a.max_ctas) grid = a.max_ctas;
  if (grid <= 0) return cudaSuccess;
  kernel<<<grid, team, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch(int mode, const dg::StageArgs3& a, cudaStream_t s) {
  static int cap_v[64] = {0}, cap_rk[64] = {0}, cap_rhs[64] = {0}, cap_s[64] = {0}, cap_f[64] = {0};
  switch (mode) {
    case dg::MODE_FUSED_RK:
      if constexpr (FUSED3) return launch_k(fused3d, SMEM_FUSED, TEAMF, a, s, cap_f);
      return cudaErrorNotSupported;
    case dg::MODE_VOLUME: return launch_k(volume3d, SMEM_VOL, TEAM, a, s, cap_v);
    case dg::MODE_SURFACE_RK: return launch_k(surface3d<dg::MODE_SURFACE_RK>, SMEM_SURF, TEAMS, a, s, cap_rk);
    case dg::MODE_RHS: return launch_k(surface3d<dg::MODE_RHS>, SMEM_SURF, TEAMS, a, s, cap_rhs);
    case dg::MODE_SURFACE: return launch_k(surface3d<dg::MODE_SURFACE>, SMEM_SURF, TEAMS, a, s, cap_s);
    default: return cudaErrorInvalidValue;
  }
}

size_t ops_bytes() { return OPS; }
void pack_ops(const double* Dr, const double* Ds, const double* Dt, const double* LIFT, const int* Fmask, void* out) {
  unsigned char* o = static_cast<unsigned char*>(out);
  for (size_t i = 0; i < OPS; ++i) o[i] = 0;
  T4* dv = reinterpret_cast<T4*>(o);
  for (int j = 0; j < NP; ++j)
    for (int n = 0; n < NP; ++n) {
      T4& e = dv[j * RPD + n];
      e.x = static_cast<T>(Dr[n * NP + j]);
      e.y = static_cast<T>(Ds[n * NP + j]);
      e.z = static_cast<T>(Dt[n * NP + j]);
    }
  T* lv = reinterpret_cast<T*>(o + DVB);
  for (int m = 0; m < NF; ++m)
    for (int n = 0; n < NP; ++n) lv[m * RPM + n] = static_cast<T>(LIFT[n * NF + m]);
  int32_t* fm = reinterpret_cast<int32_t*>(o + DVB + LVB);
  for (int m = 0; m < NF; ++m) fm[m] = Fmask[m];
}

dg::KernelInfo3 info() {
  dg::KernelInfo3 k;
  k.N = N;
  k.prec = (int)sizeof(T);
  k.threads = TEAM;
  k.rows_per_warp = R;
  k.smem_volume = SMEM_VOL;
  k.smem_surface = SMEM_SURF;
  k.staged = STAGEQ ? 1 : 0;
  k.fused = FUSED3 ? 1 : 0;
  k.smem_fused = FUSED3 ? SMEM_FUSED : 0;
  return k;
}

}  // namespace

namespace dg {
KernelModule3 DG_CAT(dg_module3_, DG_TAG)() {
  KernelModule3 m;
  m.N = N;
  m.prec = (int)sizeof(T);
  m.ops_bytes = &ops_bytes;
  m.pack_ops = &pack_ops;
  m.launch = &launch;
  m.info = &info;
  m.staged = STAGEQ ? 1 : 0;
  m.fused = FUSED3 ? 1 : 0;
  return m;
}
}  // namespace dg
