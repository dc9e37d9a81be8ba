// Internal interface between the runtime (runtime.cu) and the per-(N, precision)
// kernel modules (inst/k_N*_f*.cu, each its own CUDA module with its own
// __constant__ bank holding Dr, Ds and LIFT).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dg {

// Device data layout ("tile-blocked"): elements are grouped
// in tiles of TILE = 32 (one warp lane per element).  A field f of the local
// partition is stored as  f[t][n][lane]  (t = k / 32, lane = k % 32, n = node),
// i.e. offset (t*Np + n)*32 + lane, followed by the halo "ghost" face values.
// Every warp-wide access to node n of a tile is one contiguous 128 B (fp32) /
// 256 B (fp64) transaction.
constexpr int TILE = 32;

// Per-tile geometry block: geo[t][c][lane], NGEO components.
//   c = 0..3   rx, sx, ry, sy
//   c = 4+3f   nx_f,  5+3f ny_f,  6+3f hF_f                 (f = 0,1,2)
//              hF = Fsc/2 (constant material, the 1/2 of reading A3) or Fsc (material)
//   c = 13+f   Bsc_f  (+1 interior, -1 PEC, reading A7)
//   material only (NGEO_MAT):
//   c = 16, 17 1/mu, 1/eps
//   c = 18+4f  wEH = Y+/(Y+ + Y-), wHH = alpha/(Y+ + Y-), wHE = Z+/(Z+ + Z-), wEE = alpha/(Z+ + Z-)
constexpr int NGEO_CONST = 16;
constexpr int NGEO_MAT = 32;
// Compressed connectivity (KernelModule::compressed, constant material): the geometry block is
// rx, sx, ry, sy only, and vmapP holds one word per face, [t][3][32] (conn_word below).
constexpr int NGEO_Z = 4;
constexpr int ZC_PEC = -(1 << 30);  // added to a decoded point code: PEC wall (Bsc = -1, idP = idM)

// Face f's outward normal and L = |v| = sJ_f / J = Fsc_f of an affine element, from its geometric
// factors (SURVEY §8(c) O6 with rx = ys/J, sx = -yr/J, ry = -xs/J, sy = xr/J, J > 0):
//   f0: v = (yr, -xr)/J = (-sx, -sy);  f1: (ys - yr, xr - xs)/J = (rx + sx, ry + sy);  f2: (-ys, xs)/J = (-rx, -ry)
template <typename TT>
__host__ __device__ inline void face_normal(int f, TT rx, TT sx, TT ry, TT sy, TT& nx, TT& ny, TT& L) {
  const TT vx = f == 0 ? -sx : (f == 1 ? rx + sx : -rx);
  const TT vy = f == 0 ? -sy : (f == 1 ? ry + sy : -ry);
  L = sqrt(vx * vx + vy * vy);
  nx = vx / L;
  ny = vy / L;
}

// One connectivity word per (element, face), kernel-decoded into the per-point neighbour codes:
//   bits 0-1 kind: 0 PEC wall, 1 neighbour in the same tile, 2 neighbour elsewhere on this rank,
//                  3 neighbour on another rank (halo);
//   bits 2-3 the neighbour's face f' (kinds 1, 2);
//   bits 4-31 kind 1: the neighbour's column (tile lane); kind 2: its device slot;
//             kind 3: the ghost index of the face's point i = 0 (its points follow in i order).
// The neighbour's face point is i' = Nfp-1-i when faces f and f' run the same way round (traversal
// (+1, +1, -1) for faces (0, 1, 2)), else i (the O7 reversal rule).
__host__ __device__ constexpr uint32_t conn_word(uint32_t kind, uint32_t fp, uint32_t payload) {
  return (kind & 3u) | ((fp & 3u) << 2) | (payload << 4);
}

enum StageMode : int {
  MODE_FUSED_RK = 0,    // volume + flux + LIFT + LSERK4 update (one kernel per stage)
  MODE_VOLUME = 1,      // volume term only -> out (split mode, and dg_eval_rhs(1))
  MODE_SURFACE_RK = 2,  // flux + LIFT added to rhsV (in), then the LSERK4 update
  MODE_RHS = 3,         // full d/dt -> out (dg_eval_rhs(0))
  MODE_SURFACE = 4,     // surface term only -> out (dg_eval_rhs(2))
};

struct StageArgs {
  const void* q_in;        // [3][fstride] T, tile-blocked + ghosts
  void* q_out;             // [3][fstride] T   (RK modes)
  void* res;               // [3][vstride] T   (RK modes, read if a != 0, written if write_res)
  const void* rhsv;        // [3][vstride] T   (MODE_SURFACE_RK)
  void* out;               // [3][vstride] T   (MODE_VOLUME / MODE_RHS / MODE_SURFACE)
  const void* geo;         // [ntiles][NGEO][32] T
  const int32_t* vmapP;    // [ntiles][3 Nfp][32] offsets into a field (tile-blocked or ghost)
  const int32_t* tiles;    // optional list of tile (group) ids to process (NULL: 0..ntiles-1)
  const void* ops;         // packed operators (KernelModule::pack_ops layout), device memory
  int64_t fstride;         // elements between fields of q (local + ghosts)
  int64_t vstride;         // elements between fields of res / rhsv / out
  int32_t ntiles;          // number of tiles (groups, KernelModule::tile_group) to process
  int32_t write_res;       // RK modes: store the residual (0 on the last stage)
  int32_t scale_volume;    // MODE_VOLUME with material: apply 1/mu, 1/eps (dg_eval_rhs only)
  int32_t reverse;         // walk the tiles last to first (dg_options.tile_order = 1: odd LSERK4 stages)
  int32_t max_ctas;        // host only: cap on the persistent grid (0 = every resident CTA)
  double a, b, dt;         // LSERK4 stage coefficients and step
  double alpha;            // flux parameter (constant-material kernels)
};

struct KernelInfo {
  int N, prec;                       // prec = 4 or 8
  int threads, slots, row_groups, rows_per_group;
  size_t smem_bytes;
  int contraction;   // 0 FMA, 1 fp64 DMMA, 2 fp32 3xTF32 mma.sync, 3 fp32 3xTF32 tcgen05 (dg.h)
  int residual_tma;  // LSERK4 residual staged by TMA
  int teams_cap;     // DG_C
  int flags;         // bit 0 DG_FF (flux first), bit 1 DG_OG (operators via L1), bit 2 DG_FX, bit 3 DG_IL
};

struct KernelModule {
  int N = 0, prec = 0;
  // size of, and host packing into, the kernels' shared-memory operator layout:
  // Dr, Ds [Np][Np], LIFT [Np][3Nfp] (fp64 host, rounded once to T); the runtime
  // uploads the packed block once and passes it as StageArgs::ops
  size_t (*ops_bytes)() = nullptr;
  void (*pack_ops)(const double* Dr, const double* Ds, const double* LIFT, void* out) = nullptr;
  // launch one stage kernel; material selects the A12 flux
  cudaError_t (*launch)(int mode, bool material, const StageArgs& a, cudaStream_t s) = nullptr;
  KernelInfo (*info)() = nullptr;
  bool (*check_fmask)(const int* Fmask) = nullptr;
  // column swizzle of the tile-blocked layout: element `lane` of node row n lives at
  // column swz_col(swizzle, n, lane) (0 = plain layout)
  int swizzle = 0;
  // tiles per work unit: the stage kernels walk groups of tile_group consecutive tiles (4 for the
  // tcgen05 kernels: M = 128 elements); StageArgs::ntiles and ::tiles count and list GROUPS, and
  // a neighbour in the same group is read from shared memory (vmapP code < 0)
  int tile_group = 1;
  // 0: the tuned module of this (N, precision) (csrc/tune.json); 1: the tcgen05 variant module
  // (fp32 only; dg_options.kernel_variant = 1)
  int variant = 0;
  // 1: compressed connectivity for constant-material contexts (NGEO_Z geometry rows, conn words)
  int compressed = 0;
};

// Column of element e (0..31) of node row n in the tile-blocked layout, swizzle mode swm:
// e ^ (swm * s(n)).  s(n) = n & 3 for the DMMA layout (swm = 4: B-fragment loads of rows
// 4k..4k+3 conflict free); for the 3xTF32 layout (swm = 8) s(n) = (n & 3) ^ ((n >> 2) & 1),
// which keeps both of its fragment patterns bank-conflict free: A fragments read rows
// 4j + {0..3} (s = 4 distinct values for every j), C fragments rows 8t + 2i + h, i = 0..3
// (s(h), s(2+h), s(4+h), s(6+h) distinct).  An XOR of a multiple of 8 keeps 8-element groups
// contiguous, so global accesses stay 32 B-sector aligned.  The map is its own inverse.
__host__ __device__ constexpr int swz_col(int swm, int n, int e) {
  return e ^ (swm * (swm == 8 ? ((n & 3) ^ ((n >> 2) & 1)) : (n & 3)));
}

// Registry: one entry per compiled (N, prec); nullptr if not compiled.
const KernelModule* find_module(int N, int prec, int variant = 0);

}  // namespace dg
