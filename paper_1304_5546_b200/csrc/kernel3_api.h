// Internal interface between runtime3d.cu and the per-(N, precision) 3D kernel modules
// (inst/k3_N*_f*.cu; kernels3d.cuh).  SURVEY.md §8(f) row 4.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace dg {

// Per-tile geometry block of the 3D kernels: geo3[t][NGEO3][32]
//   rows 0..8   rx, ry, rz, sx, sy, sz, tx, ty, tz
//   rows 9+4f   nx_f, 10+4f ny_f, 11+4f nz_f, 12+4f hF_f = Fsc_f / 2   (faces f = 0..3)
//   rows 25+f   Bsc_f (+1 interior, -1 PEC)
constexpr int NGEO3 = 32;

struct StageArgs3 {
  const void* q_in;       // [6][fstride] T tile-blocked
  void* q_out;            // [6][fstride]
  void* res;              // [6][vstride]
  const void* rhsv;       // [6][vstride] volume term (K1 output, K2 input)
  void* out;              // [6][vstride]
  const void* geo;        // [ntiles][NGEO3][32]
  const int32_t* vmapP;   // [ntiles][4 Nfp][32] neighbour node: >= 0 offset within a global field;
                          // < 0 (KernelModule3::staged) same tile, shared-memory offset -(1 + code)
  const void* ops;        // packed operators (KernelModule3::pack_ops)
  int64_t fstride, vstride;
  int32_t ntiles, write_res, max_ctas;
  double a, b, dt, alpha;
};

struct KernelInfo3 {
  int N, prec, threads, rows_per_warp;
  size_t smem_volume, smem_surface;
  int staged;  // 1: the surface kernel stages the tile's fields in shared memory
  int fused;   // 1: the fused stage kernel (MODE_FUSED_RK) exists for this (N, precision)
  size_t smem_fused;
};

struct KernelModule3 {
  int N = 0, prec = 0;
  size_t (*ops_bytes)() = nullptr;
  void (*pack_ops)(const double* Dr, const double* Ds, const double* Dt, const double* LIFT, const int* Fmask,
                   void* out) = nullptr;
  // mode: MODE_VOLUME (K1 -> out), MODE_SURFACE_RK (K2 + rhsv -> LSERK4), MODE_RHS (K2 + rhsv -> out),
  // MODE_SURFACE (K2 alone -> out), MODE_FUSED_RK (the fused stage kernel, when `fused`)
  cudaError_t (*launch)(int mode, const StageArgs3& a, cudaStream_t s) = nullptr;
  KernelInfo3 (*info)() = nullptr;
  // 1: the surface kernel stages the tile's fields in shared memory, so a neighbour node in the same
  // 32-element tile is coded as a shared-memory offset: vmapP code = -(1 + n * 32 + lane)
  int staged = 0;
  // 1: MODE_FUSED_RK runs the fused stage kernel (volume + flux + LIFT + LSERK4 in one launch; it
  // always stages the tile's fields, so the runtime codes same-tile neighbours as shared offsets)
  int fused = 0;
};

const KernelModule3* find_module3(int N, int prec);

}  // namespace dg
