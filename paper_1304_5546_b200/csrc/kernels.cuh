// Stage kernels of the nodal-DG TM Maxwell operator for one (N, precision).
//
// Included once per translation unit (inst/k_N<N>_<prec>.cu) with
//   DG_N   polynomial degree,  DG_T  float | double,  DG_TAG  e.g. N5_f32
// so every (N, T) gets kernels with compile-time sizes (the paper's run-time
// code generation, done as C++ templates).
//
// Work decomposition:
//   * a 32-element tile is owned by a "team" of P warps (one team per CTA);
//     the volume and LIFT contractions run on one of three paths (DG_MMA):
//     FMA (one lane per element, warp g computing output rows [gR, gR+R)),
//     fp64 DMMA (mma.sync m8n8k4, 8 rows per warp) or fp32 3xTF32 (mma.sync
//     m16n8k8 with elements as M, hi/lo operand split);
//   * tile-blocked field layout (kernel_api.h): every warp access to node n of
//     a tile is one contiguous 128 B / 256 B line; a per-path column swizzle
//     keeps the shared-memory fragment loads bank-conflict free;
//   * operators in shared memory ("matrix-in-local"), packed
//     per path: broadcast LDS.128 rows (FMA) or per-lane MMA fragments;
//   * persistent CTAs walk their tiles through S shared-memory slots: TMA bulk
//     copies (cp.async.bulk + mbarrier) bring a tile's Hx, Hy, Ez, geometry
//     (and, DG_RT, residual); cp.async gathers bring cross-tile neighbour
//     traces q[vmapP] (same-tile ones are read from shared memory; vmapP is
//     fetched two tiles ahead); with one slot the next tile's TMA sources are
//     prefetched into L2 (cp.async.bulk.prefetch.L2) while the tile computes.
//
// Per tile, per stage (eq. 9 with readings A1/A2; eq. 6 chain
// rule; 1/2 eq. 5 flux, reading A3; A12 for materials; LSERK4, A10):
//   A  volume:  u = Dr Ez, v = Ds Ez;  w = Dr (rx Hy - ry Hx) + Ds (sx Hy - sy Hx)
//               rhsHx = -(ry u + sy v), rhsHy = rx u + sx v, rhsEz = w
//   B  flux:    per face point (split over the team), jumps [q] = q- - q+,
//               Fsc-scaled upwind flux written in place of q+ in shared memory
//   C  lift:    rhs += LIFT f
//   D  update:  res = a res + dt rhs;  q_out = q_in + b res
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cuda_runtime.h>

#include "kernel_api.h"

#ifndef DG_N
#error "DG_N must be defined"
#endif

#define DG_CAT2(a, b) a##b
#define DG_CAT(a, b) DG_CAT2(a, b)

namespace {

using T = DG_T;
constexpr bool F32 = sizeof(T) == 4;
constexpr int N = DG_N;
constexpr int NP = (N + 1) * (N + 2) / 2;
constexpr int NFP = N + 1;
constexpr int NF = 3 * NFP;
constexpr int TL = dg::TILE;

// Tuning knobs (per (N, precision) from csrc/tune.json via build.py; defaults
// below were measured at C4, N=5):
//   DG_R  max output rows per warp  -> team size P = ceil(Np / R)
//   DG_S  shared-memory slots per team (1 or 2)
//   DG_C  cap on resident teams per SM (sets the register budget via launch bounds)
//   DG_MMA fp64 only: volume and LIFT contractions on the FP64 tensor cores (DMMA,
//          mma.sync m8n8k4) -- one 8-row m-tile per warp -- instead of DFMA
#ifndef DG_MMA
#define DG_MMA 0  // chosen per (N, precision) by tools/tune.py
#endif
constexpr bool USE_MMA = !F32 && (DG_MMA == 1 || DG_MMA == 2 || DG_MMA == 4);
// DG_MMA=4 (fp64): the DMMA contractions split into (row group, n-tile) units -- PU warps per team (a
// multiple of 4, so every SM sub-partition holds the same number of warps: with one team per SM and
// PR = 6 row groups the one-row-group-per-warp team leaves two sub-partitions with twice the DMMAs of
// the other two); warp w owns n-tile w % 4 and row groups w / 4 + i PU / 4, so the B fragments (fields)
// it loads serve all of its units
constexpr bool DMMA_U = !F32 && DG_MMA == 4;
#ifndef DG_PU
#define DG_PU 8
#endif
// DG_WS (DMMA_U, fused stage): warp-specialised team -- the PU DMMA warps run volume -> LIFT -> LSERK4
// epilogue of tile t while WF = 4 flux warps gather the neighbour traces of tile t+1 and form its flux
// into the other of two flux buffers (mbarrier hand-off), so the flux leaves the DMMA warps' critical path
#ifndef DG_WS
#define DG_WS 0
#endif
#ifndef DG_WF
#define DG_WF 4
#endif
constexpr int WF = DG_WF;  // flux warps
// fp32 only: the same contractions as 3xTF32 products on the tensor cores (mma.sync
// m16n8k8: A = fields, elements x nodes; B = operator^T), split hi + lo so the result
// keeps fp32 accuracy -- DG_MMA=1: one 16-element m-tile per warp, two warps per tile;
// DG_MMA=2: four warps, each an m-tile x one field set (Hx, Hy | Ez)
constexpr bool USE_TF = F32 && (DG_MMA == 1 || DG_MMA == 2);
// fp32 only, DG_MMA=3: the contractions on the 5th-generation tensor cores (tcgen05.mma kind::tf32,
// accumulators and A operands in TMEM), 3xTF32 split; 128-element groups (kernels_tc.cuh)
constexpr bool USE_TC = F32 && DG_MMA == 3;
#ifndef DG_VARIANT
#define DG_VARIANT 0  // 0: the tuned module of this (N, precision); 1: the tcgen05 variant module
#endif
constexpr bool TF_SPLIT = USE_TF && DG_MMA == 2;  // 4 warps: m-tile x {Hx, Hy | Ez}
constexpr bool DMMA_SPLIT = USE_MMA && DG_MMA == 2;  // 2 PR warps: row group x {Hx, Hy | Ez}
constexpr bool WS = (DMMA_U || (USE_TF && !TF_SPLIT)) && DG_WS;  // fp64 DMMA unit teams; fp32 3xTF32 (2 m-tile warps)
// DG_WS = 2: the helper warps also run the LSERK4 epilogue of the previous tile (the DMMA warps hand the
// rhs over in a shared-memory buffer and release the tile's fields right after the LIFT: the epilogue
// reads q_in and the residual from global memory / L2)
constexpr bool WS2 = WS && DMMA_U && DG_WS == 2;
#ifndef DG_EI
#define DG_EI 0
#endif
constexpr bool EI = WS && DMMA_U && DG_EI;  // the previous tile's epilogue inside the volume k-steps
constexpr int PR = (NP + 7) / 8;                     // DMMA row groups (8 output rows each)
#ifndef DG_R
#define DG_R (sizeof(DG_T) == 4 ? 8 : 6)
#endif
constexpr int R_TARGET = USE_MMA ? 8 : DG_R;  // max rows per warp
static_assert(!DMMA_U || DG_PU % 4 == 0, "DG_PU: a multiple of 4 warps");
constexpr int UST = DG_PU / 4;                     // DMMA_U: row-group stride between a warp's units
constexpr int UW = DMMA_U ? (PR + UST - 1) / UST : 1;  // DMMA_U: units (row groups) per warp
constexpr int P = USE_TF ? (TF_SPLIT ? 4 : 2)
                          : DMMA_U ? DG_PU
                          : USE_MMA ? (DMMA_SPLIT ? 2 * PR : PR) : (NP + R_TARGET - 1) / R_TARGET;  // warps per tile
constexpr int R = (NP + P - 1) / P;                // rows per warp
constexpr int RP = P * R;                          // padded rows (extra rows are zero)
constexpr int TEAM = P * 32;

// operator columns are consumed in groups of VC: fp32 pairs (one LDS.128 = Dr,Ds of 2 columns)
constexpr int VC = F32 ? 2 : 1;
constexpr int NPC = (NP + VC - 1) / VC;  // Dr/Ds column groups
constexpr int NFC = (NF + VC - 1) / VC;  // LIFT column groups
// padded face points per element (flux buffer width; TF32: whole k-steps of 8, pad rows zero)
constexpr int NFE = USE_TF ? 8 * ((NF + 7) / 8) : NFC * VC;

// shared-memory layout (bytes; each piece a multiple of 16 B)
//   ops : DV[NPC][RP] (fp32 float4 {Dr_j, Ds_j, Dr_j+1, Ds_j+1} | fp64 double2 {Dr_j, Ds_j})
//         LV[NFC][RP] (fp32 float2 {L_m, L_m+1} | fp64 double L_m)
//   S slots of { q [3][NP][32], geo [NGEO][32], sp [3][NFE][32] }
// (vmapP codes and the LSERK4 residual live in registers)
//   MMA ops (fp64): AV[KV][P][32] double2 {Dr, Ds} and AL[KL][P][32] double LIFT, each lane
//         holding its m8n8k4 A-fragment element (row 8g + lane/4, column 4k + lane%4)
constexpr int KV = (NP + 3) / 4;  // MMA k-steps of the volume contraction
constexpr int KL = (NF + 3) / 4;  // MMA k-steps of the LIFT contraction
//   TF32 ops (fp32): BV[KVT][NT][hi, lo][32] float4 {Dr b0, Dr b1, Ds b0, Ds b1} and
//         BL[KLT][NT][32] float4 {hi b0, hi b1, lo b0, lo b1}, each lane holding its
//         m16n8k8 B-fragment elements (k = 8ks + lane%4 (+4), n = 8nt + lane/4)
constexpr int NT = (NP + 7) / 8;   // TF32 n-tiles (8 output rows each)
constexpr int KVT = (NP + 7) / 8;  // TF32 k-steps of the volume contraction
constexpr int KLT = (NF + 7) / 8;  // TF32 k-steps of the LIFT contraction
constexpr int RPL = (RP + 1) & ~1;  // LIFT rows padded to even
constexpr size_t DVB = USE_TF ? (size_t)KVT * NT * 32 * 32
                              : USE_MMA ? (size_t)KV * PR * 32 * 16 : (size_t)NPC * RP * 2 * VC * sizeof(T);
constexpr size_t LVB = USE_TF ? (size_t)KLT * NT * 32 * 16
                              : USE_MMA ? (size_t)KL * PR * 32 * 8 : (size_t)NFC * RPL * VC * sizeof(T);
constexpr size_t OPB = ((DVB + LVB + 15) / 16) * 16;
// DG_OG (tensor-core paths): the per-lane operator fragments are read from global memory
// through L1 (ld.global.nc) instead of a shared-memory copy per CTA, freeing OPB bytes of
// shared memory per team (more resident teams); every resident team shares the L1 copy
#ifndef DG_OG
#define DG_OG 0
#endif
constexpr bool OPS_GLOBAL = DG_OG;  // FMA path: the broadcast row loads go through L1 as well
constexpr size_t OPB_SMEM = OPS_GLOBAL ? 0 : OPB;
template <typename V>
__device__ __forceinline__ V ldop(const V* p) {
  if constexpr (OPS_GLOBAL) return __ldg(p);
  else return *p;
}
// Column swizzle of the tile-blocked layout: element e of node row n is stored at
// column swz_col(SWM, n, e) (kernel_api.h).  Identity for the FMA kernels; for the DMMA kernels
// it makes the B-fragment loads (4 rows x 8 elements) bank-conflict free, for the
// TF32 kernels the A-fragment loads (8 elements x 4 nodes).
constexpr int SWM = USE_MMA ? 4 : (USE_TF ? 8 : 0);  // identity for the FMA and tcgen05 kernels
__host__ __device__ constexpr int colx(int n, int e) { return dg::swz_col(SWM, n, e); }
constexpr size_t QB = (size_t)3 * NP * TL * sizeof(T);
// DG_ZC (constant-material kernels, not with DG_FX): compressed connectivity (SURVEY §8(f) row 3,
// PAPER.md:893-903).  Per tile the geometry block is only rx, sx, ry, sy (dg::NGEO_Z rows): the face
// normals and Fsc are derived on chip from them (affine elements, kernel_api.h), and instead of one
// neighbour code per face point there is one connectivity word per face (dg::conn_word), decoded into
// the per-point codes with the O7 reversal rule when the codes are fetched.
// DG_ZC = 2: geometry only -- the 4-row geometry block and derived face geometry, but one code per
// face point as uncompressed (a PEC point's code carries dg::ZC_PEC): no decode work per point.
#ifndef DG_ZC
#define DG_ZC 0
#endif
constexpr bool ZC = DG_ZC != 0;        // 4-row geometry block, face geometry derived on chip
constexpr bool ZC_CONN = DG_ZC == 1;   // one connectivity word per face (decoded per point)
__host__ __device__ constexpr int ngeo(bool mat) { return mat ? dg::NGEO_MAT : (ZC ? dg::NGEO_Z : dg::NGEO_CONST); }
__host__ __device__ constexpr size_t geo_bytes(bool mat) { return (size_t)ngeo(mat) * TL * sizeof(T); }
constexpr size_t SPB = (size_t)3 * NFE * TL * sizeof(T);
// DG_RT (TF32 path only): the LSERK4 residual of the slot's tile also arrives by TMA into
// shared memory (frees ~12 NT registers per thread) instead of a register prefetch.
#ifndef DG_RT
#define DG_RT 1
#endif
constexpr bool RES_TMA = (USE_TF || DMMA_U) && DG_RT;
// DG_TS (3xTF32 path, one slot, residual by TMA): the LSERK4 epilogue writes the new residual and q
// IN PLACE into the tile's shared-memory residual and field buffers, and one thread streams both tiles
// out with TMA bulk stores (cp.async.bulk.global.shared::cta) -- 6 bulk copies per tile instead of
// 72 scattered 4-byte STG per thread; the next tile's TMA load into the slot waits for the stores'
// shared-memory reads (cp.async.bulk.wait_group.read)
#ifndef DG_TS
#define DG_TS 0
#endif
constexpr bool TMA_ST = DG_TS != 0;  // (also the warp-specialised DMMA kernel, stage_kernel_ws)
// DG_RB (one slot, residual by TMA): the residual arrives on its own mbarrier, waited for after the
// LIFT, so the top-of-tile wait covers only the fields and geometry the volume phase needs
#ifndef DG_RB
#define DG_RB 0
#endif
constexpr bool RES_SEP = DG_RB != 0;
// DG_TS = 2 (3xTF32 path): the same in-place epilogue, but the tile is then written out by all threads
// with coalesced 16-byte streaming stores (after a barrier) instead of TMA bulk stores
constexpr bool SMEM_ST = DG_TS == 2;
// DG_FF: phase order of the fused kernels.  0: volume -> flux -> LIFT (the volume
// accumulators stay live across the flux phase); 1: flux -> volume -> LIFT (nothing but the
// face-point codes is live during the flux phase, so the peak register count drops)
#ifndef DG_FF
#define DG_FF 0
#endif
constexpr bool FLUX_FIRST = DG_FF;
// DG_FF = 2 (DMMA_U tiles): flux first WITHOUT a barrier before the volume -- the barrier the LIFT needs
// comes after the volume, so a warp's flux arithmetic and its volume DMMAs are one instruction stream
// the scheduler can interleave (the flux fills issue slots while the DMMA pipe works)
constexpr bool FLUX_FIRST_NB = DG_FF == 2;
__host__ __device__ constexpr size_t slot_bytes(bool surf, bool mat, bool rk) {
  return QB + geo_bytes(mat) + (surf ? SPB : 0) + (RES_TMA && rk ? QB : 0);
}
// DG_WP (FMA path): the volume operands W1 = rx Hy - ry Hx, W2 = sx Hy - sy Hx are formed ONCE per tile
// into a shared-memory buffer (every warp of the team splits the (node, element) pairs) instead of by
// every warp for every column it consumes -- P times fewer of those products, and the volume loop
// becomes pure loads + FMAs (4 per operator row and column)
#ifndef DG_WP
#define DG_WP 0
#endif
constexpr bool WPRE = DG_WP && DG_MMA == 0;
// DG_GL: each thread waits for its own cross-tile neighbour gathers (cp.async) right before its flux
// points -- the thread that gathers a point is the thread that forms its flux -- instead of at the top
// of the tile, so the gather latency hides behind the volume phase.  With S = 3 the gathers are also
// ISSUED at the tile's own start (after its barrier) rather than right after the previous tile's LIFT,
// where their queued copies hold up that tile's epilogue stores
#ifndef DG_GL
#define DG_GL 0
#endif
// DG_PD: L2 prefetch distance in tiles beyond the next TMA (cp.async.bulk.prefetch.L2 of tile it + PD
// (S = 1) or it + 1 + PD (S = 2, 3) while tile it computes)
#ifndef DG_PD
#define DG_PD 1
#endif
constexpr size_t BARB = 64;  // mbarriers: one per slot
constexpr size_t WPB = WPRE ? (size_t)2 * NP * TL * sizeof(T) : 0;  // DG_WP buffer: W1, W2 [NP][32]
// S = 3 is the split pipeline: two {q, geo} buffers (tile t+1's fields and geometry stream in
// while t computes) and ONE {flux, residual} buffer, refilled in the tile's own flow (residual
// by TMA at the start of the tile, next tile's neighbour gathers right after the LIFT).
__host__ __device__ constexpr size_t smem_total(int S, bool surf, bool mat, bool rk) {
  return WPB + (S == 3 ? BARB + OPB_SMEM + 2 * (QB + geo_bytes(mat)) + (surf ? SPB : 0) + (RES_TMA && rk ? QB : 0)
                       : BARB + OPB_SMEM + S * slot_bytes(surf, mat, rk));
}
// Slots per team: 2 = double-buffered (tile t+1 streams in while t computes), 1 = latency
// hidden across resident teams instead.  Measured at C4 (N=5): fp32 is issue-bound and
// prefers more resident teams (1 slot), fp64 is latency-bound and prefers 2 slots.
#ifndef DG_S
#define DG_S (sizeof(DG_T) == 4 ? 1 : 2)
#endif
__host__ __device__ constexpr int nslots(bool, bool) { return DG_S; }
constexpr bool GATHER_WAIT_LATE = DG_GL;            // each thread waits for its own gathers at its flux
constexpr bool GATHER_LATE = DG_GL && DG_S == 3;     // S = 3: and issues them at the tile's own start
static_assert(!TMA_ST || (USE_TF && RES_TMA && DG_S == 1) || (DMMA_U && DG_WS && RES_TMA),
              "DG_TS: 3xTF32 path with DG_RT = 1 and one slot, or the warp-specialised DMMA kernel with DG_RT = 1");
constexpr int CTAS_BY_SMEM = (int)((227 * 1024) / smem_total(nslots(true, false), true, false, true));
#ifndef DG_C
#define DG_C 5  // measured (C4 fp32): 5 teams x 128 registers beats 8 x 80 (spills) and 4 x 168
#endif
constexpr int MIN_CTAS = CTAS_BY_SMEM < 1 ? 1 : (CTAS_BY_SMEM > DG_C ? DG_C : CTAS_BY_SMEM);
// Face points per thread.  Face-major (when P divides Nfp): warp g owns points i = g + jP of
// every face f, k = f KPF + j, so each face's nx, ny, Fsc, Bsc are loaded once per warp;
// otherwise point m = g + kP (balanced when P does not divide Nfp).
constexpr bool FACE_MAJOR = NFP % P == 0;
constexpr int KPF = (NFP + P - 1) / P;
constexpr int KPT = FACE_MAJOR ? 3 * KPF : (NF + P - 1) / P;
__device__ __forceinline__ int point_of(int g, int k) {  // face point of slot k of warp g, NF if none
  if constexpr (FACE_MAJOR) return (k / KPF) * NFP + g + (k % KPF) * P;
  else return g + k * P < NF ? g + k * P : NF;
}
// DG_FX (3xTF32 path, one warp per m-tile): the flux is computed straight into the LIFT
// A fragments -- lane (grp, tig) of m-tile warp g owns the (element, face point) pairs
// e = 16g + grp (+8), m = 8ks + tig (+4) -- so the flux never goes through shared memory
// and no barrier separates the flux from the LIFT.  The lane also gathers its own
// cross-tile neighbour traces (cp.async into the flux buffer, read back by the same lane).
#ifndef DG_FX
#define DG_FX 0
#endif
constexpr bool FX = F32 && DG_MMA == 1 && DG_FX;
static_assert(!(FX && DG_ZC), "DG_ZC (compressed connectivity) is not implemented with DG_FX");
static_assert(!(USE_TC && DG_ZC), "DG_ZC (compressed connectivity) is not implemented in the tcgen05 kernels");
// DG_IL (3xTF32 path): issue the three split products pass by pass across all n-tiles and
// accumulators (lo*hi for all, then hi*lo, then hi*hi) instead of accumulator by accumulator,
// so consecutive MMAs into one accumulator are NT x fields instructions apart
#ifndef DG_IL
#define DG_IL 0
#endif
constexpr bool IL = DG_IL;
// DG_WB: the stage's q_out and residual stores with the default (write-back) cache policy instead
// of streaming (st.global.cs, evict-first), so the lines the stage writes last can stay in L2
// for the next stage, which walks the tiles in the opposite order (StageArgs::reverse)
#ifndef DG_WB
#define DG_WB 0
#endif
template <typename V>
__device__ __forceinline__ void st_out(V* p, const V& v) {
  if constexpr (DG_WB) *p = v;
  else __stcs(p, v);
}
constexpr int KLT_ = (NF + 7) / 8;
constexpr int KCODE = FX ? 4 * KLT_ : KPT;  // codes per thread
static_assert(!(FX && GATHER_WAIT_LATE), "DG_GL is not implemented with DG_FX");
static_assert(DG_FF != 2 || DMMA_U, "DG_FF = 2 is implemented for the DMMA_U tiles only");
struct PointElem { int m, e; };
__device__ __forceinline__ PointElem pair_of(int g, int lane, int k) {  // m = NF: no point
  if constexpr (FX) {
    const int ks = k >> 2, r = k & 3;
    const int m = 8 * ks + (lane & 3) + 4 * (r >> 1);
    return {m < NF ? m : NF, 16 * g + (lane >> 2) + 8 * (r & 1)};
  } else {
    return {point_of(g, k), lane};
  }
}

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
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory"); }

// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_barrier(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// Decode the connectivity word of face f of tile element e into face point i's neighbour code (the
// uncompressed vmapP code: >= 0 an offset into a field, < 0 a same-tile shared-memory offset,
// + dg::ZC_PEC on a PEC wall).  vstride = the ghost region's start in a field.
__device__ __forceinline__ int32_t zc_decode(uint32_t w, int f, int i, int e, int64_t vstride) {
  const uint32_t kind = w & 3u, fp = (w >> 2) & 3u, pay = w >> 4;
  if (kind == 3u) return (int32_t)(vstride + pay + i);
  if (kind == 0u) {
    const int own = fmask(f, i);
    return -(1 + own * TL + colx(own, e)) + dg::ZC_PEC;
  }
  const int ip = ((f == 2) == (fp == 2u)) ? NFP - 1 - i : i;  // O7 reversal rule
  const int rs = (ip * (2 * N + 3 - ip)) >> 1;                // row_start(ip)
  const int n2 = fp == 0u ? ip : rs + (fp == 1u ? N - ip : 0);  // fmask(fp, ip)
  if (kind == 1u) return -(1 + n2 * TL + colx(n2, (int)(pay & 31u)));
  return (int32_t)((((int64_t)(pay >> 5)) * NP + n2) * TL + colx(n2, (int)(pay & 31u)));
}

template <int MODE>
struct ModeTraits {
  static constexpr bool vol = (MODE == dg::MODE_FUSED_RK || MODE == dg::MODE_VOLUME || MODE == dg::MODE_RHS);
  static constexpr bool surf = (MODE != dg::MODE_VOLUME);
  static constexpr bool rk = (MODE == dg::MODE_FUSED_RK || MODE == dg::MODE_SURFACE_RK);
};

using DV_t = typename std::conditional<F32, float4, double2>::type;
using LV_t = typename std::conditional<F32, float2, double>::type;

// ---------------------------------------------------------------- phase A: volume
template <typename DVT>  // DVT = DV_t (a template parameter so the other precision's branch is discarded)
__device__ __forceinline__ void volume_rows(const T* __restrict__ sq, const DVT* __restrict__ DV, int n0, int lane,
                                            T rx, T sx, T ry, T sy, T (&rhx)[R], T (&rhy)[R], T (&rez)[R],
                                            const T* __restrict__ sw = nullptr) {
  T u[R], v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { u[r] = T(0); v[r] = T(0); rez[r] = T(0); }
#pragma unroll
  for (int jc = 0; jc < NPC; ++jc) {
    if constexpr (F32) {
      const int j0 = 2 * jc;
      const int j1 = (2 * jc + 1 < NP) ? 2 * jc + 1 : NP - 1;  // pad column has zero Dr/Ds
      const T ez0 = sq[(2 * NP + j0) * TL + lane], ez1 = sq[(2 * NP + j1) * TL + lane];
      T w10, w20, w11, w21;
      if constexpr (WPRE) {
        w10 = sw[j0 * TL + lane];
        w20 = sw[(NP + j0) * TL + lane];
        w11 = sw[j1 * TL + lane];
        w21 = sw[(NP + j1) * TL + lane];
      } else {
        const T hx0 = sq[(0 * NP + j0) * TL + lane], hx1 = sq[(0 * NP + j1) * TL + lane];
        const T hy0 = sq[(1 * NP + j0) * TL + lane], hy1 = sq[(1 * NP + j1) * TL + lane];
        w10 = rx * hy0 - ry * hx0;
        w20 = sx * hy0 - sy * hx0;
        w11 = rx * hy1 - ry * hx1;
        w21 = sx * hy1 - sy * hx1;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const DVT d = ldop(DV + jc * RP + n0 + r);
        u[r] = fmaf(d.x, ez0, u[r]);
        v[r] = fmaf(d.y, ez0, v[r]);
        rez[r] = fmaf(d.x, w10, rez[r]);
        rez[r] = fmaf(d.y, w20, rez[r]);
        u[r] = fmaf(d.z, ez1, u[r]);
        v[r] = fmaf(d.w, ez1, v[r]);
        rez[r] = fmaf(d.z, w11, rez[r]);
        rez[r] = fmaf(d.w, w21, rez[r]);
      }
    } else {
      const int j = jc;
      const T ez = sq[(2 * NP + j) * TL + lane];
      T w1, w2;
      if constexpr (WPRE) {
        w1 = sw[j * TL + lane];
        w2 = sw[(NP + j) * TL + lane];
      } else {
        const T hx = sq[(0 * NP + j) * TL + lane];
        const T hy = sq[(1 * NP + j) * TL + lane];
        w1 = rx * hy - ry * hx;
        w2 = sx * hy - sy * hx;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const DVT d = ldop(DV + j * RP + n0 + r);
        u[r] = fma(d.x, ez, u[r]);
        v[r] = fma(d.y, ez, v[r]);
        rez[r] = fma(d.x, w1, rez[r]);
        rez[r] = fma(d.y, w2, rez[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    rhx[r] = -(ry * u[r] + sy * v[r]);
    rhy[r] = rx * u[r] + sx * v[r];
  }
}

// ---------------------------------------------------------------- phase B: flux
// Face points point_of(g, k) of this thread's element; the Fsc-scaled flux
// (the vector f^k of eq. 8) overwrites the neighbour trace q+ in place.
// Neighbour index codes (vmapP, runtime.cu): >= 0 an offset into a field in
// global memory (gathered into sp); < 0 a neighbour in the SAME tile, read
// straight from the tile's shared-memory fields at offset -(1 + code).
// The flux of face point m (face f) of tile element e: gg = the tile's geometry + e.
// ZC: this element's face normals and half-Fsc, from rx, sx, ry, sy (dg::face_normal; rsqrt)
template <typename TT>
__device__ __forceinline__ void zc_faces(const TT* __restrict__ gg, TT (&fz)[3][3]) {
  const TT rx = gg[0 * TL], sx = gg[1 * TL], ry = gg[2 * TL], sy = gg[3 * TL];
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    const TT vx = f == 0 ? -sx : (f == 1 ? rx + sx : -rx);
    const TT vy = f == 0 ? -sy : (f == 1 ? ry + sy : -ry);
    const TT l2 = vx * vx + vy * vy, ri = rsqrt(l2);
    fz[f][0] = vx * ri;
    fz[f][1] = vy * ri;
    fz[f][2] = TT(0.5) * l2 * ri;  // Fsc / 2 = |v| / 2
  }
}

template <bool MAT, typename TT>
__device__ __forceinline__ void flux_one(const TT* __restrict__ sq, const TT* __restrict__ gg,
                                         const TT* __restrict__ sp, int code, int m, int f, int e, TT alpha,
                                         TT& fHx, TT& fHy, TT& fEz, const TT (*fzg)[3] = nullptr) {
    const int i = m - f * NFP;
    const int fm = f == 0 ? i : (f == 1 ? row_start(i) + N - i : row_start(i));
    TT nx, ny, hF, bsc;
    if constexpr (ZC && !MAT) {  // derived face geometry (zc_faces); PEC points flagged in the code
      nx = fzg[f][0];
      ny = fzg[f][1];
      hF = fzg[f][2];
      const bool pec = code < dg::ZC_PEC;
      bsc = pec ? TT(-1) : TT(1);
      if (pec) code -= dg::ZC_PEC;
    } else {
      nx = gg[(4 + 3 * f) * TL];
      ny = gg[(5 + 3 * f) * TL];
      hF = gg[(6 + 3 * f) * TL];
      bsc = gg[(13 + f) * TL];
    }
    const int pm = m * TL + colx(m, e);                               // this point in sp
    const TT* pp = code < 0 ? sq + (-1 - code) : sp + pm;             // neighbour trace, field 0
    const int fs = code < 0 ? NP * TL : NFE * TL;                     // field stride of that source
    const int om = fm * TL + colx(fm, e);                             // own face node in sq
    const TT dHx = sq[0 * NP * TL + om] - pp[0];
    const TT dHy = sq[1 * NP * TL + om] - pp[fs];
    const TT dEz = sq[2 * NP * TL + om] - bsc * pp[2 * fs];
    if constexpr (!MAT) {
      const TT ndotdH = nx * dHx + ny * dHy;
      fHx = hF * (ny * dEz + alpha * (nx * ndotdH - dHx));
      fHy = hF * (-nx * dEz + alpha * (ny * ndotdH - dHy));
      fEz = hF * (ny * dHx - nx * dHy - alpha * dEz);
    } else {
      const TT wEH = gg[(18 + 4 * f) * TL], wHH = gg[(19 + 4 * f) * TL];
      const TT wHE = gg[(20 + 4 * f) * TL], wEE = gg[(21 + 4 * f) * TL];
      const TT dHt = nx * dHy - ny * dHx;
      const TT gH = wEH * dEz + wHH * dHt;
      fHx = hF * (ny * gH);
      fHy = -hF * (nx * gH);
      fEz = -hF * (wHE * dHt + wEE * dEz);
    }
}

template <bool MAT>
__device__ __forceinline__ void flux_points(const T* __restrict__ sq, const T* __restrict__ gg, T* __restrict__ sp,
                                            const int32_t (&vmc)[KCODE], int g, int lane, T alpha) {
  if constexpr (GATHER_WAIT_LATE) {  // this thread's own neighbour gathers (DG_GL)
    if constexpr (DG_S == 2) cp_async_wait_group<1>();  // (the next tile's group may stay in flight)
    else cp_async_wait_all();
  }
  T fz[3][3];
  if constexpr (ZC && !MAT) zc_faces(gg, fz);
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int m = point_of(g, k);
    if (m >= NF) break;
    const int f = FACE_MAJOR ? k / KPF : (m < NFP ? 0 : (m < 2 * NFP ? 1 : 2));  // compile-time if face-major
    T fHx, fHy, fEz;
    flux_one<MAT>(sq, gg, sp, vmc[k], m, f, lane, alpha, fHx, fHy, fEz, fz);
    const int pm = m * TL + colx(m, lane);
    sp[0 * NFE * TL + pm] = fHx;
    sp[1 * NFE * TL + pm] = fHy;
    sp[2 * NFE * TL + pm] = fEz;
  }
}

// ---------------------------------------------------------------- DMMA (fp64 tensor core) path
// D(8x8) += A(8x4) B(4x8), fp64: lane holds A[lane/4][lane%4], B[lane%4][lane/4],
// C[lane/4][2(lane%4) + {0,1}].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Volume term of one tile on the tensor cores: warp row group g owns rows [8g, 8g+8), the
// four 8-element n-tiles of the tile are the columns.  u = Dr Ez, v = Ds Ez,
// w = Dr W1 + Ds W2 with W1 = rx Hy - ry Hx, W2 = sx Hy - sy Hx per element
// (same algebra as volume_rows), accumulated over KV k-steps of 4 nodes.  Field set FS
// (as tf_tile): 0 all, 1 only u, v (-> Hx, Hy), 2 only w (-> Ez).
template <int FS, typename AVT>
__device__ __forceinline__ void volume_mma(const double* __restrict__ sq, const double* __restrict__ sg,
                                           const AVT* __restrict__ AV, int g, int lane, double (&u)[4][2],
                                           double (&v)[4][2], double (&w)[4][2]) {
  double rxb[4], sxb[4], ryb[4], syb[4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const int eb = 8 * nt + (lane >> 2);
    rxb[nt] = sg[0 * TL + eb];
    sxb[nt] = sg[1 * TL + eb];
    ryb[nt] = sg[2 * TL + eb];
    syb[nt] = sg[3 * TL + eb];
    u[nt][0] = u[nt][1] = v[nt][0] = v[nt][1] = w[nt][0] = w[nt][1] = 0.0;
  }
  constexpr bool UV = FS != 2, WW = FS != 1;
  double w2acc[4][2] = {};  // Ds W2 in its own accumulator: 4 independent DMMA chains per n-tile
#pragma unroll
  for (int ks = 0; ks < KV; ++ks) {
    const int j = 4 * ks + (lane & 3);
    const int jc = j < NP ? j : NP - 1;  // padded k rows: A is zero there
    const AVT a = ldop(AV + (ks * PR + g) * 32 + lane);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int addr = jc * TL + colx(jc, 8 * nt + (lane >> 2));
      if constexpr (UV) {
        const double ez = sq[2 * NP * TL + addr];
        dmma(u[nt][0], u[nt][1], a.x, ez);
        dmma(v[nt][0], v[nt][1], a.y, ez);
      }
      if constexpr (WW) {
        const double hx = sq[0 * NP * TL + addr], hy = sq[1 * NP * TL + addr];
        dmma(w[nt][0], w[nt][1], a.x, rxb[nt] * hy - ryb[nt] * hx);
        dmma(w2acc[nt][0], w2acc[nt][1], a.y, sxb[nt] * hy - syb[nt] * hx);
      }
    }
  }
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    w[nt][0] += w2acc[nt][0];
    w[nt][1] += w2acc[nt][1];
  }
}

// rhs += LIFT f on the tensor cores (f in sp, swizzled [c][NF][32]); fields of set FS.
template <int FS>
__device__ __forceinline__ void lift_mma(const double* __restrict__ sp, const double* __restrict__ AL, int g,
                                         int lane, double (&rhx)[4][2], double (&rhy)[4][2], double (&rez)[4][2]) {
#pragma unroll
  for (int ks = 0; ks < KL; ++ks) {
    const int m = 4 * ks + (lane & 3);
    const int mc = m < NF ? m : NF - 1;
    const double a = ldop(AL + (ks * PR + g) * 32 + lane);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int addr = mc * TL + colx(mc, 8 * nt + (lane >> 2));
      if constexpr (FS != 2) {
        dmma(rhx[nt][0], rhx[nt][1], a, sp[0 * NFE * TL + addr]);
        dmma(rhy[nt][0], rhy[nt][1], a, sp[1 * NFE * TL + addr]);
      }
      if constexpr (FS != 1) dmma(rez[nt][0], rez[nt][1], a, sp[2 * NFE * TL + addr]);
    }
  }
}

// ---------------------------------------------------------------- 3xTF32 (fp32 tensor core) path
// D(16x8) += A(16x8) B(8x8), tf32 operands, fp32 accumulation.  Lane (grp = lane/4,
// tig = lane%4) holds A[grp][tig], A[grp+8][tig], A[grp][tig+4], A[grp+8][tig+4];
// B[tig][grp], B[tig+4][grp]; C[grp][2tig + {0,1}], C[grp+8][2tig + {0,1}].
__device__ __forceinline__ void tmma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// x = hi + lo: hi = x rounded to nearest (ties away) at tf32's 10 mantissa bits by integer
// add + mask -- the same rounding as cvt.rna.tf32 for finite x, without its NaN/Inf
// handling (4 more instructions) -- and lo = (x - hi) rounded the same way.  x - hi is exact
// in fp32 but has up to 13 mantissa bits below tf32's; handing it to the MMA unrounded would
// TRUNCATE it (a biased 2^-21 |x| error); rounded, |x - hi - lo| <= 2^-22 |x|, unbiased -- the
// same treatment the host gives the operator's lo parts (pack_ops)
__device__ __forceinline__ uint32_t rna_tf32(uint32_t u) { return (u + 0x1000u) & 0xFFFFE000u; }
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = rna_tf32(__float_as_uint(x));
  lo = rna_tf32(__float_as_uint(x - __uint_as_float(hi)));
}
// c += A B with A = ah + al, B = bh + bl; the al bl term (~2^-22 relative) is dropped
__device__ __forceinline__ void tmma3(float (&c)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], float bh0,
                                      float bh1, float bl0, float bl1) {
  tmma(c, al, __float_as_uint(bh0), __float_as_uint(bh1));
  tmma(c, ah, __float_as_uint(bl0), __float_as_uint(bl1));
  tmma(c, ah, __float_as_uint(bh0), __float_as_uint(bh1));
}

// One tile on the 3xTF32 path (fp32): elements are the MMA rows -- the warp owns
// elements e = 16 mt + lane/4 (+8) of m-tile mt -- and each n-tile is 8 output rows, so
// the padding is only Np -> 8 NT.  Volume (u = Dr Ez, v = Ds Ez, w = Dr W1 + Ds W2, as
// volume_rows) -> flux (flux_points, one lane per element, all P warps) -> LIFT ->
// material scaling -> LSERK4.  FS selects the output fields the warp owns: 0 all three
// (DG_MMA=1: P = 2 warps, one per m-tile), 1 = Hx, Hy (from u, v) and 2 = Ez (from w)
// (DG_MMA=2: P = 4 warps, m-tile x field set: half the registers per warp, twice the warps).
// C-fragment register r of n-tile nt is element ee[r >> 1], row 8nt + 2(lane%4) + (r & 1).
struct NoHook {
  __device__ void operator()() const {}
};
// WSM (warp-specialised kernel, stage_kernel_ws): the flux is formed by the flux warps -- flux_wait()
// blocks until this tile's flux is in sp, flux_done() releases sp after the LIFT has read it
template <int MODE, bool MAT, int FS, bool WSM = false, typename TT, typename HOOK, typename FW = NoHook,
          typename FD = NoHook>
__device__ __forceinline__ void tf_tile(const dg::StageArgs& p, const TT* __restrict__ sq, const TT* __restrict__ sg,
                                        TT* __restrict__ sp, const TT* __restrict__ sr,
                                        const unsigned char* __restrict__ ops, const int32_t (&vmc)[KCODE],
                                        int tile, int g, int mt, int lane, TT alpha, bool read_res,
                                        const HOOK& after_lift, const FW& flux_wait = FW(), const FD& flux_done = FD()) {
  using MT = ModeTraits<MODE>;
  static_assert(!WSM || (!FLUX_FIRST && !FX && MODE == dg::MODE_FUSED_RK), "warp-specialised tiles: fused stage");
  constexpr int NFLD = FS == 0 ? 3 : (FS == 1 ? 2 : 1);  // output fields F0 .. F0 + NFLD - 1
  constexpr int F0 = FS == 2 ? 2 : 0;
  constexpr bool UV = FS != 2, WW = FS != 1;  // this warp forms u, v (Hx, Hy) / w (Ez)
  const int tig = lane & 3;
  const int ee[2] = {16 * mt + (lane >> 2), 16 * mt + (lane >> 2) + 8};
  // Lane-invariant shared-memory offsets.  A fragments read node rows 8ks + 4kh + tig, whose
  // swizzle (swz_col: s = tig ^ kh) depends only on kh (compile-time per register): row offsets
  // are compile-time.  Rows past Np / 3Nfp meet zero B rows; they read the next field, the
  // geometry block (fields) or zeroed pad rows (flux), all finite.  C fragments: row
  // 8nt + 2tig + h, element ee[i].
  int abase[2][2];  // [kh][i]
#pragma unroll
  for (int kh = 0; kh < 2; ++kh)
#pragma unroll
    for (int i = 0; i < 2; ++i) abase[kh][i] = tig * TL + colx(4 * kh + tig, ee[i]);
  int cbase[4];  // C register r -> row (2tig + (r & 1)) offset + swizzled column of ee[r >> 1]
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int n = 2 * tig + (r & 1);
    cbase[r] = n * TL + colx(n, ee[r >> 1]);
  }
  auto row_ok = [&](int nt, int r) { return NT * 8 == NP || nt < NT - 1 || 8 * nt + 2 * tig + (r & 1) < NP; };
  const int64_t tbase = (int64_t)tile * NP * TL;
  if constexpr (FLUX_FIRST && MT::surf && !FX) {
    flux_points<MAT>(sq, sg + lane, sp, vmc, g, lane, alpha);
    __syncthreads();
  }
  TT acc[NFLD][NT][4];  // acc[f]: field F0 + f
  if constexpr (MT::vol) {
    TT rxe[2], sxe[2], rye[2], sye[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      rxe[i] = sg[0 * TL + ee[i]];
      sxe[i] = sg[1 * TL + ee[i]];
      rye[i] = sg[2 * TL + ee[i]];
      sye[i] = sg[3 * TL + ee[i]];
    }
    // UV: u accumulates in acc[0], v in acc[1] (turned into rhsHx, rhsHy below); WW: w in acc[NFLD-1]
#pragma unroll
    for (int f = 0; f < NFLD; ++f)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[f][nt][r] = TT(0);
    const float4* BV = reinterpret_cast<const float4*>(ops) + lane;
#pragma unroll
    for (int ks = 0; ks < KVT; ++ks) {
      uint32_t ezh[4], ezl[4], w1h[4], w1l[4], w2h[4], w2l[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {  // A register r: element ee[r & 1], node 8ks + tig + 4(r >> 1)
        const int i = r & 1;
        const TT* a = sq + abase[r >> 1][i] + (8 * ks + 4 * (r >> 1)) * TL;
        if constexpr (UV) split_tf32(a[2 * NP * TL], ezh[r], ezl[r]);
        if constexpr (WW) {
          const TT hx = a[0], hy = a[NP * TL];
          split_tf32(rxe[i] * hy - rye[i] * hx, w1h[r], w1l[r]);
          split_tf32(sxe[i] * hy - sye[i] * hx, w2h[r], w2l[r]);
        }
      }
      if constexpr (IL) {
        float4 bh[NT], bl[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          bh[nt] = ldop(BV + (ks * NT + nt) * 64);
          bl[nt] = ldop(BV + (ks * NT + nt) * 64 + 32);
        }
        auto U = [](float x) { return __float_as_uint(x); };
        // pass p: (A part, B part) = (lo, hi), (hi, lo), (hi, hi); small terms first
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const float4 b = pass == 1 ? bl[nt] : bh[nt];
            if constexpr (UV) {
              tmma(acc[0][nt], pass == 0 ? ezl : ezh, U(b.x), U(b.y));
              tmma(acc[1][nt], pass == 0 ? ezl : ezh, U(b.z), U(b.w));
            }
            if constexpr (WW) tmma(acc[NFLD - 1][nt], pass == 0 ? w1l : w1h, U(b.x), U(b.y));
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const float4 b = pass == 1 ? bl[nt] : bh[nt];
            if constexpr (WW) tmma(acc[NFLD - 1][nt], pass == 0 ? w2l : w2h, U(b.z), U(b.w));
          }
        }
      } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float4 bh = ldop(BV + (ks * NT + nt) * 64);  // hi and lo: 32 lanes x 16 B contiguous each
        const float4 bl = ldop(BV + (ks * NT + nt) * 64 + 32);
        if constexpr (UV) {
          tmma3(acc[0][nt], ezh, ezl, bh.x, bh.y, bl.x, bl.y);
          tmma3(acc[1][nt], ezh, ezl, bh.z, bh.w, bl.z, bl.w);
        }
        if constexpr (WW) {
          tmma3(acc[NFLD - 1][nt], w1h, w1l, bh.x, bh.y, bl.x, bl.y);
          tmma3(acc[NFLD - 1][nt], w2h, w2l, bh.z, bh.w, bl.z, bl.w);
        }
      }
      }
    }
    if constexpr (UV) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int i = r >> 1;
          const TT u = acc[0][nt][r], v = acc[1][nt][r];
          acc[0][nt][r] = -(rye[i] * u + sye[i] * v);
          acc[1][nt][r] = rxe[i] * u + sxe[i] * v;
        }
    }
  } else if constexpr (MODE == dg::MODE_SURFACE_RK) {
    const TT* __restrict__ rv = static_cast<const TT*>(p.rhsv) + tbase;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int f = 0; f < NFLD; ++f)
          acc[f][nt][r] = row_ok(nt, r) ? rv[(F0 + f) * p.vstride + 8 * nt * TL + cbase[r]] : TT(0);
  } else {
#pragma unroll
    for (int f = 0; f < NFLD; ++f)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[f][nt][r] = TT(0);
  }
  // LSERK4 residual -> registers (DG_RT=0; in flight during the surface phase)
  TT rr[NFLD][NT][4];
  if constexpr (MT::rk && !RES_TMA) {
    if (read_res) {
      const TT* __restrict__ res = static_cast<const TT*>(p.res) + tbase;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int f = 0; f < NFLD; ++f)
            rr[f][nt][r] = row_ok(nt, r) ? __ldcs(res + (F0 + f) * p.vstride + 8 * nt * TL + cbase[r]) : TT(0);
    }
  }
  if constexpr (MT::surf) {
    if constexpr (WSM) {
      flux_wait();
    } else if constexpr (!FLUX_FIRST && !FX) {
      flux_points<MAT>(sq, sg + lane, sp, vmc, g, lane, alpha);
      __syncthreads();
    }
    const float4* BL = reinterpret_cast<const float4*>(ops + DVB) + lane;
#pragma unroll
    for (int ks = 0; ks < KLT; ++ks) {
      uint32_t fh[NFLD][4], fl[NFLD][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if constexpr (FX) {  // A register r: element ee[r & 1], face point 8ks + tig + 4(r >> 1)
          const int m = 8 * ks + tig + 4 * (r >> 1);
          TT fv[3] = {TT(0), TT(0), TT(0)};
          if (m < NF) {
            const int f = m < NFP ? 0 : (m < 2 * NFP ? 1 : 2);
            flux_one<MAT>(sq, sg + ee[r & 1], sp, vmc[4 * ks + r], m, f, ee[r & 1], alpha, fv[0], fv[1], fv[2]);
          }
#pragma unroll
          for (int f = 0; f < NFLD; ++f) split_tf32(fv[F0 + f], fh[f][r], fl[f][r]);
        } else {
          const TT* a = sp + abase[r >> 1][r & 1] + (8 * ks + 4 * (r >> 1)) * TL;
#pragma unroll
          for (int f = 0; f < NFLD; ++f) split_tf32(a[(F0 + f) * NFE * TL], fh[f][r], fl[f][r]);
        }
      }
      if constexpr (IL) {
        float4 b[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = ldop(BL + (ks * NT + nt) * 32);
#pragma unroll
        for (int pass = 0; pass < 3; ++pass)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int f = 0; f < NFLD; ++f) {
              const float x = pass == 1 ? b[nt].z : b[nt].x, y = pass == 1 ? b[nt].w : b[nt].y;
              tmma(acc[f][nt], pass == 0 ? fl[f] : fh[f], __float_as_uint(x), __float_as_uint(y));
            }
      } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float4 b = ldop(BL + (ks * NT + nt) * 32);
#pragma unroll
        for (int f = 0; f < NFLD; ++f) tmma3(acc[f][nt], fh[f], fl[f], b.x, b.y, b.z, b.w);
      }
      }
    }
  }
  if constexpr (WSM) flux_done();
  after_lift();  // split pipeline (S = 3): the flux buffer is free, the residual must be in
  if constexpr (MAT) {
    if (MODE != dg::MODE_VOLUME || p.scale_volume) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const TT imu = sg[16 * TL + ee[i]], ieps = sg[17 * TL + ee[i]];
#pragma unroll
        for (int f = 0; f < NFLD; ++f)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) acc[f][nt][2 * i + h] *= (F0 + f == 2 ? ieps : imu);
      }
    }
  }
  const TT a = static_cast<TT>(p.a), b = static_cast<TT>(p.b), dt = static_cast<TT>(p.dt);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (!row_ok(nt, r)) continue;
      const int o = 8 * nt * TL + cbase[r];
      if constexpr (MT::rk) {
        TT* __restrict__ res = static_cast<TT*>(p.res) + tbase;
        TT* __restrict__ qo = static_cast<TT*>(p.q_out) + tbase;
#pragma unroll
        for (int f = 0; f < NFLD; ++f) {
          const int c = F0 + f;
          TT rs = dt * acc[f][nt][r];
          if (read_res) rs = fma(a, RES_TMA ? sr[c * NP * TL + o] : rr[f][nt][r], rs);
          const TT qn = fma(b, rs, sq[c * NP * TL + o]);
          if constexpr (TMA_ST) {  // in place; the bulk stores follow the tile (stage_kernel)
            const_cast<TT*>(sr)[c * NP * TL + o] = rs;
            const_cast<TT*>(sq)[c * NP * TL + o] = qn;
          } else {
            if (p.write_res) st_out(res + c * p.vstride + o, rs);
            st_out(qo + c * p.fstride + o, qn);
          }
        }
      } else {
        TT* __restrict__ out = static_cast<TT*>(p.out) + tbase;
#pragma unroll
        for (int f = 0; f < NFLD; ++f) out[(F0 + f) * p.vstride + o] = acc[f][nt][r];
      }
    }
  if constexpr (TMA_ST && !SMEM_ST && MT::rk) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ---------------------------------------------------------------- phase C: lift
template <typename LVT>
__device__ __forceinline__ void lift_rows(const T* __restrict__ sp, const LVT* __restrict__ LV, int n0, int lane,
                                          T (&rhx)[R], T (&rhy)[R], T (&rez)[R]) {
#pragma unroll
  for (int mc = 0; mc < NFC; ++mc) {
    if constexpr (F32) {
      const int m0 = 2 * mc, m1 = 2 * mc + 1;  // m1 may be the zero pad column
      const T a0 = sp[(0 * NFE + m0) * TL + lane], a1 = sp[(0 * NFE + m1) * TL + lane];
      const T b0 = sp[(1 * NFE + m0) * TL + lane], b1 = sp[(1 * NFE + m1) * TL + lane];
      const T c0 = sp[(2 * NFE + m0) * TL + lane], c1 = sp[(2 * NFE + m1) * TL + lane];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const LVT l = ldop(LV + mc * RPL + n0 + r);
        rhx[r] = fmaf(l.x, a0, rhx[r]);
        rhy[r] = fmaf(l.x, b0, rhy[r]);
        rez[r] = fmaf(l.x, c0, rez[r]);
        rhx[r] = fmaf(l.y, a1, rhx[r]);
        rhy[r] = fmaf(l.y, b1, rhy[r]);
        rez[r] = fmaf(l.y, c1, rez[r]);
      }
    } else {
      const int m = mc;
      const T a0 = sp[(0 * NFE + m) * TL + lane];
      const T b0 = sp[(1 * NFE + m) * TL + lane];
      const T c0 = sp[(2 * NFE + m) * TL + lane];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const LVT l = ldop(LV + m * RPL + n0 + r);
        rhx[r] = fma(l, a0, rhx[r]);
        rhy[r] = fma(l, b0, rhy[r]);
        rez[r] = fma(l, c0, rez[r]);
      }
    }
  }
}

// One tile on the DMMA path (fp64): volume (tensor cores) -> flux (one lane per
// element, as the FMA path) -> LIFT (tensor cores) -> material scaling -> LSERK4
// update.  Each lane owns C-fragment rows n = 8 rg + lane/4 (rg = the warp's row group)
// and the element pairs e = 8nt + 2(lane%4) + {0,1}; stores are 16 B pairs (e, e+1 stay
// adjacent under the column swizzle).  FS = field set (volume_mma): DG_MMA=2 gives each
// row group two warps, one for Hx, Hy and one for Ez.
template <int MODE, bool MAT, int FS, typename TT, typename HOOK>
__device__ __forceinline__ void mma_tile(const dg::StageArgs& p, const TT* __restrict__ sq, const TT* __restrict__ sg,
                                         TT* __restrict__ sp, const unsigned char* __restrict__ ops,
                                         const int32_t (&vmc)[KCODE], int tile, int g, int rg, int lane, TT alpha,
                                         bool read_res, const HOOK& after_lift) {
  using MT = ModeTraits<MODE>;
  using V2 = typename std::conditional<sizeof(TT) == 8, double2, float2>::type;
  constexpr bool ACT[3] = {FS != 2, FS != 2, FS != 1};  // output fields of this warp
  const int n = 8 * rg + (lane >> 2);  // this lane's output row
  const int nc = n < NP ? n : NP - 1;
  if constexpr (FLUX_FIRST && MT::surf) {
    flux_points<MAT>(sq, sg + lane, sp, vmc, g, lane, alpha);
    __syncthreads();
  }
  TT rhx[4][2], rhy[4][2], rez[4][2];
  if constexpr (MT::vol) {
    TT u[4][2], v[4][2];
    volume_mma<FS>(sq, sg, reinterpret_cast<const V2*>(ops), rg, lane, u, v, rez);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ec = 8 * nt + 2 * (lane & 3) + h;
        const TT rx = sg[0 * TL + ec], sx = sg[1 * TL + ec], ry = sg[2 * TL + ec], sy = sg[3 * TL + ec];
        rhx[nt][h] = -(ry * u[nt][h] + sy * v[nt][h]);
        rhy[nt][h] = rx * u[nt][h] + sx * v[nt][h];
      }
  } else if constexpr (MODE == dg::MODE_SURFACE_RK) {
    const TT* __restrict__ rv = static_cast<const TT*>(p.rhsv);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t off = ((int64_t)tile * NP + nc) * TL + colx(nc, 8 * nt + 2 * (lane & 3));
      const V2 x = *reinterpret_cast<const V2*>(rv + off);
      const V2 y = *reinterpret_cast<const V2*>(rv + p.vstride + off);
      const V2 z = *reinterpret_cast<const V2*>(rv + 2 * p.vstride + off);
      rhx[nt][0] = x.x; rhx[nt][1] = x.y;
      rhy[nt][0] = y.x; rhy[nt][1] = y.y;
      rez[nt][0] = z.x; rez[nt][1] = z.y;
    }
  } else {
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) rhx[nt][h] = rhy[nt][h] = rez[nt][h] = TT(0);
  }
  // LSERK4 residual pairs -> registers (in flight during the surface phase)
  V2 rr[3][4];
  if constexpr (MT::rk) {
    if (read_res) {
      const TT* __restrict__ res = static_cast<const TT*>(p.res);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int64_t off = ((int64_t)tile * NP + nc) * TL + colx(nc, 8 * nt + 2 * (lane & 3));
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (ACT[c]) rr[c][nt] = __ldcs(reinterpret_cast<const V2*>(res + c * p.vstride + off));
      }
    }
  }
  if constexpr (MT::surf) {
    if constexpr (!FLUX_FIRST) {
      flux_points<MAT>(sq, sg + lane, sp, vmc, g, lane, alpha);
      __syncthreads();
    }
    lift_mma<FS>(sp, reinterpret_cast<const TT*>(ops + DVB), rg, lane, rhx, rhy, rez);
  }
  after_lift();
  if constexpr (MAT) {
    if (MODE != dg::MODE_VOLUME || p.scale_volume) {
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int ec = 8 * nt + 2 * (lane & 3) + h;
          const TT imu = sg[16 * TL + ec], ieps = sg[17 * TL + ec];
          rhx[nt][h] *= imu;
          rhy[nt][h] *= imu;
          rez[nt][h] *= ieps;
        }
    }
  }
  if (n >= NP) return;
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const int col = colx(n, 8 * nt + 2 * (lane & 3));
    const int64_t off = ((int64_t)tile * NP + n) * TL + col;
    const TT r3[3][2] = {{rhx[nt][0], rhx[nt][1]}, {rhy[nt][0], rhy[nt][1]}, {rez[nt][0], rez[nt][1]}};
    if constexpr (MT::rk) {
      TT* __restrict__ res = static_cast<TT*>(p.res);
      TT* __restrict__ qo = static_cast<TT*>(p.q_out);
      const TT a = static_cast<TT>(p.a), b = static_cast<TT>(p.b), dt = static_cast<TT>(p.dt);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (!ACT[c]) continue;
        V2 rs;
        rs.x = dt * r3[c][0];
        rs.y = dt * r3[c][1];
        if (read_res) {
          rs.x = fma(a, rr[c][nt].x, rs.x);
          rs.y = fma(a, rr[c][nt].y, rs.y);
        }
        if (p.write_res) st_out(reinterpret_cast<V2*>(res + c * p.vstride + off), rs);
        const V2 qi = *reinterpret_cast<const V2*>(sq + (c * NP + n) * TL + col);
        V2 qn;
        qn.x = fma(b, rs.x, qi.x);
        qn.y = fma(b, rs.y, qi.y);
        st_out(reinterpret_cast<V2*>(qo + c * p.fstride + off), qn);
      }
    } else {
      TT* __restrict__ out = static_cast<TT*>(p.out);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (!ACT[c]) continue;
        V2 o;
        o.x = r3[c][0];
        o.y = r3[c][1];
        *reinterpret_cast<V2*>(out + c * p.vstride + off) = o;
      }
    }
  }
}

// One tile on the DMMA path split into (row group, n-tile) units (DG_MMA=4): warp g owns n-tile
// nt = g % 4 (elements 8nt .. 8nt+7) and row groups rg_i = g / 4 + i UST (i < UW; rg_i >= PR: none).
// Per k-step the warp loads the B fragments of its n-tile once (Ez, and W1, W2 formed from Hx, Hy)
// and issues them against the A fragments (operator rows) of each of its row groups.  Same algebra as
// mma_tile: u = Dr Ez, v = Ds Ez, w = Dr W1 + Ds W2 -> flux -> rhs += LIFT f -> 1/mu, 1/eps -> LSERK4.
// WSM (warp-specialised kernel, stage_kernel_ws): the flux is formed by the flux warps -- flux_wait()
// blocks until this tile's flux is in sp, flux_done() releases sp after the LIFT has read it
// WSE (DG_WS = 2): the LSERK4 epilogue runs in the helper warps -- after the LIFT and the material
// scaling this tile's rhs goes to the shared-memory accumulator buffer sacc ([3][NP][32], the tile
// layout) instead of through the update
template <int MODE, bool MAT, bool WSM = false, bool WSE = false, typename TT, typename HOOK, typename FW = NoHook,
          typename FD = NoHook>
__device__ __forceinline__ void mma_tile_u(const dg::StageArgs& p, const TT* __restrict__ sq, const TT* __restrict__ sg,
                                           TT* __restrict__ sp, const TT* __restrict__ sr,
                                           const unsigned char* __restrict__ ops, const int32_t (&vmc)[KCODE],
                                           int tile, int g, int lane, TT alpha, bool read_res, const HOOK& after_lift,
                                           const FW& flux_wait = FW(), const FD& flux_done = FD(),
                                           TT* __restrict__ sacc = nullptr) {
  using MT = ModeTraits<MODE>;
  static_assert(!WSM || (!FLUX_FIRST && MODE == dg::MODE_FUSED_RK), "warp-specialised tiles: fused stage, volume first");
  using V2 = double2;
  const int nt = g & 3, rg0 = g >> 2;
  auto rg_of = [&](int i) { return rg0 + i * UST; };
  auto unit_ok = [&](int i) { return (UW - 1) * UST + (P / 4 - 1) < PR || rg_of(i) < PR; };  // compile-time when full
  const int eb = 8 * nt + (lane >> 2);             // B-fragment element of this lane
  const int ec0 = 8 * nt + 2 * (lane & 3);         // C-fragment elements ec0, ec0 + 1
  if constexpr (FLUX_FIRST && MT::surf) {
    flux_points<MAT>(sq, sg + lane, sp, vmc, g, lane, alpha);
    if constexpr (!FLUX_FIRST_NB) __syncthreads();
  }
  TT rhx[UW][2], rhy[UW][2], rez[UW][2];
  if constexpr (MT::vol) {
    const TT rxb = sg[0 * TL + eb], sxb = sg[1 * TL + eb], ryb = sg[2 * TL + eb], syb = sg[3 * TL + eb];
    TT u[UW][2], v[UW][2], w2a[UW][2];
#pragma unroll
    for (int i = 0; i < UW; ++i) u[i][0] = u[i][1] = v[i][0] = v[i][1] = rez[i][0] = rez[i][1] = w2a[i][0] = w2a[i][1] = TT(0);
    const V2* AV = reinterpret_cast<const V2*>(ops);
#pragma unroll
    for (int ks = 0; ks < KV; ++ks) {
      const int j = 4 * ks + (lane & 3);
      const int jc = j < NP ? j : NP - 1;  // padded k rows: A is zero there
      const int addr = jc * TL + colx(jc, eb);
      const TT ez = sq[2 * NP * TL + addr], hx = sq[addr], hy = sq[NP * TL + addr];
      const TT w1 = rxb * hy - ryb * hx, w2 = sxb * hy - syb * hx;
#pragma unroll
      for (int i = 0; i < UW; ++i) {
        if (!unit_ok(i)) continue;
        const V2 a = ldop(AV + (ks * PR + rg_of(i)) * 32 + lane);
        dmma(u[i][0], u[i][1], a.x, ez);
        dmma(v[i][0], v[i][1], a.y, ez);
        dmma(rez[i][0], rez[i][1], a.x, w1);
        dmma(w2a[i][0], w2a[i][1], a.y, w2);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ec = ec0 + h;
      const TT rx = sg[0 * TL + ec], sx = sg[1 * TL + ec], ry = sg[2 * TL + ec], sy = sg[3 * TL + ec];
#pragma unroll
      for (int i = 0; i < UW; ++i) {
        rez[i][h] += w2a[i][h];
        rhx[i][h] = -(ry * u[i][h] + sy * v[i][h]);
        rhy[i][h] = rx * u[i][h] + sx * v[i][h];
      }
    }
  } else if constexpr (MODE == dg::MODE_SURFACE_RK) {
    const TT* __restrict__ rv = static_cast<const TT*>(p.rhsv);
#pragma unroll
    for (int i = 0; i < UW; ++i) {
      if (!unit_ok(i)) continue;
      const int n = 8 * rg_of(i) + (lane >> 2), nc = n < NP ? n : NP - 1;
      const int64_t off = ((int64_t)tile * NP + nc) * TL + colx(nc, ec0);
      const V2 x = *reinterpret_cast<const V2*>(rv + off);
      const V2 y = *reinterpret_cast<const V2*>(rv + p.vstride + off);
      const V2 z = *reinterpret_cast<const V2*>(rv + 2 * p.vstride + off);
      rhx[i][0] = x.x; rhx[i][1] = x.y;
      rhy[i][0] = y.x; rhy[i][1] = y.y;
      rez[i][0] = z.x; rez[i][1] = z.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < UW; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) rhx[i][h] = rhy[i][h] = rez[i][h] = TT(0);
  }
  V2 rr[UW][3];  // LSERK4 residual pairs (in flight during the surface phase; RES_TMA: staged in sr)
  if constexpr (MT::rk && !RES_TMA && !WSE) {
    if (read_res) {
      const TT* __restrict__ res = static_cast<const TT*>(p.res);
#pragma unroll
      for (int i = 0; i < UW; ++i) {
        if (!unit_ok(i)) continue;
        const int n = 8 * rg_of(i) + (lane >> 2), nc = n < NP ? n : NP - 1;
        const int64_t off = ((int64_t)tile * NP + nc) * TL + colx(nc, ec0);
#pragma unroll
        for (int c = 0; c < 3; ++c) rr[i][c] = __ldcs(reinterpret_cast<const V2*>(res + c * p.vstride + off));
      }
    }
  }
  if constexpr (MT::surf) {
    if constexpr (WSM) {
      flux_wait();
    } else if constexpr (!FLUX_FIRST) {
      flux_points<MAT>(sq, sg + lane, sp, vmc, g, lane, alpha);
      __syncthreads();
    } else if constexpr (FLUX_FIRST_NB) {
      __syncthreads();  // every warp's flux is in sp
    }
    const TT* AL = reinterpret_cast<const TT*>(ops + DVB);
#pragma unroll
    for (int ks = 0; ks < KL; ++ks) {
      const int m = 4 * ks + (lane & 3);
      const int mc = m < NF ? m : NF - 1;
      const int addr = mc * TL + colx(mc, eb);
      const TT f0 = sp[0 * NFE * TL + addr], f1 = sp[1 * NFE * TL + addr], f2 = sp[2 * NFE * TL + addr];
#pragma unroll
      for (int i = 0; i < UW; ++i) {
        if (!unit_ok(i)) continue;
        const TT a = ldop(AL + (ks * PR + rg_of(i)) * 32 + lane);
        dmma(rhx[i][0], rhx[i][1], a, f0);
        dmma(rhy[i][0], rhy[i][1], a, f1);
        dmma(rez[i][0], rez[i][1], a, f2);
      }
    }
  }
  if constexpr (WSM) flux_done();
  if constexpr (!WSE) after_lift();
  if constexpr (MAT) {
    if (MODE != dg::MODE_VOLUME || p.scale_volume) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const TT imu = sg[16 * TL + ec0 + h], ieps = sg[17 * TL + ec0 + h];
#pragma unroll
        for (int i = 0; i < UW; ++i) {
          rhx[i][h] *= imu;
          rhy[i][h] *= imu;
          rez[i][h] *= ieps;
        }
      }
    }
  }
  if constexpr (WSE) {  // rhs -> sacc (after_lift: the tile's buffers are released, sacc is free)
    after_lift();
#pragma unroll
    for (int i = 0; i < UW; ++i) {
      if (!unit_ok(i)) continue;
      const int n = 8 * rg_of(i) + (lane >> 2);
      if (n >= NP) continue;
      const int col = colx(n, ec0);
      const TT r3[3][2] = {{rhx[i][0], rhx[i][1]}, {rhy[i][0], rhy[i][1]}, {rez[i][0], rez[i][1]}};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        V2 o;
        o.x = r3[c][0];
        o.y = r3[c][1];
        *reinterpret_cast<V2*>(sacc + (c * NP + n) * TL + col) = o;
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < UW; ++i) {
    if (!unit_ok(i)) continue;
    const int n = 8 * rg_of(i) + (lane >> 2);
    if (n >= NP) continue;
    const int col = colx(n, ec0);
    const int64_t off = ((int64_t)tile * NP + n) * TL + col;
    const TT r3[3][2] = {{rhx[i][0], rhx[i][1]}, {rhy[i][0], rhy[i][1]}, {rez[i][0], rez[i][1]}};
    if constexpr (MT::rk) {
      TT* __restrict__ res = static_cast<TT*>(p.res);
      TT* __restrict__ qo = static_cast<TT*>(p.q_out);
      const TT a = static_cast<TT>(p.a), b = static_cast<TT>(p.b), dt = static_cast<TT>(p.dt);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        V2 rs;
        rs.x = dt * r3[c][0];
        rs.y = dt * r3[c][1];
        if (read_res) {
          const V2 ro = RES_TMA ? *reinterpret_cast<const V2*>(sr + (c * NP + n) * TL + col) : rr[i][c];
          rs.x = fma(a, ro.x, rs.x);
          rs.y = fma(a, ro.y, rs.y);
        }
        const V2 qi = *reinterpret_cast<const V2*>(sq + (c * NP + n) * TL + col);
        V2 qn;
        qn.x = fma(b, rs.x, qi.x);
        qn.y = fma(b, rs.y, qi.y);
        if constexpr (WSM && TMA_ST) {  // in place; stage_kernel_ws streams the tile out by TMA
          *reinterpret_cast<V2*>(const_cast<TT*>(sr) + (c * NP + n) * TL + col) = rs;
          *reinterpret_cast<V2*>(const_cast<TT*>(sq) + (c * NP + n) * TL + col) = qn;
        } else {
          if (p.write_res) st_out(reinterpret_cast<V2*>(res + c * p.vstride + off), rs);
          st_out(reinterpret_cast<V2*>(qo + c * p.fstride + off), qn);
        }
      }
    } else {
      TT* __restrict__ out = static_cast<TT*>(p.out);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        V2 o;
        o.x = r3[c][0];
        o.y = r3[c][1];
        *reinterpret_cast<V2*>(out + c * p.vstride + off) = o;
      }
    }
  }
  if constexpr (WSM && TMA_ST) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}


// DG_EI (warp-specialised DMMA kernel): the LSERK4 epilogue of tile t-1 is interleaved into the
// volume DMMAs of tile t (epi_step(ks) at every k-step), so its stores and their register hazards
// overlap the DMMA pipe instead of following the LIFT.  Per tile: volume (+ epilogue steps of the
// previous tile) -> geometry into registers -> after_volume() (barrier among the DMMA warps: the
// previous epilogue is done, the tile's residual may be loaded) -> flux_wait() -> release() (the
// tile's {q, geo} buffer is no longer read: TMA of tile t+2) -> LIFT -> flux_done() -> material
// scaling -> rhs (held for the next tile's epilogue steps).
template <bool MAT, typename TT, typename EPI, typename AV_, typename FW, typename REL, typename FD>
__device__ __forceinline__ void mma_tile_u_ei(const TT* __restrict__ sq, const TT* __restrict__ sg,
                                              const TT* __restrict__ sp, const unsigned char* __restrict__ ops,
                                              int g, int lane, TT (&rhs)[UW][3][2], const EPI& epi_step,
                                              const AV_& after_volume, const FW& flux_wait, const REL& release,
                                              const FD& flux_done) {
  using V2 = double2;
  const int nt = g & 3, rg0 = g >> 2;
  auto rg_of = [&](int i) { return rg0 + i * UST; };
  auto unit_ok = [&](int i) { return (UW - 1) * UST + (P / 4 - 1) < PR || rg_of(i) < PR; };
  const int eb = 8 * nt + (lane >> 2);
  const int ec0 = 8 * nt + 2 * (lane & 3);
  const TT rxb = sg[0 * TL + eb], sxb = sg[1 * TL + eb], ryb = sg[2 * TL + eb], syb = sg[3 * TL + eb];
  TT u[UW][2], v[UW][2], w[UW][2], w2a[UW][2];
#pragma unroll
  for (int i = 0; i < UW; ++i) u[i][0] = u[i][1] = v[i][0] = v[i][1] = w[i][0] = w[i][1] = w2a[i][0] = w2a[i][1] = TT(0);
  const V2* AV = reinterpret_cast<const V2*>(ops);
  // epilogue steps start EI_LAG k-steps in, so the previous tile's q_in (loaded from L2 at the top of the
  // tile) has arrived by the time its first step consumes it
  constexpr int EI_LAG = KV >= 3 * UW + 3 ? 3 : (KV > 3 * UW ? KV - 3 * UW : 0);
#pragma unroll
  for (int ks = 0; ks < KV; ++ks) {
    if (ks >= EI_LAG) epi_step(ks - EI_LAG);
    const int j = 4 * ks + (lane & 3);
    const int jc = j < NP ? j : NP - 1;
    const int addr = jc * TL + colx(jc, eb);
    const TT ez = sq[2 * NP * TL + addr], hx = sq[addr], hy = sq[NP * TL + addr];
    const TT w1 = rxb * hy - ryb * hx, w2 = sxb * hy - syb * hx;
#pragma unroll
    for (int i = 0; i < UW; ++i) {
      if (!unit_ok(i)) continue;
      const V2 a = ldop(AV + (ks * PR + rg_of(i)) * 32 + lane);
      dmma(u[i][0], u[i][1], a.x, ez);
      dmma(v[i][0], v[i][1], a.y, ez);
      dmma(w[i][0], w[i][1], a.x, w1);
      dmma(w2a[i][0], w2a[i][1], a.y, w2);
    }
  }
#pragma unroll
  for (int ks = KV - EI_LAG; ks < 3 * UW; ++ks) epi_step(ks);  // (k-steps fewer than epilogue steps)
  TT gx[2][4], mf[2][2];  // the tile's geometry (and material factors) of this lane's two elements
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int ec = ec0 + h;
    gx[h][0] = sg[0 * TL + ec];
    gx[h][1] = sg[1 * TL + ec];
    gx[h][2] = sg[2 * TL + ec];
    gx[h][3] = sg[3 * TL + ec];
    if constexpr (MAT) {
      mf[h][0] = sg[16 * TL + ec];
      mf[h][1] = sg[17 * TL + ec];
    }
  }
  after_volume();
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < UW; ++i) {
      const TT rx = gx[h][0], sx = gx[h][1], ry = gx[h][2], sy = gx[h][3];
      rhs[i][2][h] = w[i][h] + w2a[i][h];
      rhs[i][0][h] = -(ry * u[i][h] + sy * v[i][h]);
      rhs[i][1][h] = rx * u[i][h] + sx * v[i][h];
    }
  flux_wait();
  release();
  const TT* AL = reinterpret_cast<const TT*>(ops + DVB);
#pragma unroll
  for (int ks = 0; ks < KL; ++ks) {
    const int m = 4 * ks + (lane & 3);
    const int mc = m < NF ? m : NF - 1;
    const int addr = mc * TL + colx(mc, eb);
    const TT f0 = sp[0 * NFE * TL + addr], f1 = sp[1 * NFE * TL + addr], f2 = sp[2 * NFE * TL + addr];
#pragma unroll
    for (int i = 0; i < UW; ++i) {
      if (!unit_ok(i)) continue;
      const TT a = ldop(AL + (ks * PR + rg_of(i)) * 32 + lane);
      dmma(rhs[i][0][0], rhs[i][0][1], a, f0);
      dmma(rhs[i][1][0], rhs[i][1][1], a, f1);
      dmma(rhs[i][2][0], rhs[i][2][1], a, f2);
    }
  }
  flux_done();
  if constexpr (MAT) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < UW; ++i) {
        rhs[i][0][h] *= mf[h][0];
        rhs[i][1][h] *= mf[h][0];
        rhs[i][2][h] *= mf[h][1];
      }
  }
}

// Persistent, software-pipelined stage kernel (one team per CTA).
template <int MODE, bool MAT>
__global__ void __launch_bounds__(TEAM, MIN_CTAS) stage_kernel(const dg::StageArgs p) {
  using MT = ModeTraits<MODE>;
  constexpr int NG = ngeo(MAT);
  constexpr int S = nslots(MT::surf, MAT);
  constexpr size_t SLOT = slot_bytes(MT::surf, MAT, MT::rk);
  constexpr size_t GB = geo_bytes(MAT);
  constexpr int CH = 16 / (int)sizeof(T);
  constexpr int QC = NP * TL / CH;  // 16 B chunks per field tile
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const T* __restrict__ q = static_cast<const T*>(p.q_in);
  const T* __restrict__ geo = static_cast<const T*>(p.geo);
  const int tid = threadIdx.x;
  const int first = blockIdx.x, stride = gridDim.x;
  const int n_it = first < p.ntiles ? (p.ntiles - first + stride - 1) / stride : 0;
  if (n_it == 0) return;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);  // [0, S): slots, [S]: residual
  const unsigned char* opbase = OPS_GLOBAL ? static_cast<const unsigned char*>(p.ops) : smem_raw + BARB;
  const DV_t* DV = reinterpret_cast<const DV_t*>(opbase);
  const LV_t* LV = reinterpret_cast<const LV_t*>(opbase + DVB);
  unsigned char* slots = smem_raw + BARB + OPB_SMEM;
  T* const sw = reinterpret_cast<T*>(smem_raw + smem_total(S, MT::surf, MAT, MT::rk) - WPB);  // DG_WP buffer
  const unsigned char* opsrc = OPS_GLOBAL ? static_cast<const unsigned char*>(p.ops) : smem_raw + BARB;
  constexpr bool S3 = S == 3;      // split pipeline: slots A0, A1 = {q, geo}; one B = {flux, residual}
  constexpr size_t AB = QB + GB;
  auto sq_of = [&](int s) { return reinterpret_cast<T*>(slots + (S3 ? s * AB : s * SLOT)); };
  auto sg_of = [&](int s) { return reinterpret_cast<T*>(slots + (S3 ? s * AB : s * SLOT) + QB); };
  auto sp_of = [&](int s) { return reinterpret_cast<T*>(slots + (S3 ? 2 * AB : s * SLOT + QB + GB)); };
  auto sr_of = [&](int s) {
    return reinterpret_cast<T*>(slots + (S3 ? 2 * AB : s * SLOT + QB + GB) + (MT::surf ? SPB : 0));
  };
  auto slot_of_it = [&](int it) { return S3 ? (it & 1) : it % S; };
  const bool read_res = MT::rk && p.a != 0.0;
  const int g = tid >> 5, lane = tid & 31;

  auto tile_of = [&](int it) {
    const int sidx = first + it * stride;
    const int j = p.reverse ? p.ntiles - 1 - sidx : sidx;
    return p.tiles ? p.tiles[j] : j;
  };
  // vmapP codes of this thread's face points (m = g + k P) of tile `it`
  auto load_codes = [&](int it, int32_t (&v)[KCODE]) {
    if constexpr (MT::surf && ZC_CONN && !MAT) {  // one word per face, decoded per point
      const uint32_t* src = reinterpret_cast<const uint32_t*>(p.vmapP) + (int64_t)tile_of(it) * 3 * TL;
#pragma unroll
      for (int k = 0; k < KCODE; ++k) {
        const PointElem pe = pair_of(g, lane, k);
        if (pe.m < NF) {
          const int f = pe.m / NFP;
          v[k] = zc_decode(__ldg(src + f * TL + pe.e), f, pe.m - f * NFP, pe.e, p.vstride);
        } else {
          v[k] = -1;
        }
      }
    } else if constexpr (MT::surf) {
      const int32_t* src = p.vmapP + (int64_t)tile_of(it) * NF * TL;
#pragma unroll
      for (int k = 0; k < KCODE; ++k) {
        const PointElem pe = pair_of(g, lane, k);
        v[k] = pe.m < NF ? __ldg(src + pe.m * TL + pe.e) : -1;
      }
    }
  };
  // fields + geometry of tile `it`: four TMA bulk copies issued by one thread (with S != 3 the
  // residual too, on the same barrier)
  auto issue_tma = [&](int it) {
    if (tid == 0) {
      const int tile = tile_of(it);
      const int s = slot_of_it(it);
      uint64_t* bar = bars + s;
      constexpr bool rt = RES_TMA && MT::rk && !S3;
      constexpr bool rsep = rt && RES_SEP;  // residual on its own barrier (DG_RB)
      mbar_expect_tx(bar, (unsigned)(QB + GB + (rt && !rsep && read_res ? QB : 0)));
      T* sq = sq_of(s);
#pragma unroll
      for (int c = 0; c < 3; ++c)
        tma_load_1d(sq + c * NP * TL, q + c * p.fstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3), bar);
      tma_load_1d(sg_of(s), geo + (int64_t)tile * NG * TL, (unsigned)GB, bar);
      if (rt && read_res) {
        const T* res = static_cast<const T*>(p.res);
        uint64_t* rbar = rsep ? bars + 2 : bar;
        if (rsep) mbar_expect_tx(rbar, (unsigned)QB);
#pragma unroll
        for (int c = 0; c < 3; ++c)
          tma_load_1d(sr_of(s) + c * NP * TL, res + c * p.vstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3), rbar);
      }
    }
  };
  // S = 3: the residual of tile `it` into the B buffer, on barrier 2
  auto issue_res = [&](int it) {
    if (RES_TMA && MT::rk && S3 && tid == 0 && read_res) {
      const int tile = tile_of(it);
      const T* res = static_cast<const T*>(p.res);
      mbar_expect_tx(bars + 2, (unsigned)QB);
#pragma unroll
      for (int c = 0; c < 3; ++c)
        tma_load_1d(sr_of(0) + c * NP * TL, res + c * p.vstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3), bars + 2);
    }
  };
  // one slot: pull the next tile's TMA sources into L2 while this tile computes, so the TMA
  // issued after the epilogue reads L2 rather than DRAM (cp.async.bulk.prefetch.L2)
  auto prefetch_l2 = [&](int it) {
    if (tid == 0) {
      const int tile = tile_of(it);
#pragma unroll
      for (int c = 0; c < 3; ++c) bulk_prefetch_l2(q + c * p.fstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3));
      bulk_prefetch_l2(geo + (int64_t)tile * NG * TL, (unsigned)GB);
      if (RES_TMA && MT::rk && read_res) {
        const T* res = static_cast<const T*>(p.res);
#pragma unroll
        for (int c = 0; c < 3; ++c) bulk_prefetch_l2(res + c * p.vstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3));
      }
    }
  };
  // cross-tile neighbour traces of tile `it` (same-tile ones are read from shared memory)
  auto issue_gather = [&](int it, const int32_t (&v)[KCODE]) {
    if constexpr (MT::surf) {
      T* sp = sp_of(slot_of_it(it));
#pragma unroll
      for (int k = 0; k < KCODE; ++k) {
        const PointElem pe = pair_of(g, lane, k);
        if (pe.m < NF && v[k] >= 0) {
          const T* src = q + v[k];
          T* dst = sp + pe.m * TL + colx(pe.m, pe.e);
#pragma unroll
          for (int c = 0; c < 3; ++c) cp_async_small<sizeof(T)>(dst + c * NFE * TL, src + c * p.fstride);
        }
      }
    }
  };

  // prologue: barriers, operators (once per persistent CTA), zero flux pad columns, first tiles
  if (tid == 0) {
    for (int b = 0; b < S; ++b) mbar_init(bars + b, 1);  // S = 3: A0, A1, residual
    if (RES_SEP && S == 1) mbar_init(bars + 2, 1);         // DG_RB: the residual's own barrier
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const int4* src = reinterpret_cast<const int4*>(p.ops);
    int4* dst = reinterpret_cast<int4*>(smem_raw + BARB);
    for (int i = tid; i < (int)(OPB_SMEM / 16); i += TEAM) cp_async16(dst + i, src + i);
    if constexpr (MT::surf && NFE > NF) {
      constexpr int PADN = (NFE - NF) * TL;
      for (int i = tid; i < (S3 ? 1 : S) * 3 * PADN; i += TEAM) {
        const int s = i / (3 * PADN), rem = i - s * 3 * PADN;
        const int c = rem / PADN, rem2 = rem - c * PADN;
        sp_of(s)[(c * NFE + NF) * TL + rem2] = T(0);
      }
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  int32_t vc0[KCODE], vc1[KCODE], vc2[KCODE];  // codes of tiles it, it+1, it+2
  load_codes(0, vc0);
  if (n_it > 1) load_codes(1, vc1);
  issue_tma(0);
#pragma unroll 1
  for (int d = (S == 1 ? 1 : 2); d < (S == 1 ? 0 : 1) + DG_PD && d < n_it; ++d) prefetch_l2(d);  // DG_PD > 1
  if constexpr (!GATHER_LATE) issue_gather(0, vc0);
  cp_async_commit();

  const int n0 = g * R;
  const T alpha = static_cast<T>(p.alpha);
  for (int it = 0; it < n_it; ++it) {
    const int s = slot_of_it(it);
    if constexpr (!GATHER_WAIT_LATE) cp_async_wait_all();                  // gathers of tile it
    mbar_wait(bars + s, (unsigned)(S3 ? (it >> 1) & 1 : (it / S) & 1));  // TMA: fields + geometry of tile it
    __syncthreads();
    const int tile = tile_of(it);
    if (S == 2 && it + 1 < n_it) {
      issue_tma(it + 1);
      issue_gather(it + 1, vc1);
      cp_async_commit();
    }
    if (S3) {
      if (it + 1 < n_it) issue_tma(it + 1);  // into the other {q, geo} buffer (its tile it-1 is done)
      issue_res(it);                         // B's residual: read by this tile's epilogue only
      if constexpr (GATHER_LATE) {           // this tile's gathers: needed at its flux, after the volume
        issue_gather(it, vc0);
        cp_async_commit();
      }
    }
    // L2 prefetch distance: S = 1 issues tile it+1's TMA after this tile, S = 2/3 at the next tile
    constexpr int PFD = (S == 1 ? 0 : 1) + DG_PD;
    if (it + PFD < n_it) prefetch_l2(it + PFD);
    if (it + 2 < n_it) load_codes(it + 2, vc2);
    // after the LIFT (S = 3): every warp is done with the flux buffer -> the next tile's
    // neighbour gathers go into it; the epilogue then needs this tile's residual
    auto after_lift = [&]() {
      if constexpr (RES_SEP && S == 1) {
        if (RES_TMA && MT::rk && read_res) mbar_wait(bars + 2, (unsigned)(it & 1));
      }
      if constexpr (S3) {
        if constexpr (!GATHER_LATE) {
          __syncthreads();
          if (it + 1 < n_it) issue_gather(it + 1, vc1);
          cp_async_commit();
        }
        if (RES_TMA && MT::rk && read_res) mbar_wait(bars + 2, (unsigned)(it & 1));
      }
    };

    const T* sq = sq_of(s);
    const T* gg = sg_of(s) + lane;
    T* sp = sp_of(s);
    if constexpr (DMMA_U) {
      mma_tile_u<MODE, MAT>(p, sq, sg_of(s), sp, sr_of(s), opsrc, vc0, tile, g, lane, alpha, read_res, after_lift);
    } else if constexpr (USE_MMA) {
      if constexpr (DMMA_SPLIT) {
        if (g < PR)
          mma_tile<MODE, MAT, 1>(p, sq, sg_of(s), sp, opsrc, vc0, tile, g, g, lane, alpha, read_res, after_lift);
        else
          mma_tile<MODE, MAT, 2>(p, sq, sg_of(s), sp, opsrc, vc0, tile, g, g - PR, lane, alpha, read_res, after_lift);
      } else {
        mma_tile<MODE, MAT, 0>(p, sq, sg_of(s), sp, opsrc, vc0, tile, g, g, lane, alpha, read_res, after_lift);
      }
    } else if constexpr (USE_TF) {
      if constexpr (TF_SPLIT) {
        if (g < 2)
          tf_tile<MODE, MAT, 1>(p, sq, sg_of(s), sp, sr_of(s), opsrc, vc0, tile, g, g & 1, lane, alpha, read_res, after_lift);
        else
          tf_tile<MODE, MAT, 2>(p, sq, sg_of(s), sp, sr_of(s), opsrc, vc0, tile, g, g & 1, lane, alpha, read_res, after_lift);
      } else {
        tf_tile<MODE, MAT, 0>(p, sq, sg_of(s), sp, sr_of(s), opsrc, vc0, tile, g, g, lane, alpha, read_res, after_lift);
      }
    } else {
    if constexpr (WPRE && MT::vol) {  // W1, W2 of the tile, once (DG_WP)
      const T* sgs = sg_of(s);
      for (int i = tid; i < NP * TL; i += TEAM) {
        const int e = i & (TL - 1);
        const T hx = sq[i], hy = sq[NP * TL + i];
        sw[i] = sgs[0 * TL + e] * hy - sgs[2 * TL + e] * hx;
        sw[NP * TL + i] = sgs[1 * TL + e] * hy - sgs[3 * TL + e] * hx;
      }
      if constexpr (!(FLUX_FIRST && MT::surf)) __syncthreads();
    }
    if constexpr (FLUX_FIRST && MT::surf) {
      flux_points<MAT>(sq, gg, sp, vc0, g, lane, alpha);
      __syncthreads();
    }
    T rhx[R], rhy[R], rez[R];
    if constexpr (MT::vol) {
      volume_rows(sq, DV, n0, lane, gg[0 * TL], gg[1 * TL], gg[2 * TL], gg[3 * TL], rhx, rhy, rez, sw);
    } else if constexpr (MODE == dg::MODE_SURFACE_RK) {
      const T* __restrict__ rv = static_cast<const T*>(p.rhsv);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int n = n0 + r < NP ? n0 + r : NP - 1;
        const int64_t off = ((int64_t)tile * NP + n) * TL + lane;
        rhx[r] = rv[off];
        rhy[r] = rv[p.vstride + off];
        rez[r] = rv[2 * p.vstride + off];
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) { rhx[r] = T(0); rhy[r] = T(0); rez[r] = T(0); }
    }
    // LSERK4 residual of this tile -> registers (in flight during the surface phase)
    T rr[3][R];
    if constexpr (MT::rk) {
      if (read_res) {
        const T* __restrict__ res = static_cast<const T*>(p.res);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int n = n0 + r < NP ? n0 + r : NP - 1;
#pragma unroll
          for (int c = 0; c < 3; ++c) rr[c][r] = __ldcs(res + c * p.vstride + ((int64_t)tile * NP + n) * TL + lane);
        }
      }
    }
    if constexpr (MT::surf) {
      if constexpr (!FLUX_FIRST) {
        flux_points<MAT>(sq, gg, sp, vc0, g, lane, alpha);
        __syncthreads();
      }
      lift_rows(sp, LV, n0, lane, rhx, rhy, rez);
    }
    after_lift();
    // material factors 1/mu, 1/eps (reading A12).  In split mode the volume kernel
    // writes the UNSCALED rhsV and the surface kernel scales the sum.
    if constexpr (MAT) {
      if (MODE != dg::MODE_VOLUME || p.scale_volume) {
        const T imu = gg[16 * TL], ieps = gg[17 * TL];
#pragma unroll
        for (int r = 0; r < R; ++r) { rhx[r] *= imu; rhy[r] *= imu; rez[r] *= ieps; }
      }
    }
    if constexpr (MT::rk) {
      T* __restrict__ res = static_cast<T*>(p.res);
      T* __restrict__ qo = static_cast<T*>(p.q_out);
      const T a = static_cast<T>(p.a), b = static_cast<T>(p.b), dt = static_cast<T>(p.dt);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int n = n0 + r;
        if (RP != NP && n >= NP) break;
        const int64_t off = ((int64_t)tile * NP + n) * TL + lane;
        const T rhs[3] = {rhx[r], rhy[r], rez[r]};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          T rs = dt * rhs[c];
          if (read_res) rs = fma(a, rr[c][r], rs);
          if (p.write_res) st_out(res + c * p.vstride + off, rs);
          st_out(qo + c * p.fstride + off, fma(b, rs, sq[(c * NP + n) * TL + lane]));
        }
      }
    } else {
      T* __restrict__ out = static_cast<T*>(p.out);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int n = n0 + r;
        if (RP != NP && n >= NP) break;
        const int64_t off = ((int64_t)tile * NP + n) * TL + lane;
        out[off] = rhx[r];
        out[p.vstride + off] = rhy[r];
        out[2 * p.vstride + off] = rez[r];
      }
    }
    }  // !USE_MMA
    if constexpr (SMEM_ST && MT::rk) {  // the tile's new residual and fields, coalesced (DG_TS = 2)
      __syncthreads();
      using V4 = typename std::conditional<F32, float4, double2>::type;
      constexpr int PER = 16 / (int)sizeof(T);
      const int64_t t0 = (int64_t)tile * NP * TL;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int o = PER * tid; o < NP * TL; o += PER * TEAM) {
          if (p.write_res)
            __stcs(reinterpret_cast<V4*>(static_cast<T*>(p.res) + c * p.vstride + t0 + o),
                   *reinterpret_cast<const V4*>(sr_of(s) + c * NP * TL + o));
          __stcs(reinterpret_cast<V4*>(static_cast<T*>(p.q_out) + c * p.fstride + t0 + o),
                 *reinterpret_cast<const V4*>(sq_of(s) + c * NP * TL + o));
        }
    } else if constexpr (TMA_ST && MT::rk) {  // the tile's new residual and fields, from shared memory (DG_TS)
      __syncthreads();
      if (tid == 0) {
        const int64_t t0 = (int64_t)tile * NP * TL;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (p.write_res) tma_store_1d(static_cast<T*>(p.res) + c * p.vstride + t0, sr_of(s) + c * NP * TL, (unsigned)(QB / 3));
          tma_store_1d(static_cast<T*>(p.q_out) + c * p.fstride + t0, sq_of(s) + c * NP * TL, (unsigned)(QB / 3));
        }
        bulk_commit();
      }
    }
    if (S == 1 && it + 1 < n_it) {
      if constexpr (!(TMA_ST && MT::rk)) __syncthreads();
      if (SMEM_ST && MT::rk) __syncthreads();                 // every thread's stores have read the slot
      if (TMA_ST && !SMEM_ST && MT::rk && tid == 0) bulk_wait_read();  // the slot's bulk stores have read it
      issue_tma(it + 1);
      issue_gather(it + 1, vc1);
      cp_async_commit();
    }
#pragma unroll
    for (int k = 0; k < KCODE; ++k) { vc0[k] = vc1[k]; vc1[k] = vc2[k]; }
  }
  if (TMA_ST && !SMEM_ST && MT::rk && tid == 0) bulk_wait_all();  // smem stays valid until the stores are done
}


// ---------------------------------------------------------------- warp-specialised fused stage (DG_WS)
// Shared memory: mbarriers | operators | A0, A1 = {q, geo} (tile t in A[t & 1], TMA) | F0, F1 flux
// buffers | the residual buffer (RES_TMA).  mbarriers: 0, 1 A loaded (tx); 2 residual loaded (tx);
// 3, 4 flux of F[b] formed (WF x 32 arrivals); 5, 6 F[b] read by the LIFT (TEAM_M arrivals).
// DMMA warps (0 .. PU-1), tile t, b = t & 1:  wait A[b] -> (thread 0: residual TMA) -> volume ->
//   wait flux[b] -> LIFT -> release F[b] -> wait residual -> epilogue -> named barrier -> (thread 0: TMA of
//   tile t+2 into A[b]; its L2 prefetch of tile t+3)
// flux warps (PU .. PU+3), tile t:  wait A[b] -> wait F[b] released by the LIFT of tile t-2 -> cp.async
//   gathers of the cross-tile neighbour traces into F[b] -> wait own copies -> flux -> arrive flux[b].
// A[b] is free once the DMMA warps' epilogue of tile t is done: their LIFT waited for the flux warps'
// flux of tile t, the flux warps' last use of A[b].
constexpr size_t BARW = 128;  // the warp-specialised kernel's 9 mbarriers
constexpr int TEAM_M = P * 32;
constexpr int TEAM_WS = TEAM_M + WF * 32;
constexpr int KF = (NF + WF - 1) / WF;  // face points per flux thread: m = gf + k WF, element = lane
static_assert(!(WS && ZC_CONN), "DG_WS reads per-point neighbour codes (not with DG_ZC = 1)");
__host__ __device__ constexpr size_t ws_smem(bool mat) {
  return BARW + OPB_SMEM + 2 * (QB + geo_bytes(mat)) + 2 * SPB + (RES_TMA || WS2 ? QB : 0);
}
static_assert(!(WS2 && RES_TMA), "DG_WS = 2 reads the residual in the helper warps (DG_RT = 0)");
#ifndef DG_WSC
#define DG_WSC 1  // resident warp-specialised CTAs per SM the register budget is sized for
#endif
template <int MODE, bool MAT>
__global__ void __launch_bounds__(TEAM_WS, DG_WSC) stage_kernel_ws(const dg::StageArgs p) {
  static_assert(MODE == dg::MODE_FUSED_RK, "the warp-specialised kernel runs the fused stage");
  constexpr int NG = ngeo(MAT);
  constexpr size_t GB = geo_bytes(MAT);
  constexpr size_t AB = QB + GB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const T* __restrict__ q = static_cast<const T*>(p.q_in);
  const T* __restrict__ geo = static_cast<const T*>(p.geo);
  const int tid = threadIdx.x, g = tid >> 5, lane = tid & 31;
  const int first = blockIdx.x, stride = gridDim.x;
  const int n_it = first < p.ntiles ? (p.ntiles - first + stride - 1) / stride : 0;
  if (n_it == 0) return;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  unsigned char* abuf = smem_raw + BARW + OPB_SMEM;
  auto sq_of = [&](int b) { return reinterpret_cast<T*>(abuf + b * AB); };
  auto sg_of = [&](int b) { return reinterpret_cast<T*>(abuf + b * AB + QB); };
  auto sp_of = [&](int b) { return reinterpret_cast<T*>(abuf + 2 * AB + b * SPB); };
  T* const sr = reinterpret_cast<T*>(abuf + 2 * AB + 2 * SPB);
  const bool read_res = p.a != 0.0;
  auto tile_of = [&](int it) {
    const int sidx = first + it * stride;
    const int j = p.reverse ? p.ntiles - 1 - sidx : sidx;
    return p.tiles ? p.tiles[j] : j;
  };
  auto issue_tma = [&](int it) {  // fields + geometry of tile it into A[it & 1]
    const int tile = tile_of(it), b = it & 1;
    mbar_expect_tx(bars + b, (unsigned)AB);
#pragma unroll
    for (int c = 0; c < 3; ++c)
      tma_load_1d(sq_of(b) + c * NP * TL, q + c * p.fstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3), bars + b);
    tma_load_1d(sg_of(b), geo + (int64_t)tile * NG * TL, (unsigned)GB, bars + b);
  };
  auto prefetch_l2 = [&](int it) {
    const int tile = tile_of(it);
#pragma unroll
    for (int c = 0; c < 3; ++c) bulk_prefetch_l2(q + c * p.fstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3));
    bulk_prefetch_l2(geo + (int64_t)tile * NG * TL, (unsigned)GB);
    if ((RES_TMA || WS2) && read_res) {
      const T* res = static_cast<const T*>(p.res);
#pragma unroll
      for (int c = 0; c < 3; ++c) bulk_prefetch_l2(res + c * p.vstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3));
    }
  };
  T* const sacc = sr;  // WS2: the rhs hand-over buffer (in place of the residual buffer)
  // prologue: barriers, operators, the first two tiles
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) mbar_init(bars + b, 1);
    mbar_init(bars + 2, 1);
    mbar_init(bars + 7, TEAM_M);  // WS2: rhs of the tile in sacc (DMMA warps arrive)
    mbar_init(bars + 8, WF * 32);  // WS2: sacc consumed by the epilogue (helper warps arrive)
    for (int b = 0; b < 2; ++b) mbar_init(bars + 3 + b, WF * 32);
    for (int b = 0; b < 2; ++b) mbar_init(bars + 5 + b, TEAM_M);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const int4* src = reinterpret_cast<const int4*>(p.ops);
    int4* dst = reinterpret_cast<int4*>(smem_raw + BARW);
    for (int i = tid; i < (int)(OPB_SMEM / 16); i += TEAM_WS) cp_async16(dst + i, src + i);
    if constexpr (NFE > NF) {  // zero flux pad columns (3xTF32 k-steps of 8) of both flux buffers
      constexpr int PADN = (NFE - NF) * TL;
      for (int i = tid; i < 2 * 3 * PADN; i += TEAM_WS) {
        const int b = i / (3 * PADN), rem = i - b * 3 * PADN;
        const int c = rem / PADN, rem2 = rem - c * PADN;
        sp_of(b)[(c * NFE + NF) * TL + rem2] = T(0);
      }
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  if (tid == 0) {
    issue_tma(0);
    if (n_it > 1) issue_tma(1);
    if (n_it > 2) prefetch_l2(2);
  }
  const T alpha = static_cast<T>(p.alpha);
  if (EI && g < P) {  // ---------------------------------- DMMA warps, interleaved epilogue (DG_EI)
    static_assert(!EI || (RES_TMA && !TMA_ST && !WS2), "DG_EI: residual by TMA, streaming stores");
    using V2 = double2;
    const int nt = g & 3, rg0 = g >> 2;
    const int ec0 = 8 * nt + 2 * (lane & 3);
    const T a = static_cast<T>(p.a), bq = static_cast<T>(p.b), dt = static_cast<T>(p.dt);
    T pend[UW][3][2];  // rhs of the previous tile, applied by the epilogue steps
    int ptile = -1;    // the previous tile (-1: none)
    auto unit_n = [&](int i) { return 8 * (rg0 + i * UST) + (lane >> 2); };
    V2 qpre[UW][3];    // q_in of the previous tile (global / L2), loaded before the first epilogue step
    auto epi_step = [&](int k) {
      if (ptile < 0 || k >= 3 * UW) return;
      const int i = k / 3, c = k % 3;
      const int n = unit_n(i);
      if (n >= NP) return;
      const int col = colx(n, ec0);
      const int64_t off = ((int64_t)ptile * NP + n) * TL + col;
      V2 rs;
      rs.x = dt * pend[i][c][0];
      rs.y = dt * pend[i][c][1];
      if (read_res) {
        const V2 ro = *reinterpret_cast<const V2*>(sr + (c * NP + n) * TL + col);
        rs.x = fma(a, ro.x, rs.x);
        rs.y = fma(a, ro.y, rs.y);
      }
      V2 qn;
      qn.x = fma(bq, rs.x, qpre[i][c].x);
      qn.y = fma(bq, rs.y, qpre[i][c].y);
      if (p.write_res) st_out(reinterpret_cast<V2*>(static_cast<T*>(p.res) + c * p.vstride + off), rs);
      st_out(reinterpret_cast<V2*>(static_cast<T*>(p.q_out) + c * p.fstride + off), qn);
    };
    auto load_qpre = [&]() {
      if (ptile < 0) return;
#pragma unroll
      for (int i = 0; i < UW; ++i) {
        const int n = unit_n(i);
        const int nc = n < NP ? n : NP - 1;
        const int64_t off = ((int64_t)ptile * NP + nc) * TL + colx(nc, ec0);
#pragma unroll
        for (int c = 0; c < 3; ++c) qpre[i][c] = __ldg(reinterpret_cast<const V2*>(q + c * p.fstride + off));
      }
    };
    for (int it = 0; it < n_it; ++it) {
      const int b = it & 1;
      const int tile = tile_of(it);
      load_qpre();
      if (ptile >= 0 && read_res) mbar_wait(bars + 2, (unsigned)((it - 1) & 1));  // residual of tile it-1
      mbar_wait(bars + b, (unsigned)((it >> 1) & 1));
      auto after_volume = [&]() {
        named_barrier(1, TEAM_M);  // every DMMA warp is done with the previous epilogue (sr) and the volume
        if (read_res && tid == 0) {
          mbar_expect_tx(bars + 2, (unsigned)QB);
          const T* res = static_cast<const T*>(p.res);
#pragma unroll
          for (int c = 0; c < 3; ++c)
            tma_load_1d(sr + c * NP * TL, res + c * p.vstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3), bars + 2);
        }
      };
      auto flux_wait = [&]() { mbar_wait(bars + 3 + b, (unsigned)((it >> 1) & 1)); };
      auto release = [&]() {  // the flux warps are done with A[b] (flux of tile it), the DMMA warps too
        if (tid == 0) {
          if (it + 2 < n_it) issue_tma(it + 2);
          if (it + 3 < n_it) prefetch_l2(it + 3);
        }
      };
      auto flux_done = [&]() { mbar_arrive(bars + 5 + b); };
      mma_tile_u_ei<MAT>(sq_of(b), sg_of(b), sp_of(b), smem_raw + BARW, g, lane, pend, epi_step, after_volume,
                         flux_wait, release, flux_done);
      ptile = tile;
    }
    // the last tile's epilogue
    load_qpre();
    if (read_res) mbar_wait(bars + 2, (unsigned)((n_it - 1) & 1));
#pragma unroll
    for (int k = 0; k < 3 * UW; ++k) epi_step(k);
  } else if (g < P) {  // ------------------------------------------------------------- DMMA warps
    const int32_t nocodes[KCODE] = {};
    for (int it = 0; it < n_it; ++it) {
      const int b = it & 1;
      const int tile = tile_of(it);
      if (TMA_ST && tid == 0 && it >= 1) {  // tile it-1's bulk stores have read A[b ^ 1] and sr
        bulk_wait_read();
        if (it + 1 < n_it) issue_tma(it + 1);
      }
      mbar_wait(bars + b, (unsigned)((it >> 1) & 1));
      if (RES_TMA && read_res && tid == 0) {  // sr is free: the previous epilogue ended at the named barrier
        mbar_expect_tx(bars + 2, (unsigned)QB);
        const T* res = static_cast<const T*>(p.res);
#pragma unroll
        for (int c = 0; c < 3; ++c)
          tma_load_1d(sr + c * NP * TL, res + c * p.vstride + (int64_t)tile * NP * TL, (unsigned)(QB / 3), bars + 2);
      }
      auto flux_wait = [&]() { mbar_wait(bars + 3 + b, (unsigned)((it >> 1) & 1)); };
      auto flux_done = [&]() { mbar_arrive(bars + 5 + b); };
      auto after_lift = [&]() {
        if (RES_TMA && read_res) mbar_wait(bars + 2, (unsigned)(it & 1));
        if constexpr (TMA_ST) named_barrier(1, TEAM_M);  // no DMMA warp still reads A[b] in its volume
      };
      if constexpr (WS2) {
        // after the LIFT: every DMMA warp is done with A[b] -> TMA of tile it+2; then wait for sacc
        auto release = [&]() {
          named_barrier(1, TEAM_M);
          if (tid == 0) {
            if (it + 2 < n_it) issue_tma(it + 2);
            if (it + 3 < n_it) prefetch_l2(it + 3);
          }
          if (it >= 1) mbar_wait(bars + 8, (unsigned)((it - 1) & 1));  // epilogue of tile it-1 read sacc
        };
        mma_tile_u<MODE, MAT, true, true>(p, sq_of(b), sg_of(b), sp_of(b), sr, smem_raw + BARW, nocodes, tile, g,
                                          lane, alpha, read_res, release, flux_wait, flux_done, sacc);
        mbar_arrive(bars + 7);  // release: the rhs of tile it is in sacc
        continue;
      }
      if constexpr (USE_TF)
        tf_tile<MODE, MAT, 0, true>(p, sq_of(b), sg_of(b), sp_of(b), sr, smem_raw + BARW, nocodes, tile, g, g, lane,
                                    alpha, read_res, after_lift, flux_wait, flux_done);
      else
        mma_tile_u<MODE, MAT, true>(p, sq_of(b), sg_of(b), sp_of(b), sr, smem_raw + BARW, nocodes, tile, g, lane,
                                    alpha, read_res, after_lift, flux_wait, flux_done);
      named_barrier(1, TEAM_M);  // every contraction warp is done with A[b] and sr
      if (tid == 0) {
        if constexpr (TMA_ST) {  // the new q and residual of the tile, written in place (DG_TS)
          const int64_t t0 = (int64_t)tile * NP * TL;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (p.write_res) tma_store_1d(static_cast<T*>(p.res) + c * p.vstride + t0, sr + c * NP * TL, (unsigned)(QB / 3));
            tma_store_1d(static_cast<T*>(p.q_out) + c * p.fstride + t0, sq_of(b) + c * NP * TL, (unsigned)(QB / 3));
          }
          bulk_commit();
        } else {
          if (it + 2 < n_it) issue_tma(it + 2);
        }
        if (it + 3 < n_it) prefetch_l2(it + 3);
      }
    }
    if (TMA_ST && tid == 0) bulk_wait_all();
  } else {  // ------------------------------------------------------------------ flux warps
    const int gf = g - P;
    // WS2: LSERK4 update of tile j from sacc (rhs), q_in and the residual (global), elementwise over
    // the tile's physical offsets (every array shares the tile layout): coalesced 16-byte accesses
    auto epilogue = [&](int j) {
      mbar_wait(bars + 7, (unsigned)(j & 1));
      const int64_t t0 = (int64_t)tile_of(j) * NP * TL;
      const T a = static_cast<T>(p.a), bb = static_cast<T>(p.b), dt = static_cast<T>(p.dt);
      const T* __restrict__ res = static_cast<const T*>(p.res) + t0;
      T* __restrict__ reso = static_cast<T*>(p.res) + t0;
      T* __restrict__ qo = static_cast<T*>(p.q_out) + t0;
      const T* __restrict__ qi = q + t0;
      using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
#pragma unroll 2
      for (int o = 2 * (tid - TEAM_M); o < NP * TL; o += 2 * WF * 32) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const V2 r = *reinterpret_cast<const V2*>(sacc + c * NP * TL + o);
          V2 rs;
          rs.x = dt * r.x;
          rs.y = dt * r.y;
          if (read_res) {
            const V2 ro = __ldcs(reinterpret_cast<const V2*>(res + c * p.vstride + o));
            rs.x = fma(a, ro.x, rs.x);
            rs.y = fma(a, ro.y, rs.y);
          }
          const V2 qv = __ldg(reinterpret_cast<const V2*>(qi + c * p.fstride + o));
          V2 qn;
          qn.x = fma(bb, rs.x, qv.x);
          qn.y = fma(bb, rs.y, qv.y);
          if (p.write_res) st_out(reinterpret_cast<V2*>(reso + c * p.vstride + o), rs);
          st_out(reinterpret_cast<V2*>(qo + c * p.fstride + o), qn);
        }
      }
      mbar_arrive(bars + 8);
    };
    int32_t cc[KF], cn[KF];  // neighbour codes of tiles it, it+1
    auto load_codes = [&](int it, int32_t (&v)[KF]) {
      const int32_t* src = p.vmapP + (int64_t)tile_of(it) * NF * TL;
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int m = gf + k * WF;
        v[k] = m < NF ? __ldg(src + m * TL + lane) : -1;
      }
    };
    load_codes(0, cc);
    for (int it = 0; it < n_it; ++it) {
      const int b = it & 1;
      if (it + 1 < n_it) load_codes(it + 1, cn);
      if (it >= 2) mbar_wait(bars + 5 + b, (unsigned)(((it >> 1) + 1) & 1));  // F[b]: LIFT of tile it-2 done
      T* sp = sp_of(b);
#pragma unroll
      for (int k = 0; k < KF; ++k) {  // cross-tile neighbour traces (same-tile ones: from A[b])
        const int m = gf + k * WF;
        if (m < NF && cc[k] >= 0) {
          const T* src = q + cc[k];
          T* dst = sp + m * TL + colx(m, lane);
#pragma unroll
          for (int c = 0; c < 3; ++c) cp_async_small<sizeof(T)>(dst + c * NFE * TL, src + c * p.fstride);
        }
      }
      cp_async_commit();
      mbar_wait(bars + b, (unsigned)((it >> 1) & 1));  // A[b]: own traces, same-tile neighbours, geometry
      cp_async_wait_all();
      const T* sq = sq_of(b);
      const T* gg = sg_of(b) + lane;
      T fz[3][3];
      if constexpr (ZC && !MAT) zc_faces(gg, fz);
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int m = gf + k * WF;
        if (m >= NF) break;
        const int f = m / NFP;
        T fHx, fHy, fEz;
        flux_one<MAT>(sq, gg, sp, cc[k], m, f, lane, alpha, fHx, fHy, fEz, fz);
        const int pm = m * TL + colx(m, lane);
        sp[0 * NFE * TL + pm] = fHx;
        sp[1 * NFE * TL + pm] = fHy;
        sp[2 * NFE * TL + pm] = fEz;
      }
      mbar_arrive(bars + 3 + b);  // release: the flux of tile it is in F[b]
      if constexpr (WS2) {
        if (it >= 1) epilogue(it - 1);
      }
#pragma unroll
      for (int k = 0; k < KF; ++k) cc[k] = cn[k];
    }
    if constexpr (WS2) epilogue(n_it - 1);
  }
}

#include "kernels_tc.cuh"

template <int MODE, bool MAT>
cudaError_t launch_one(const dg::StageArgs& a, cudaStream_t s) {
  if constexpr (USE_TC) {
    return tc::launch_one<MODE, MAT>(a, s);
  } else {
  using MT = ModeTraits<MODE>;
  if constexpr (WS && MODE == dg::MODE_FUSED_RK) {  // warp-specialised fused stage: one CTA per SM
    constexpr size_t smem = ws_smem(MAT);
    static int grid_ws[64] = {0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 64) return cudaErrorInvalidDevice;
    if (grid_ws[dev] == 0) {
      e = cudaFuncSetAttribute(stage_kernel_ws<MODE, MAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return cudaGetLastError(), e;
      int per_sm = 0, sms = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stage_kernel_ws<MODE, MAT>, TEAM_WS, smem);
      if (e != cudaSuccess) return e;
      e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (e != cudaSuccess) return e;
      grid_ws[dev] = (per_sm > 0 ? per_sm : 1) * sms;
    }
    int grid = a.ntiles < grid_ws[dev] ? a.ntiles : grid_ws[dev];
    if (a.max_ctas > 0 && grid > a.max_ctas) grid = a.max_ctas;
    if (grid <= 0) return cudaSuccess;
    stage_kernel_ws<MODE, MAT><<<grid, TEAM_WS, smem, s>>>(a);
    return cudaGetLastError();
  }
  constexpr size_t smem = smem_total(nslots(MT::surf, MAT), MT::surf, MAT, MT::rk);
  static int grid_cap[64] = {0};  // resident CTAs (whole GPU) per device ordinal
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64) return cudaErrorInvalidDevice;
  if (grid_cap[dev] == 0) {
    e = cudaFuncSetAttribute(stage_kernel<MODE, MAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cudaGetLastError(), e;
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stage_kernel<MODE, MAT>, TEAM, smem);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    grid_cap[dev] = (per_sm > 0 ? per_sm : 1) * sms;
  }
  int grid = a.ntiles < grid_cap[dev] ? a.ntiles : grid_cap[dev];
  if (a.max_ctas > 0 && grid > a.max_ctas) grid = a.max_ctas;
  if (grid <= 0) return cudaSuccess;
  stage_kernel<MODE, MAT><<<grid, TEAM, smem, s>>>(a);
  return cudaGetLastError();
  }
}

cudaError_t launch(int mode, bool mat, const dg::StageArgs& a, cudaStream_t s) {
#ifdef DG_TUNE_ONLY  // autotuning builds: only the fused constant-material kernel
  if (mode == dg::MODE_FUSED_RK && !mat) return launch_one<dg::MODE_FUSED_RK, false>(a, s);
  return cudaErrorNotSupported;
#else
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
#endif
}

// Host: pack Dr, Ds [Np][Np] and LIFT [Np][3Nfp] (fp64, row-major) into the
// kernels' shared-memory operator layout (rounded once to T; padded rows and
// columns are zero).
size_t ops_bytes() { return USE_TC ? tc::OPS : OPB; }
void pack_ops(const double* Dr, const double* Ds, const double* LIFT, void* out) {
  unsigned char* o = static_cast<unsigned char*>(out);
  if constexpr (USE_TC) {
    tc::pack(Dr, Ds, LIFT, o);
    return;
  }
  for (size_t i = 0; i < OPB; ++i) o[i] = 0;
  if constexpr (USE_MMA) {  // A fragments: lane -> (row 8g + lane/4, column 4k + lane%4)
    T* av = reinterpret_cast<T*>(o);
    T* al = reinterpret_cast<T*>(o + DVB);
    for (int g = 0; g < PR; ++g)
      for (int ln = 0; ln < 32; ++ln) {
        const int n = 8 * g + ln / 4;
        for (int ks = 0; ks < KV; ++ks) {
          const int j = 4 * ks + ln % 4;
          T* e = av + ((size_t)(ks * PR + g) * 32 + ln) * 2;
          if (n < NP && j < NP) {
            e[0] = static_cast<T>(Dr[n * NP + j]);
            e[1] = static_cast<T>(Ds[n * NP + j]);
          }
        }
        for (int ks = 0; ks < KL; ++ks) {
          const int m = 4 * ks + ln % 4;
          if (n < NP && m < NF) al[(size_t)(ks * PR + g) * 32 + ln] = static_cast<T>(LIFT[n * NF + m]);
        }
      }
    return;
  }
  if constexpr (USE_TF) {  // B fragments: lane -> (k = 8ks + lane%4 (+4), output row 8nt + lane/4)
    auto tf32_hi = [](double x) {  // round to nearest (ties away) at 10 mantissa bits, as cvt.rna.tf32
      const float f = static_cast<float>(x);
      uint32_t u;
      std::memcpy(&u, &f, 4);
      u = (u + 0x1000u) & 0xFFFFE000u;
      float h;
      std::memcpy(&h, &u, 4);
      return h;
    };
    float* bv = reinterpret_cast<float*>(o);
    float* bl = reinterpret_cast<float*>(o + DVB);
    for (int nt = 0; nt < NT; ++nt)
      for (int ln = 0; ln < 32; ++ln) {
        const int n = 8 * nt + ln / 4;
        for (int ks = 0; ks < KVT; ++ks)
          for (int kh = 0; kh < 2; ++kh) {
            const int j = 8 * ks + ln % 4 + 4 * kh;
            const double dr = (n < NP && j < NP) ? Dr[n * NP + j] : 0.0;
            const double ds = (n < NP && j < NP) ? Ds[n * NP + j] : 0.0;
            float* e = bv + ((size_t)(ks * NT + nt) * 64 + ln) * 4;  // float4 hi; float4 lo 32 lanes on
            e[0 + kh] = tf32_hi(dr);
            e[2 + kh] = tf32_hi(ds);
            e[128 + kh] = tf32_hi(dr - tf32_hi(dr));  // lo parts rounded to tf32 here (free), not
            e[130 + kh] = tf32_hi(ds - tf32_hi(ds));  // truncated by the MMA
          }
        for (int ks = 0; ks < KLT; ++ks)
          for (int kh = 0; kh < 2; ++kh) {
            const int m = 8 * ks + ln % 4 + 4 * kh;
            const double l = (n < NP && m < NF) ? LIFT[n * NF + m] : 0.0;
            float* e = bl + ((size_t)(ks * NT + nt) * 32 + ln) * 4;
            e[kh] = tf32_hi(l);
            e[2 + kh] = tf32_hi(l - tf32_hi(l));
          }
      }
    return;
  }
  T* dv = reinterpret_cast<T*>(o);
  for (int jc = 0; jc < NPC; ++jc)
    for (int n = 0; n < RP; ++n)
      for (int k = 0; k < VC; ++k) {
        const int j = jc * VC + k;
        T* e = dv + ((size_t)(jc * RP + n) * VC + k) * 2;
        if (n < NP && j < NP) {
          e[0] = static_cast<T>(Dr[n * NP + j]);
          e[1] = static_cast<T>(Ds[n * NP + j]);
        }
      }
  T* lv = reinterpret_cast<T*>(o + DVB);
  for (int mc = 0; mc < NFC; ++mc)
    for (int n = 0; n < RP; ++n)
      for (int k = 0; k < VC; ++k) {
        const int m = mc * VC + k;
        if (n < NP && m < NF) lv[(size_t)(mc * RPL + n) * VC + k] = static_cast<T>(LIFT[n * NF + m]);
      }
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
  k.threads = USE_TC ? tc::NTH : (WS ? TEAM_WS : TEAM);
  k.slots = USE_TC ? 1 : nslots(true, false);
  k.row_groups = P;
  k.rows_per_group = R;
  k.smem_bytes = USE_TC ? tc::smem_bytes(false) : (WS ? ws_smem(false) : smem_total(nslots(true, false), true, false, true));
  k.contraction = USE_TC ? 3 : (USE_TF ? 2 : (USE_MMA ? 1 : 0));
  k.residual_tma = RES_TMA ? 1 : 0;
  k.teams_cap = DG_C;
  k.flags = USE_TC ? 0 : (FLUX_FIRST ? 1 : 0) | (OPS_GLOBAL ? 2 : 0) | (FX ? 4 : 0) | (USE_TF && IL ? 8 : 0) |
                         (ZC_CONN ? 16 : 0) | (ZC && !ZC_CONN ? 32 : 0) | (WPRE ? 64 : 0) | (DMMA_U ? 128 : 0) | (WS ? 256 : 0);
  return k;
}

}  // namespace

namespace dg {
KernelModule DG_CAT(dg_module_, DG_TAG)() {
  KernelModule m;
  m.N = N;
  m.prec = (int)sizeof(T);
  m.ops_bytes = &ops_bytes;
  m.pack_ops = &pack_ops;
  m.launch = &launch;
  m.info = &info;
  m.check_fmask = &check_fmask;
  m.swizzle = SWM;
  m.tile_group = USE_TC ? tc::TG : 1;
  m.variant = DG_VARIANT;
  m.compressed = DG_ZC;
  return m;
}
}  // namespace dg
