/*
 * dg3.h -- C ABI of the 3D tetrahedral Maxwell hot path (the paper's
 *          "hedge" workload, "Three Dimensions", figures).
 *
 * The library advances (Hx, Hy, Hz, Ex, Ey, Ez) of
 *     dH/dt = -curl E,   dE/dt = curl H      (eps = mu = 1; the 3D form of PAPER.md:167-181)
 * on K straight-sided, face-conforming tetrahedra with the nodal DG method of order N: the
 * semi-discrete operator of eq. 9 one dimension up (d/dx = rx Dr + sx Ds + tx Dt),
 * the upwind flux in the 1/2 jump form of reading A3, PEC walls (E+ = -E-, H+ = H-),
 * LSERK4 in time.  Kernels: the paper's two-kernel structure -- a volume kernel and a surface +
 * LIFT kernel with the LSERK4 update fused (kernels3d.cuh).  Single GPU, constant material.
 *
 * Conventions: reference tetrahedron {r,s,t >= -1, r+s+t <= -1}; warp-and-blend
 * nodes, t slowest, r fastest; faces f0 (v0,v1,v2) t = -1, f1 (v0,v1,v3) s = -1, f2 (v1,v2,v3)
 * r+s+t = -1, f3 (v0,v2,v3) r = -1, each face's nodes in increasing node index; canonical field
 * layout [K][Np]; EToV 0-based [K][4]; negatively oriented elements have local vertices 1 <-> 2
 * swapped (count in dg3_sizes).
 *
 * Ownership, errors and threading are those of dg.h: pointers are borrowed for the call; every
 * function returns dg_status (dg_last_error() describes the last failure); after DG_E_CUDA the
 * context is poisoned.  A context with options.device = -1 is host-only (setup and exports only).
 */
#ifndef DG3_H_
#define DG3_H_

#include <stdint.h>

#include "dg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dg3_ctx dg3_ctx;

/* Maximum N with compiled 3D device kernels (shared-memory bound at fp64). */
#define DG3_MAX_KERNEL_N 5

/* Build a 3D context.  options: abi_version, N (setup 1..15, kernels 1..DG3_MAX_KERNEL_N),
 * precision (4|8), device, alpha, stream, max_ctas and fused are used (fused = 1: one fused stage
 * kernel -- volume, flux, LIFT and LSERK4 update -- per stage wherever its tile fits in shared memory,
 * else, and with fused = 0, the volume kernel then the surface+LIFT+RK kernel); rank/nranks must be
 * 0/1; the other fields are ignored.  VX, VY, VZ [Nv] (host fp64), EToV [K][4] (host int64, 0-based). */
dg_status dg3_setup(const dg_options* opts, int64_t Nv, const double* VX, const double* VY, const double* VZ,
                    int64_t K, const int64_t* EToV, dg3_ctx** out);

/* Np = (N+1)(N+2)(N+3)/6, Nfp = (N+1)(N+2)/2, K, re-oriented element count.  NULL skips. */
dg_status dg3_sizes(const dg3_ctx* c, int64_t* Np, int64_t* Nfp, int64_t* K, int64_t* n_swapped);

/* fields[6] = (Hx, Hy, Hz, Ex, Ey, Ez), each fp64 [K][Np], host or this device's memory.
 * set: resets the LSERK4 residual; get: synchronises the stream. */
dg_status dg3_set_fields(dg3_ctx* c, const double* const* fields);
dg_status dg3_get_fields(dg3_ctx* c, double* const* fields);

/* nsteps LSERK4 steps of size dt > 0 (2 kernel launches per stage), enqueued on the stream. */
dg_status dg3_run(dg3_ctx* c, double dt, int64_t nsteps);

/* Synchronise; DG_E_DIVERGED if any field value is non-finite. */
dg_status dg3_sync(dg3_ctx* c);

/* d/dt of the current fields into out[6] (host fp64 [K][Np]): which 0 full, 1 volume, 2 surface. */
dg_status dg3_eval_rhs(dg3_ctx* c, int32_t which, double* const* out);

/* 1/2 sum_k J_k sum_fields u^T M u (host fp64 from downloaded fields). */
dg_status dg3_energy(dg3_ctx* c, double* E);

/* Verification exports (host fp64; valid on host-only contexts).  NULL skips an output.
 * r, s, t [Np]; Dr, Ds, Dt [Np][Np]; LIFT [Np][4 Nfp]; Fmask [4][Nfp]. */
dg_status dg3_get_operators(const dg3_ctx* c, double* r, double* s, double* t, double* Dr, double* Ds, double* Dt,
                            double* LIFT, int32_t* Fmask);
/* EToE [K][4], EToF [K][4], vmapP [K][4][Nfp] (canonical k Np + n; boundary = own node). */
dg_status dg3_get_maps(const dg3_ctx* c, int32_t* EToE, int8_t* EToF, int64_t* vmapP);
/* Node coordinates x, y, z [K][Np]. */
dg_status dg3_get_nodes(const dg3_ctx* c, double* x, double* y, double* z);
/* Geometry: gfac [K][9] = (rx, ry, rz, sx, sy, sz, tx, ty, tz); J [K]; per face [K][4]: nx, ny, nz, sJ, Fsc. */
dg_status dg3_get_geometry(const dg3_ctx* c, double* gfac, double* J, double* nx, double* ny, double* nz,
                           double* sJ, double* Fsc);

/* Measurement: the stream; per-launch CUDA-event timing (launches[1] volume, [2] surface+RK). */
dg_status dg3_stream(const dg3_ctx* c, void** stream);
dg_status dg3_profile(dg3_ctx* c, int32_t enable);
dg_status dg3_get_kernel_stats(dg3_ctx* c, dg_kernel_stats* out);

void dg3_destroy(dg3_ctx* c);

#ifdef __cplusplus
}
#endif
#endif /* DG3_H_ */
