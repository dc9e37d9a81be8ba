/*
 * dg.h -- C ABI of the B200-native nodal-DG 2D TM Maxwell hot path
 *         (arxiv 1304.5546, "GPU nodal DG", PAPER.md).
 *
 * The library advances the transverse-magnetic Maxwell fields (Hx, Hy, Ez)
 *     mu dHx/dt = -dEz/dy,  mu dHy/dt = +dEz/dx,  eps dEz/dt = dHy/dx - dHx/dy
 * (eq. 2a-c, with the eq. 2b sign reading A1 of DESIGN.md)
 * on K straight-sided, face-conforming triangles with the
 * nodal DG method of order N: the semi-discrete operator of eq. 9
 * (reading A2) with the upwind flux 1/2 * eq. 5
 * (reading A3), PEC walls Ez = 0 (
 * reading A7), optional piecewise-constant eps/mu (reading A12), integrated in
 * time by the 5-stage low-storage RK4 (reading A10).
 *
 * dg_setup builds everything on the host in fp64 (nodes, Dr/Ds, LIFT,
 * geometric factors, connectivity, face maps, partition) and uploads it;
 * dg_run enqueues the hand-written sm_100a kernels.  No CPU fallback exists:
 * a context created with device >= 0 fails with DG_E_CUDA if no device is
 * usable.  A context created with device = -1 is HOST-ONLY: the setup and the
 * verification exports work, every compute call returns DG_E_STATE.
 *
 * Conventions:
 *  - reference triangle {r,s >= -1, r+s <= 0}; warp-and-blend nodes, r
 *    fastest, rows bottom->top; faces f0=(v0,v1), f1=(v1,v2), f2=(v2,v0);
 *  - canonical field layout [K][Np] (element-major, node order above);
 *    canonical global DOF index k*Np + n;
 *  - EToV is 0-based; clockwise elements are re-oriented by swapping local
 *    vertices 1 <-> 2 (the count is returned by dg_sizes);
 *  - Fmask_f lists face nodes in increasing node index.
 *
 * Ownership: every pointer argument is borrowed for the duration of the call;
 * dg_setup copies what it keeps.  Output arrays are caller-allocated with the
 * sizes given by dg_sizes / dg_halo_sizes.  Device memory is owned by the
 * context and released by dg_destroy.
 *
 * Errors: every function returns dg_status and never aborts; dg_last_error()
 * returns a thread-local message for the last failure.  After DG_E_CUDA or
 * DG_E_NCCL the context is poisoned: only dg_destroy is valid.
 *
 * Threading: one context per host thread (or process); contexts are
 * independent.  dg_run_group drives several contexts from one thread.
 */
#ifndef DG_H_
#define DG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_ABI_VERSION 2

typedef struct dg_ctx dg_ctx;

typedef enum {
  DG_OK = 0,
  DG_E_ARG = 1,                /* invalid argument (null pointer, size, dt <= 0 ...) */
  DG_E_DEGREE = 2,             /* N outside [1, 15] for setup, or no kernel compiled for N */
  DG_E_MESH_DEGENERATE = 3,    /* |J| < 1e-14 * (longest edge)^2 */
  DG_E_MESH_NONMANIFOLD = 4,   /* an edge shared by > 2 elements */
  DG_E_MESH_NONCONFORMING = 5, /* face nodes of neighbours differ by > 1e-8 * edge length */
  DG_E_UNSUPPORTED_BC = 6,     /* bctag value other than 0 (auto) / 1 (PEC), or PEC on an interior face */
  DG_E_CUDA = 7,               /* CUDA failure or no usable device; context poisoned */
  DG_E_NCCL = 8,               /* NCCL failure; context poisoned */
  DG_E_OOM = 9,                /* device or host allocation failed */
  DG_E_DIVERGED = 10,          /* non-finite field value found by dg_sync */
  DG_E_STATE = 11              /* call not valid in this state (host-only context, poisoned ...) */
} dg_status;

typedef struct {
  int32_t abi_version;   /* must be DG_ABI_VERSION */
  int32_t N;             /* polynomial degree: setup accepts 1..15; kernels are compiled for 1..DG_MAX_KERNEL_N */
  int32_t precision;     /* 4 = fp32, 8 = fp64 arithmetic on the device */
  int32_t device;        /* CUDA ordinal; -1 = host-only context (no device is touched) */
  double alpha;          /* flux parameter: 1 = upwind (default), 0 = central */
  int32_t rank;          /* this process' partition index, 0 <= rank < nranks */
  int32_t nranks;        /* number of partitions (processes/GPUs); 1 = single GPU */
  int32_t fused;         /* kernel variant: 1 = fused single-kernel stage (default),
                            0 = split: volume kernel, then surface+LIFT+RK kernel */
  int32_t transport;     /* halo transport when nranks > 1: 0 = NCCL send/recv (one process per GPU),
                            1 = in-process group (dg_run_group, all contexts on one device) */
  const void* nccl_id;   /* 128-byte ncclUniqueId made by rank 0 and broadcast by the caller;
                            required when nranks > 1 and transport == 0, else ignored */
  const int32_t* part;   /* optional [K] element -> rank map; NULL = contiguous blocks
                            [r*K/P, (r+1)*K/P) of the input element order */
  void* stream;          /* cudaStream_t to enqueue on; NULL = the context creates its own */
  /* ---- ABI 2 ---- */
  int32_t max_ctas;      /* cap on the persistent stage kernels' grid (CTAs over the whole GPU);
                            0 = every resident CTA (default).  A small cap makes each CTA walk many
                            tiles through its shared-memory pipeline on a small mesh (slot reuse,
                            mbarrier phase flips, next-tile prefetch): the parity tests use it to
                            exercise at oracle size the code paths the full-size runs take. */
  int32_t tile_order;    /* order in which each stage walks the tiles: 0 = first to last every stage
                            (default); 1 = odd LSERK4 stages last to first.  Never changes a result. */
  int32_t check_every;   /* 0 = off (default); S > 0: dg_run checks the fields for non-finite values
                            after every S-th step on the device (one extra read of q), so dg_sync can
                            report the first step found bad */
  int32_t kernel_variant; /* 0 = the stage kernels tuned for this (N, precision) (default; see
                             dg_get_kernel_config); 1 = fp32 only: the tcgen05 kernels (5th-generation
                             tensor cores, TMEM accumulators, 128-element groups) */
} dg_options;

/* Maximum N with compiled device kernels. */
#define DG_MAX_KERNEL_N 9

/* Fill *o with defaults: abi_version, N=4, fp64, device 0, alpha 1, rank 0 of 1, fused, NCCL,
 * max_ctas 0, tile_order 0, check_every 0, kernel_variant 0. */
dg_status dg_options_default(dg_options* o);

/* Build a context (PAPER.md:139-198 problem statement; SURVEY.md §3 call stack 1).
 *   VX, VY [Nv]     vertex coordinates (host, fp64)
 *   EToV   [K][3]   0-based vertex ids (host, int64)
 *   eps, mu [K]     element permittivity / permeability (host, fp64, > 0), or both NULL for
 *                   eps = mu = 1 (the paper's constant-coefficient case)
 *   bctag  [K][3]   per face: 0 = interior, or PEC if on the boundary; 1 = PEC; NULL = all 0
 * Every rank passes the same GLOBAL mesh; the context keeps its partition. */
dg_status dg_setup(const dg_options* opts, int64_t Nv, const double* VX, const double* VY,
                   int64_t K, const int64_t* EToV, const double* eps, const double* mu,
                   const int8_t* bctag, dg_ctx** out);

/* Sizes: Np = (N+1)(N+2)/2, Nfp = N+1, local / global element counts, number of received halo
 * face points, number of re-oriented (clockwise) input elements.  Any pointer may be NULL. */
dg_status dg_sizes(const dg_ctx* c, int64_t* Np, int64_t* Nfp, int64_t* K_local, int64_t* K_global,
                   int64_t* n_halo_points, int64_t* n_swapped);

/* Global element ids of the local elements, in local order [K_local]. */
dg_status dg_local_elements(const dg_ctx* c, int64_t* gid);

/* Upload fields (fp64, canonical [K_local][Np]); resets the RK residual to 0.  Each pointer may be
 * host memory (pageable or pinned) or device memory of this context's device (detected with
 * cudaPointerGetAttributes; copied with cudaMemcpyDefault).  Enqueued on the context's stream;
 * host sources are read before the call returns. */
dg_status dg_set_fields(dg_ctx* c, const double* Hx, const double* Hy, const double* Ez);

/* Download fields (fp64, canonical [K_local][Np]) into host or device memory (as dg_set_fields);
 * synchronises the context's stream. */
dg_status dg_get_fields(dg_ctx* c, double* Hx, double* Hy, double* Ez);

/* Advance nsteps LSERK4 steps of size dt (> 0): 5 stages per step, each one evaluation of the
 * semi-discrete operator plus the low-storage update.  Enqueues on the
 * context's stream and returns without synchronising. nsteps == 0 is a no-op. */
dg_status dg_run(dg_ctx* c, double dt, int64_t nsteps);

/* Advance several in-process partitions (transport == 1 contexts of one mesh, ranks 0..n-1, all on
 * one device) in lock step; the halo exchange is a device-to-device copy.  Each fused stage runs as
 * the NCCL path runs it: the interior tiles (no halo point) first, then the partition-boundary
 * tiles (through the kernels' tile lists).  Bitwise identical to a single-partition run (SURVEY.md
 * P17). */
dg_status dg_run_group(dg_ctx* const* ctxs, int32_t n, double dt, int64_t nsteps);

/* Synchronise the stream and check all fields for non-finite values: DG_E_DIVERGED, with the
 * step index in dg_last_error().  With options.check_every = S > 0 the message names the FIRST
 * checked step at which a non-finite value appeared (exact for S = 1; for S > 1 the divergence
 * happened within the S steps before it); with S = 0 it names the step count so far. */
dg_status dg_sync(dg_ctx* c);

/* Evaluate d/dt (Hx, Hy, Ez) of the current fields (host fp64 out, canonical [K_local][Np]);
 * which: 0 = full operator, 1 = volume term only (H2), 2 = surface term only (H3-H5). */
dg_status dg_eval_rhs(dg_ctx* c, int32_t which, double* rHx, double* rHy, double* rEz);

/* Discrete energy 1/2 sum_k J_k (mu_k H^T M H + eps_k Ez^T M Ez) of the WHOLE mesh:
 * fp64 on the host from downloaded fields, then, for an NCCL context (nranks > 1, transport 0),
 * summed over the ranks with ncclAllReduce (every rank must call it; collective).  For in-process
 * group contexts (transport 1) it is the local energy: sum dg_energy_local over the group. */
dg_status dg_energy(dg_ctx* c, double* E);

/* The same sum over this context's local elements only (no communication). */
dg_status dg_energy_local(dg_ctx* c, double* E);

/* ---- verification exports (host fp64, valid on host-only contexts) ---- */

/* r, s [Np]; Dr, Ds [Np][Np]; LIFT [Np][3Nfp] (row-major); Fmask [3][Nfp].  NULL skips. */
dg_status dg_get_operators(const dg_ctx* c, double* r, double* s, double* Dr, double* Ds,
                           double* LIFT, int32_t* Fmask);

/* Per local element: rx, sx, ry, sy, J [K_local]; per face: nx, ny, sJ, Fsc [K_local][3]. */
dg_status dg_get_geometry(const dg_ctx* c, double* rx, double* sx, double* ry, double* sy,
                          double* J, double* nx, double* ny, double* sJ, double* Fsc);

/* Connectivity (global ids) and face maps (canonical global DOF k*Np+n) of the local elements:
 * EToE [K_local][3], EToF [K_local][3], vmapM / vmapP [K_local][3][Nfp].  NULL skips. */
dg_status dg_get_maps(const dg_ctx* c, int32_t* EToE, int8_t* EToF, int64_t* vmapM, int64_t* vmapP);

/* Physical node coordinates x, y [K_local][Np]. */
dg_status dg_get_nodes(const dg_ctx* c, double* x, double* y);

/* Halo list sizes: number of neighbour ranks, total sent and received face points. */
dg_status dg_halo_sizes(const dg_ctx* c, int32_t* n_nbr, int64_t* n_send, int64_t* n_recv);

/* Halo lists.  nbr [n_nbr] neighbour ranks ascending; send_off / recv_off [n_nbr+1] offsets;
 * send_gdof [n_send]: canonical global DOFs of OWN nodes sent to nbr[i] (in the receiver's
 * face-point order); recv_gdof [n_recv]: canonical global DOFs received from nbr[i];
 * recv_point [n_recv]: the local face point ((k_local*3 + f)*Nfp + i) each one feeds. */
dg_status dg_get_halo(const dg_ctx* c, int32_t* nbr, int64_t* send_off, int64_t* send_gdof,
                      int64_t* recv_off, int64_t* recv_gdof, int64_t* recv_point);

/* ---- measurement ---- */

/* The cudaStream_t the context enqueues on (so callers can record events on it). */
dg_status dg_stream(const dg_ctx* c, void** stream);

typedef struct {
  int64_t launches[4];   /* kernel launches since the last reset: [0] fused stage, [1] volume,
                            [2] surface+RK, [3] halo pack (+ other helpers) */
  double  ms[4];         /* summed CUDA-event durations per kind (only while profiling is on) */
  int64_t timed[4];      /* launches that were event-timed */
} dg_kernel_stats;

/* CUDA graphs for dg_run (single-rank contexts; default on): after one eager step, each
 * LSERK4 step (its 5 stage launches) is captured once per ping-pong parity for the current
 * dt and replayed with cudaGraphLaunch -- the same kernels and arguments, bitwise the same
 * result.  A new dt recaptures.  While profiling (dg_profile) the replayed graph is a
 * second capture with event-record nodes around every launch, and dg_run waits for each
 * step to read them (between steps, outside every bracket).  0 disables (and frees the
 * graphs after synchronising the stream). */
dg_status dg_set_graphs(dg_ctx* c, int32_t enable);

/* Turn per-launch CUDA-event timing on (1) or off (0); resets the statistics.  Eager
 * launches are bracketed by events on the launching stream; graph replays by event-record
 * nodes inside the graph (see dg_set_graphs). */
dg_status dg_profile(dg_ctx* c, int32_t enable);

/* Read the statistics (synchronises the stream when profiling is on). */
dg_status dg_get_kernel_stats(dg_ctx* c, dg_kernel_stats* out);

/* The stage-kernel configuration compiled for this context's (N, precision): the knob set
 * tools/tune.py picked (csrc/tune.json).  Host-only contexts included. */
typedef struct {
  int32_t contraction;   /* volume + LIFT contractions: 0 = CUDA-core FMA (FFMA/DFMA),
                            1 = fp64 tensor cores (DMMA, mma.sync m8n8k4),
                            2 = fp32 on tensor cores as 3xTF32 (mma.sync m16n8k8; each operand
                                split hi + lo, hi*hi + lo*hi + hi*lo in fp32 accumulation),
                            3 = fp32 as 3xTF32 on the 5th-generation tensor cores (tcgen05.mma
                                kind::tf32, M = 128 elements, A operands and accumulators in TMEM) */
  int32_t threads;       /* threads per CTA; one CTA owns one 32-element tile at a time */
  int32_t slots;         /* shared-memory pipeline slots (1 or 2) */
  int32_t residual_tma;  /* 1: the LSERK4 residual is staged into shared memory by TMA */
  int32_t teams_cap;     /* cap on resident CTAs per SM (launch bounds) */
  int32_t flags;         /* bit 0: flux phase before the volume phase (knob F);
                            bit 1: tensor-core operator fragments read through L1 from global
                            memory instead of a shared-memory copy per CTA (knob G);
                            bit 2: flux computed straight into the LIFT A fragments (knob X);
                            bit 3: 3xTF32 products issued pass by pass (knob I);
                            bit 4: compressed connectivity for constant-material contexts: one word
                                   per face instead of one code per face point, face normals and Fsc
                                   derived on chip from rx, sx, ry, sy (knob Z = 1);
                            bit 5: geometry-only compression: the face normals and Fsc derived on chip,
                                   one neighbour code per face point as uncompressed (knob Z = 2) */
  int64_t smem_bytes;    /* dynamic shared memory per CTA of the fused stage kernel */
} dg_kernel_config;
dg_status dg_get_kernel_config(const dg_ctx* c, dg_kernel_config* out);

/* Release everything.  Accepts NULL. */
void dg_destroy(dg_ctx* c);

/* Thread-local description of the last error. */
const char* dg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DG_H_ */
