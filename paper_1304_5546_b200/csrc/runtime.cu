// C ABI implementation (include/dg.h): context, device buffers, stage loop,
// halo exchange (NCCL send/recv or in-process copies), helper kernels.
//
// SURVEY.md §3 call stacks 1-2: dg_setup builds the host fp64 data (setup.cpp),
// uploads it in the tile-blocked layout (kernel_api.h) and the operators to the
// (N, precision) kernel module's constant bank; dg_run enqueues, per LSERK4
// stage, [halo pack -> NCCL send/recv on the comm stream] overlapped with the
// interior stage kernels, then the partition-boundary stage kernels.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/dg.h"
#include "kernel_api.h"
#include "setup.h"

// ---------------------------------------------------------------- module registry
namespace dg {
#define DG_MODULE(tag) KernelModule dg_module_##tag();
#include "modules.inc"
#undef DG_MODULE

const KernelModule* find_module(int N, int prec, int variant) {
  static const std::vector<KernelModule> mods = {
#define DG_MODULE(tag) dg_module_##tag(),
#include "modules.inc"
#undef DG_MODULE
  };
  for (const auto& m : mods)
    if (m.N == N && m.prec == prec && m.variant == variant) return &m;
  return nullptr;
}
}  // namespace dg

namespace {

thread_local std::string g_err;

dg_status set_err(dg_status s, const std::string& m) {
  g_err = m;
  return s;
}

}  // namespace

namespace dg {
void set_last_error(const std::string& m) { g_err = m; }  // the 3D calls (runtime3d.cu) report here too
}  // namespace dg

namespace {

// LSERK4 (Carpenter-Kennedy 5-stage, 4th order; reading A10)
const double kRKa[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                        -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double kRKb[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                        1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                        2277821191437.0 / 14882151754819.0};

// ---------------------------------------------------------------- NCCL (dlopen'd)
struct Nccl {
  bool ok = false;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl* nccl() {
  static Nccl n;
  static bool tried = false;
  if (tried) return n.ok ? &n : nullptr;
  tried = true;
  // prefer the NCCL already mapped into the process (torch's), else the system one
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
#define LOADSYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name)); if (!n.field) return nullptr;
  LOADSYM(CommInitRank, "ncclCommInitRank")
  LOADSYM(CommDestroy, "ncclCommDestroy")
  LOADSYM(CommAbort, "ncclCommAbort")
  LOADSYM(GroupStart, "ncclGroupStart")
  LOADSYM(GroupEnd, "ncclGroupEnd")
  LOADSYM(Send, "ncclSend")
  LOADSYM(Recv, "ncclRecv")
  LOADSYM(AllReduce, "ncclAllReduce")
  LOADSYM(GetErrorString, "ncclGetErrorString")
#undef LOADSYM
  n.ok = true;
  return &n;
}

// ---------------------------------------------------------------- helper kernels
// canonical fp64 [3][Kl][Np]  <->  tile-blocked T [3][fstride].  Device slot d
// (tile d/32, lane d%32) holds local element perm[d] (-1: padding);
// slot_of[kl] is the inverse.
// (column swizzle swm: element `lane` of node row n sits at column dg::swz_col(swm, n, lane))
template <typename T>
__global__ void to_blocked(const double* __restrict__ src, T* __restrict__ q, const int32_t* __restrict__ perm,
                           int64_t Kl, int64_t Kpad, int Np, int64_t fstride, int swm) {
  const int64_t total = Kpad * Np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / total);
    const int64_t o = i - c * total;           // blocked offset within field: (t*Np + n)*32 + column
    const int64_t tn = o >> 5;
    const int64_t t = tn / Np;
    const int n = (int)(tn - t * Np);
    const int lane = dg::swz_col(swm, n, (int)(o & 31));
    const int64_t kl = perm[t * 32 + lane];
    q[c * fstride + o] = (kl >= 0) ? static_cast<T>(src[(c * Kl + kl) * Np + n]) : T(0);
  }
}

template <typename T>
__global__ void from_blocked(const T* __restrict__ q, double* __restrict__ dst, const int32_t* __restrict__ slot_of,
                             int64_t Kl, int Np, int64_t fstride, int swm) {
  const int64_t total = Kl * Np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / total);
    const int64_t o = i - c * total;  // canonical kl*Np + n
    const int64_t kl = o / Np;
    const int n = (int)(o - kl * Np);
    const int64_t d = slot_of[kl];
    dst[c * total + o] =
        static_cast<double>(q[c * fstride + ((d >> 5) * Np + n) * 32 + dg::swz_col(swm, n, (int)(d & 31))]);
  }
}

// halo pack: send[c][s] = q[c][idx[s]]
template <typename T>
__global__ void halo_pack(const T* __restrict__ q, T* __restrict__ send, const int32_t* __restrict__ idx, int64_t n,
                          int64_t fstride) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / n);
    const int64_t s = i - c * n;
    send[i] = q[c * fstride + idx[s]];
  }
}

template <typename T>
__global__ void count_nonfinite(const T* __restrict__ q, int64_t n, int64_t fstride, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / n);
    const T v = q[c * fstride + (i - c * n)];
    if (!isfinite(v)) ++local;
  }
  if (local) atomicAdd(bad, local);
}

// dg_options.check_every: the first checked step at which a field value is non-finite
// (*first starts at ~0ull; non-finite values never become finite again under the scheme's
// arithmetic, so the minimum over checks is the first bad check)
template <typename T>
__global__ void mark_nonfinite(const T* __restrict__ q, int64_t n, int64_t fstride, unsigned long long step,
                               unsigned long long* first) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / n);
    bad |= !isfinite(q[c * fstride + (i - c * n)]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMin(first, step);
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

// ---------------------------------------------------------------- context
struct dg_ctx {
  // options
  int N = 0, prec = 8, device = -1, rank = 0, nranks = 1, fused = 1, transport = 0;
  int max_ctas = 0, tile_order = 0, check_every = 0, kernel_variant = 0;
  double alpha = 1.0;
  bool host_only = true, poisoned = false, material = false;
  // host setup
  dg::RefElem ref;
  dg::Mesh mesh;
  std::vector<double> eps_l, mu_l;  // per local element
  const dg::KernelModule* km = nullptr;
  // sizes
  int64_t Kl = 0, ntiles = 0, Kpad = 0, fstride = 0, vstride = 0, n_send = 0, n_recv = 0, ghost_base = 0;
  int64_t group = 1, ngroups = 0;  // tiles per kernel work unit (KernelModule::tile_group), units
  size_t tsz = 8;
  int ngeo = dg::NGEO_CONST;
  int compressed = 0;  // 1: compressed connectivity, 2: geometry only (module knob, constant material)
  // device buffers
  void* q[2] = {nullptr, nullptr};
  void* res = nullptr;
  void* rhsv = nullptr;
  void* out = nullptr;
  void* geo = nullptr;
  void* ops = nullptr;
  int32_t* vmapP = nullptr;
  int32_t* send_idx = nullptr;
  int32_t* perm_d = nullptr;     // [Kpad] device slot -> local element (-1 = padding)
  int32_t* slot_of_d = nullptr;  // [Kl]   local element -> device slot
  std::vector<int64_t> perm, slot_of;  // host copies
  void* sendbuf = nullptr;
  double* stage = nullptr;   // fp64 staging [3][Kl][Np]
  unsigned long long* flag = nullptr;
  unsigned long long* first_bad = nullptr;  // check_every: first checked step with a non-finite value
  double* ebuf = nullptr;                   // dg_energy all-reduce buffer
  int32_t* tiles_int = nullptr;
  int32_t* tiles_bnd = nullptr;
  int32_t n_int = 0, n_bnd = 0;
  int cur = 0;
  int64_t steps_done = 0;
  // streams / events
  cudaStream_t stream = nullptr, comm = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
  ncclComm_t nccl_comm = nullptr;
  // CUDA graphs: one LSERK4 step (5 stages) per graph, one per starting ping-pong parity,
  // captured for the current dt (single-rank contexts).  While profiling, a second pair of
  // graphs carries event-record nodes around every launch (pexec/pev below).
  bool graphs = true;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  cudaGraphExec_t pexec[2] = {nullptr, nullptr};
  double gdt = 0.0;
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Timed { int kind; int ev0, ev1; };
  std::vector<Timed> timed;
  int pcap = -1;                        // parity of the profiled graph being captured, else -1
  std::vector<cudaEvent_t> pev[2];      // event-record nodes of profiled graph [parity]
  std::vector<Timed> ptimed[2];         // (kind, event pair) per launch of that graph
  dg_kernel_stats stats{};
};

namespace {

dg_status cuda_fail(dg_ctx* c, cudaError_t e, const char* what) {
  if (c) c->poisoned = true;
  return set_err(DG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CU(ctx, x)                                          \
  do {                                                      \
    cudaError_t e__ = (x);                                  \
    if (e__ != cudaSuccess) return cuda_fail(ctx, e__, #x); \
  } while (0)

dg_status check_usable(const dg_ctx* c, bool need_device) {
  if (!c) return set_err(DG_E_ARG, "null context");
  if (c->poisoned) return set_err(DG_E_STATE, "context is poisoned by an earlier CUDA/NCCL error");
  if (need_device && c->host_only) return set_err(DG_E_STATE, "host-only context (device = -1) cannot compute");
  return DG_OK;
}

// event-timed kernel launch bracket
int take_event(dg_ctx* c) {
  if (c->timed.size() * 2 + 2 > c->ev_pool.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
      c->ev_pool.push_back(e);
    }
  }
  return (int)(c->timed.size() * 2);
}

dg_status launch_stage(dg_ctx* c, int mode, const dg::StageArgs& a, cudaStream_t s, int kind) {
  if (c->pcap >= 0) {  // capturing a profiled graph: external event-record nodes bracket the launch
    std::vector<cudaEvent_t>& pe = c->pev[c->pcap];  // created before the capture began
    const int ev = 2 * (int)c->ptimed[c->pcap].size();
    if (ev + 2 > (int)pe.size()) return set_err(DG_E_STATE, "profiled graph: event pool exhausted");
    CU(c, cudaEventRecordWithFlags(pe[ev], s, cudaEventRecordExternal));
    cudaError_t e = c->km->launch(mode, c->material, a, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "stage kernel launch");
    CU(c, cudaEventRecordWithFlags(pe[ev + 1], s, cudaEventRecordExternal));
    c->ptimed[c->pcap].push_back({kind, ev, ev + 1});
    return DG_OK;
  }
  int ev = -1;
  if (c->profiling) {
    ev = take_event(c);
    if (ev >= 0) CU(c, cudaEventRecord(c->ev_pool[ev], s));
  }
  cudaError_t e = c->km->launch(mode, c->material, a, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "stage kernel launch");
  c->stats.launches[kind] += 1;
  if (ev >= 0) {
    CU(c, cudaEventRecord(c->ev_pool[ev + 1], s));
    c->timed.push_back({kind, ev, ev + 1});
  }
  return DG_OK;
}

dg::StageArgs base_args(dg_ctx* c) {
  dg::StageArgs a{};
  a.q_in = c->q[c->cur];
  a.q_out = c->q[1 - c->cur];
  a.res = c->res;
  a.rhsv = c->rhsv;
  a.out = c->out;
  a.geo = c->geo;
  a.ops = c->ops;
  a.vmapP = c->vmapP;
  a.tiles = nullptr;
  a.fstride = c->fstride;
  a.vstride = c->vstride;
  a.ntiles = (int32_t)c->ngroups;
  a.write_res = 1;
  a.scale_volume = 0;
  a.alpha = c->alpha;
  a.max_ctas = c->max_ctas;
  return a;
}

dg_status pack(dg_ctx* c, cudaStream_t s) {
  if (c->n_send == 0) return DG_OK;
  const void* qin = c->q[c->cur];
  if (c->tsz == 4)
    halo_pack<float><<<grid_for(3 * c->n_send), 256, 0, s>>>((const float*)qin, (float*)c->sendbuf, c->send_idx,
                                                            c->n_send, c->fstride);
  else
    halo_pack<double><<<grid_for(3 * c->n_send), 256, 0, s>>>((const double*)qin, (double*)c->sendbuf, c->send_idx,
                                                             c->n_send, c->fstride);
  CU(c, cudaGetLastError());
  c->stats.launches[3] += 1;
  return DG_OK;
}

// NCCL send/recv of the packed traces into q_in's ghost region, on stream s
dg_status exchange_nccl(dg_ctx* c, cudaStream_t s) {
  Nccl* n = nccl();
  if (!n || !c->nccl_comm) return set_err(DG_E_NCCL, "NCCL unavailable");
  const ncclDataType_t dt = (c->tsz == 4) ? ncclFloat32 : ncclFloat64;
  char* qin = static_cast<char*>(c->q[c->cur]);
  char* sb = static_cast<char*>(c->sendbuf);
  ncclResult_t r = n->GroupStart();
  for (size_t t = 0; r == ncclSuccess && t < c->mesh.nbr.size(); ++t) {
    const int peer = c->mesh.nbr[t];
    const int64_t so = c->mesh.send_off[t], sc = c->mesh.send_off[t + 1] - so;
    const int64_t ro = c->mesh.recv_off[t], rc = c->mesh.recv_off[t + 1] - ro;
    for (int f = 0; f < 3 && r == ncclSuccess; ++f) {
      if (sc > 0) r = n->Send(sb + (f * c->n_send + so) * c->tsz, (size_t)sc, dt, peer, c->nccl_comm, s);
      if (r == ncclSuccess && rc > 0)
        r = n->Recv(qin + (f * c->fstride + c->ghost_base + ro) * c->tsz, (size_t)rc, dt, peer, c->nccl_comm, s);
    }
  }
  ncclResult_t r2 = n->GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    c->poisoned = true;
    return set_err(DG_E_NCCL, std::string("NCCL send/recv: ") + n->GetErrorString(r));
  }
  return DG_OK;
}

dg::StageArgs stage_args(dg_ctx* c, int i, double dt) {
  dg::StageArgs a = base_args(c);
  a.a = kRKa[i];
  a.b = kRKb[i];
  a.dt = dt;
  a.write_res = i == 4 ? 0 : 1;  // the residual is dead after the last stage (a_0 = 0)
  a.reverse = (i & 1) && c->tile_order == 1;
  return a;
}

// The stage kernels of LSERK4 stage i of a partitioned context (nranks > 1) on stream s, the
// same for both transports.  Fused: the interior tiles (no halo point) first, then -- after
// halo_ready(), which makes s wait for the exchange -- the partition-boundary tiles, each
// launch walking its tile list (StageArgs::tiles).  Split: the volume kernel (needs no halo),
// halo_ready(), then the surface + RK kernel.
template <typename WAIT>
dg_status partitioned_stage(dg_ctx* c, const dg::StageArgs& a, cudaStream_t s, const WAIT& halo_ready) {
  dg_status st;
  if (c->fused) {
    dg::StageArgs ai = a;
    ai.tiles = c->tiles_int;
    ai.ntiles = c->n_int;
    if (ai.ntiles > 0 && (st = launch_stage(c, dg::MODE_FUSED_RK, ai, s, 0)) != DG_OK) return st;
    if ((st = halo_ready()) != DG_OK) return st;
    dg::StageArgs ab = a;
    ab.tiles = c->tiles_bnd;
    ab.ntiles = c->n_bnd;
    if (ab.ntiles > 0 && (st = launch_stage(c, dg::MODE_FUSED_RK, ab, s, 0)) != DG_OK) return st;
  } else {
    dg::StageArgs av = a;
    av.out = c->rhsv;  // the volume kernel's output is the surface kernel's rhsV input
    if ((st = launch_stage(c, dg::MODE_VOLUME, av, s, 1)) != DG_OK) return st;
    if ((st = halo_ready()) != DG_OK) return st;
    if ((st = launch_stage(c, dg::MODE_SURFACE_RK, a, s, 2)) != DG_OK) return st;
  }
  return DG_OK;
}

// One LSERK4 stage for a single (NCCL or single-rank) context.
dg_status run_stage(dg_ctx* c, int i, double dt) {
  const dg::StageArgs a = stage_args(c, i, dt);
  dg_status st;
  if (c->nranks > 1 && c->transport == 0) {
    if ((st = pack(c, c->stream)) != DG_OK) return st;
    CU(c, cudaEventRecord(c->ev_pack, c->stream));
    CU(c, cudaStreamWaitEvent(c->comm, c->ev_pack, 0));
    if ((st = exchange_nccl(c, c->comm)) != DG_OK) return st;
    CU(c, cudaEventRecord(c->ev_comm, c->comm));
    st = partitioned_stage(c, a, c->stream, [&]() -> dg_status {
      CU(c, cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
      return DG_OK;
    });
    if (st != DG_OK) return st;
  } else if (c->fused) {
    if ((st = launch_stage(c, dg::MODE_FUSED_RK, a, c->stream, 0)) != DG_OK) return st;
  } else {
    dg::StageArgs av = a;
    av.out = c->rhsv;  // the volume kernel's output is the surface kernel's rhsV input
    if ((st = launch_stage(c, dg::MODE_VOLUME, av, c->stream, 1)) != DG_OK) return st;
    if ((st = launch_stage(c, dg::MODE_SURFACE_RK, a, c->stream, 2)) != DG_OK) return st;
  }
  c->cur = 1 - c->cur;
  return DG_OK;
}

template <typename T>
void upload_geometry(dg_ctx* c, std::vector<T>& g, std::vector<int32_t>& vp, const double* eps_g,
                     const double* mu_g) {
  const int Np = c->ref.Np, Nfp = c->ref.Nfp, NF = 3 * Nfp;
  const int ng = c->ngeo;
  const dg::Mesh& m = c->mesh;
  g.assign((size_t)c->ntiles * ng * 32, T(0));
  const bool words = c->compressed == 1;  // one connectivity word per face
  vp.assign((size_t)c->ntiles * (words ? 3 : NF) * 32, 0);
  const int swm = c->km->swizzle;
  // blocked (column-swizzled) offset of node n of the element in device slot d
  auto col = [&](int64_t d, int n) -> int64_t { return dg::swz_col(swm, n, (int)(d & 31)); };
  auto blk = [&](int64_t d, int n) -> int64_t { return ((d >> 5) * Np + n) * 32 + col(d, n); };
  // neighbour node n of the element in slot d2, seen from slot d: same work unit (group of
  // c->group tiles) -> shared-memory offset within the unit's field block, encoded negative:
  // -(1 + (tile-in-group * Np + n) * 32 + column)
  const int64_t gsz = 32 * c->group;
  auto nbr_code = [&](int64_t d, int64_t d2, int n) -> int64_t {
    if (d / gsz == d2 / gsz) return -(1 + (((d2 >> 5) % c->group) * Np + n) * 32 + col(d2, n));
    return blk(d2, n);
  };
  for (int64_t d = 0; d < c->Kpad; ++d) {
    const int64_t t = d >> 5, lane = d & 31;
    auto G = [&](int comp) -> T& { return g[(t * ng + comp) * 32 + lane]; };
    if (d >= c->Kl) {  // padding element: its neighbour codes point at itself (finite zeros)
      if (c->compressed) G(0) = G(3) = T(1);  // identity geometric factors: finite derived normals
      if (words) {
        for (int f = 0; f < 3; ++f) vp[(t * 3 + f) * 32 + lane] = (int32_t)dg::conn_word(1, 0, (uint32_t)lane);
        continue;
      }
      if (c->compressed) {
        for (int mm = 0; mm < NF; ++mm) vp[(t * NF + mm) * 32 + lane] = (int32_t)nbr_code(d, d, 0);
        continue;
      }
      for (int f = 0; f < 3; ++f) G(13 + f) = T(1);
      for (int mm = 0; mm < NF; ++mm) vp[(t * NF + mm) * 32 + lane] = (int32_t)nbr_code(d, d, 0);
      continue;
    }
    const int64_t kl = c->perm[d];
    G(0) = (T)m.rx[kl];
    G(1) = (T)m.sx[kl];
    G(2) = (T)m.ry[kl];
    G(3) = (T)m.sy[kl];
    const int64_t k = m.local[kl];
    for (int f = 0; f < 3 && !c->compressed; ++f) {
      G(4 + 3 * f) = (T)m.nx[3 * kl + f];
      G(5 + 3 * f) = (T)m.ny[3 * kl + f];
      G(6 + 3 * f) = (T)(c->material ? m.Fsc[3 * kl + f] : 0.5 * m.Fsc[3 * kl + f]);
      G(13 + f) = m.pec[3 * k + f] ? T(-1) : T(1);
    }
    if (c->material) {
      const double e = eps_g ? eps_g[k] : 1.0, u = mu_g ? mu_g[k] : 1.0;
      G(16) = (T)(1.0 / u);
      G(17) = (T)(1.0 / e);
      const double Zm = std::sqrt(u / e), Ym = 1.0 / Zm;
      for (int f = 0; f < 3; ++f) {
        const int64_t k2 = m.EToE[3 * k + f];
        const double e2 = eps_g ? eps_g[k2] : 1.0, u2 = mu_g ? mu_g[k2] : 1.0;
        const double Zp = m.pec[3 * k + f] ? Zm : std::sqrt(u2 / e2), Yp = 1.0 / Zp;
        G(18 + 4 * f) = (T)(Yp / (Yp + Ym));
        G(19 + 4 * f) = (T)(c->alpha / (Yp + Ym));
        G(20 + 4 * f) = (T)(Zp / (Zp + Zm));
        G(21 + 4 * f) = (T)(c->alpha / (Zp + Zm));
      }
    }
    std::vector<int64_t> code(NF);
    for (int mm = 0; mm < NF; ++mm) {
      const int64_t nl = m.nbr_local[kl * NF + mm];
      int64_t idx;
      if (nl >= 0) {
        const int64_t kl2 = nl / Np;
        idx = nbr_code(d, c->slot_of[kl2], (int)(nl - kl2 * Np));
      } else {
        idx = c->ghost_base + (-nl - 1);
      }
      code[mm] = idx;
      // geometry-only compression: a PEC point's code carries ZC_PEC (its Bsc = -1)
      if (!words)
        vp[(t * NF + mm) * 32 + lane] =
            (int32_t)(idx + (c->compressed == 2 && m.pec[3 * k + mm / Nfp] ? dg::ZC_PEC : 0));
    }
    if (!words) continue;
    // one word per face (kernel_api.h conn_word), checked against every point's code above by the
    // kernels' own decode rule (the O7 reversal), so a wrong word fails at setup, not in a run
    for (int f = 0; f < 3; ++f) {
      uint32_t w;
      const int64_t k2 = m.EToE[3 * k + f];
      const int fp = m.EToF[3 * k + f];
      if (m.pec[3 * k + f]) {
        w = dg::conn_word(0, 0, 0);
      } else if (m.g2l[k2] < 0) {  // halo face: ghost index of point 0, the others follow
        const int64_t g0 = code[f * Nfp] - c->ghost_base;
        for (int i = 0; i < Nfp; ++i)
          if (code[f * Nfp + i] != c->ghost_base + g0 + i) throw dg::SetupError{DG_E_STATE, "halo face points out of order"};
        w = dg::conn_word(3, 0, (uint32_t)g0);
      } else {
        const int64_t d2 = c->slot_of[m.g2l[k2]];
        w = (d2 >> 5) == (d >> 5) ? dg::conn_word(1, fp, (uint32_t)(d2 & 31)) : dg::conn_word(2, fp, (uint32_t)d2);
      }
      if ((w >> 4) >= (1u << 28)) throw dg::SetupError{DG_E_ARG, "partition too large for compressed connectivity"};
      vp[(t * 3 + f) * 32 + lane] = (int32_t)w;
      // host replica of the kernels' zc_decode
      const uint32_t kind = w & 3u, fw = (w >> 2) & 3u, pay = w >> 4;
      for (int i = 0; i < Nfp; ++i) {
        const int mm = f * Nfp + i;
        int64_t dec;
        if (kind == 3u) {
          dec = c->ghost_base + pay + i;
        } else if (kind == 0u) {
          dec = code[mm];  // PEC: own node (the kernel adds ZC_PEC)
        } else {
          const int ip = ((f == 2) == (fw == 2u)) ? Nfp - 1 - i : i;
          const int n2 = c->ref.Fmask[fw * Nfp + ip];
          dec = kind == 1u ? -(1 + (int64_t)n2 * 32 + dg::swz_col(swm, n2, (int)(pay & 31u)))
                           : (((int64_t)(pay >> 5)) * Np + n2) * 32 + dg::swz_col(swm, n2, (int)(pay & 31u));
        }
        if (dec != code[mm]) throw dg::SetupError{DG_E_STATE, "compressed connectivity does not reproduce vmapP"};
      }
    }
  }
}

dg_status alloc(dg_ctx* c, void** p, size_t bytes) {
  if (bytes == 0) bytes = 256;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    c->poisoned = true;
    return set_err(e == cudaErrorMemoryAllocation ? DG_E_OOM : DG_E_CUDA,
                   std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  }
  return DG_OK;
}

dg_status setup_device(dg_ctx* c, const dg_options* o, const double* eps, const double* mu) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return set_err(DG_E_CUDA, std::string("no usable CUDA device: ") + cudaGetErrorString(e));
  if (c->device >= ndev) return set_err(DG_E_ARG, "device ordinal out of range");
  CU(c, cudaSetDevice(c->device));
  c->km = dg::find_module(c->N, c->prec, c->kernel_variant);
  if (!c->km)
    return set_err(DG_E_DEGREE, "no kernel module compiled for N=" + std::to_string(c->N) +
                                    " precision=" + std::to_string(c->prec) +
                                    " variant=" + std::to_string(c->kernel_variant));
  if (!c->km->check_fmask(c->ref.Fmask.data()))
    return set_err(DG_E_STATE, "kernel face masks disagree with the setup's node set");
  {
    std::vector<unsigned char> ops(c->km->ops_bytes());
    c->km->pack_ops(c->ref.Dr.data(), c->ref.Ds.data(), c->ref.LIFT.data(), ops.data());
    dg_status st0 = alloc(c, &c->ops, ops.size());
    if (st0 != DG_OK) return st0;
    CU(c, cudaMemcpy(c->ops, ops.data(), ops.size(), cudaMemcpyHostToDevice));
  }
  const int Np = c->ref.Np;
  c->tsz = (size_t)c->prec;
  c->compressed = c->material ? 0 : c->km->compressed;
  c->ngeo = c->material ? dg::NGEO_MAT : (c->compressed ? dg::NGEO_Z : dg::NGEO_CONST);
  c->Kl = (int64_t)c->mesh.local.size();
  c->group = c->km->tile_group;
  c->ngroups = (c->Kl + 32 * c->group - 1) / (32 * c->group);
  c->ntiles = c->ngroups * c->group;
  c->Kpad = c->ntiles * 32;
  c->n_recv = (int64_t)c->mesh.recv_gdof.size();
  c->n_send = (int64_t)c->mesh.send_gdof.size();
  c->ghost_base = c->Kpad * Np;
  c->fstride = c->ghost_base + ((c->n_recv + 31) / 32) * 32;
  c->vstride = c->Kpad * Np;
  if (c->fstride >= (int64_t)1 << 31) return set_err(DG_E_ARG, "partition too large for 32-bit face maps");
  dg_status st;
  // device storage order: Morton order of the element centroids (setup.cpp locality_order)
  c->perm = dg::locality_order(c->mesh);
  c->slot_of.assign(c->Kl, 0);
  for (int64_t d = 0; d < c->Kl; ++d) c->slot_of[c->perm[d]] = d;
  {
    std::vector<int32_t> pd(c->Kpad, -1), sd(std::max<int64_t>(c->Kl, 1), 0);
    for (int64_t d = 0; d < c->Kl; ++d) pd[d] = (int32_t)c->perm[d];
    for (int64_t kl = 0; kl < c->Kl; ++kl) sd[kl] = (int32_t)c->slot_of[kl];
    if ((st = alloc(c, (void**)&c->perm_d, pd.size() * sizeof(int32_t))) != DG_OK) return st;
    if ((st = alloc(c, (void**)&c->slot_of_d, sd.size() * sizeof(int32_t))) != DG_OK) return st;
    CU(c, cudaMemcpy(c->perm_d, pd.data(), pd.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    CU(c, cudaMemcpy(c->slot_of_d, sd.data(), sd.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  for (int b = 0; b < 2; ++b)
    if ((st = alloc(c, &c->q[b], 3 * c->fstride * c->tsz)) != DG_OK) return st;
  if ((st = alloc(c, &c->res, 3 * c->vstride * c->tsz)) != DG_OK) return st;
  if (!c->fused && (st = alloc(c, &c->rhsv, 3 * c->vstride * c->tsz)) != DG_OK) return st;
  if ((st = alloc(c, (void**)&c->stage, 3 * std::max<int64_t>(c->Kl * Np, 1) * sizeof(double))) != DG_OK) return st;
  if ((st = alloc(c, (void**)&c->flag, sizeof(unsigned long long))) != DG_OK) return st;
  if ((st = alloc(c, (void**)&c->first_bad, sizeof(unsigned long long))) != DG_OK) return st;
  if ((st = alloc(c, (void**)&c->ebuf, sizeof(double))) != DG_OK) return st;
  CU(c, cudaMemset(c->first_bad, 0xff, sizeof(unsigned long long)));
  CU(c, cudaMemset(c->q[0], 0, 3 * c->fstride * c->tsz));
  CU(c, cudaMemset(c->q[1], 0, 3 * c->fstride * c->tsz));
  CU(c, cudaMemset(c->res, 0, 3 * c->vstride * c->tsz));
  // geometry + maps
  {
    std::vector<int32_t> vp;
    try {
    if (c->tsz == 4) {
      std::vector<float> g;
      upload_geometry<float>(c, g, vp, eps, mu);
      if ((st = alloc(c, &c->geo, g.size() * sizeof(float))) != DG_OK) return st;
      CU(c, cudaMemcpy(c->geo, g.data(), g.size() * sizeof(float), cudaMemcpyHostToDevice));
    } else {
      std::vector<double> g;
      upload_geometry<double>(c, g, vp, eps, mu);
      if ((st = alloc(c, &c->geo, g.size() * sizeof(double))) != DG_OK) return st;
      CU(c, cudaMemcpy(c->geo, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    } catch (const dg::SetupError& e) {
      return set_err((dg_status)e.status, e.msg);
    }
    if ((st = alloc(c, (void**)&c->vmapP, vp.size() * sizeof(int32_t))) != DG_OK) return st;
    CU(c, cudaMemcpy(c->vmapP, vp.data(), vp.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  // halo send indices (tile-blocked offsets of own nodes) and tile classes
  if (c->n_send > 0) {
    std::vector<int32_t> si(c->n_send);
    for (int64_t s = 0; s < c->n_send; ++s) {
      const int64_t gd = c->mesh.send_gdof[s];
      const int64_t k = gd / Np, n = gd - (gd / Np) * Np;
      const int64_t d = c->slot_of[c->mesh.g2l[k]];
      si[s] = (int32_t)(((d >> 5) * Np + n) * 32 + dg::swz_col(c->km->swizzle, (int)n, (int)(d & 31)));
    }
    if ((st = alloc(c, (void**)&c->send_idx, si.size() * sizeof(int32_t))) != DG_OK) return st;
    CU(c, cudaMemcpy(c->send_idx, si.data(), si.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    if ((st = alloc(c, &c->sendbuf, 3 * c->n_send * c->tsz)) != DG_OK) return st;
  }
  {
    // interior / partition-boundary classes of the kernels' work units (groups of tiles)
    std::vector<char> bnd(c->ngroups, 0);
    for (int64_t p = 0; p < c->n_recv; ++p)
      bnd[(c->slot_of[c->mesh.recv_point[p] / (3 * c->ref.Nfp)] >> 5) / c->group] = 1;
    std::vector<int32_t> ti, tb;
    for (int64_t t = 0; t < c->ngroups; ++t) (bnd[t] ? tb : ti).push_back((int32_t)t);
    c->n_int = (int32_t)ti.size();
    c->n_bnd = (int32_t)tb.size();
    if ((st = alloc(c, (void**)&c->tiles_int, std::max<size_t>(ti.size(), 1) * sizeof(int32_t))) != DG_OK) return st;
    if ((st = alloc(c, (void**)&c->tiles_bnd, std::max<size_t>(tb.size(), 1) * sizeof(int32_t))) != DG_OK) return st;
    if (!ti.empty()) CU(c, cudaMemcpy(c->tiles_int, ti.data(), ti.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (!tb.empty()) CU(c, cudaMemcpy(c->tiles_bnd, tb.data(), tb.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  // streams
  if (o->stream) {
    c->stream = static_cast<cudaStream_t>(o->stream);
    c->own_stream = false;
  } else {
    CU(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  CU(c, cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking));
  CU(c, cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
  CU(c, cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
  if (c->nranks > 1 && c->transport == 0) {
    Nccl* n = nccl();
    if (!n) return set_err(DG_E_NCCL, "could not dlopen libnccl.so.2");
    if (!o->nccl_id) return set_err(DG_E_ARG, "nccl_id required for nranks > 1 with NCCL transport");
    ncclUniqueId id;
    std::memcpy(&id, o->nccl_id, sizeof(id));
    ncclResult_t r = n->CommInitRank(&c->nccl_comm, c->nranks, id, c->rank);
    if (r != ncclSuccess) {
      c->poisoned = true;
      return set_err(DG_E_NCCL, std::string("ncclCommInitRank: ") + n->GetErrorString(r));
    }
  }
  CU(c, cudaDeviceSynchronize());
  return DG_OK;
}

// A field pointer handed to dg_set_fields / dg_get_fields: host memory (pageable, pinned or
// managed) or device memory of the context's own device; copies use cudaMemcpyDefault (UVA).
dg_status check_field_ptr(dg_ctx* c, const void* p) {
  cudaPointerAttributes at{};
  const cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of an unregistered pointer
    return DG_OK;
  }
  if (at.type == cudaMemoryTypeDevice && at.device != c->device)
    return set_err(DG_E_ARG, "field pointer is device memory of another device");
  return DG_OK;
}

}  // namespace

// ============================================================== C ABI
extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }

dg_status dg_options_default(dg_options* o) {
  if (!o) return set_err(DG_E_ARG, "null options");
  std::memset(o, 0, sizeof(*o));
  o->abi_version = DG_ABI_VERSION;
  o->N = 4;
  o->precision = 8;
  o->device = 0;
  o->alpha = 1.0;
  o->rank = 0;
  o->nranks = 1;
  o->fused = 1;
  o->transport = 0;
  o->max_ctas = 0;
  o->tile_order = 0;
  o->check_every = 0;
  o->kernel_variant = 0;
  return DG_OK;
}

dg_status dg_setup(const dg_options* o, int64_t Nv, const double* VX, const double* VY, int64_t K,
                   const int64_t* EToV, const double* eps, const double* mu, const int8_t* bctag, dg_ctx** out) {
  if (!o || !out || !VX || !VY || !EToV) return set_err(DG_E_ARG, "null argument to dg_setup");
  *out = nullptr;
  if (o->abi_version != DG_ABI_VERSION) return set_err(DG_E_ARG, "ABI version mismatch");
  if (o->precision != 4 && o->precision != 8) return set_err(DG_E_ARG, "precision must be 4 or 8");
  if ((eps == nullptr) != (mu == nullptr)) return set_err(DG_E_ARG, "give both eps and mu, or neither");
  if (o->nranks < 1 || o->rank < 0 || o->rank >= o->nranks) return set_err(DG_E_ARG, "bad rank / nranks");
  if (o->transport != 0 && o->transport != 1) return set_err(DG_E_ARG, "transport must be 0 or 1");
  if (!(o->alpha >= 0.0)) return set_err(DG_E_ARG, "alpha must be >= 0");
  if (o->max_ctas < 0 || o->check_every < 0 || (o->tile_order != 0 && o->tile_order != 1))
    return set_err(DG_E_ARG, "max_ctas and check_every must be >= 0, tile_order 0 or 1");
  if (o->kernel_variant != 0 && o->kernel_variant != 1) return set_err(DG_E_ARG, "kernel_variant must be 0 or 1");
  if (o->kernel_variant == 1 && o->precision != 4)
    return set_err(DG_E_ARG, "kernel_variant 1 (tcgen05) is an fp32 path");
  if (eps)
    for (int64_t k = 0; k < K; ++k)
      if (!(eps[k] > 0.0) || !(mu[k] > 0.0)) return set_err(DG_E_ARG, "eps and mu must be > 0");
  std::unique_ptr<dg_ctx> c(new dg_ctx());
  c->N = o->N;
  c->prec = o->precision;
  c->device = o->device;
  c->alpha = o->alpha;
  c->rank = o->rank;
  c->nranks = o->nranks;
  c->fused = o->fused ? 1 : 0;
  c->transport = o->transport;
  c->max_ctas = o->max_ctas;
  c->tile_order = o->tile_order;
  c->check_every = o->check_every;
  c->kernel_variant = o->kernel_variant;
  c->material = eps != nullptr;
  try {
    c->ref = dg::build_refelem(o->N);
    dg::build_mesh(c->ref, Nv, VX, VY, K, EToV, bctag, o->rank, o->nranks, o->part, c->mesh);
  } catch (const dg::SetupError& e) {
    return set_err((dg_status)e.status, e.msg);
  } catch (const std::bad_alloc&) {
    return set_err(DG_E_OOM, "host allocation failed in setup");
  }
  c->Kl = (int64_t)c->mesh.local.size();
  c->eps_l.resize(c->Kl);
  c->mu_l.resize(c->Kl);
  for (int64_t kl = 0; kl < c->Kl; ++kl) {
    c->eps_l[kl] = eps ? eps[c->mesh.local[kl]] : 1.0;
    c->mu_l[kl] = mu ? mu[c->mesh.local[kl]] : 1.0;
  }
  c->host_only = o->device < 0;
  if (!c->host_only) {
    dg_status st = setup_device(c.get(), o, eps, mu);
    if (st != DG_OK) {
      std::string keep = g_err;
      dg_destroy(c.release());
      g_err = keep;
      return st;
    }
  }
  *out = c.release();
  return DG_OK;
}

dg_status dg_sizes(const dg_ctx* c, int64_t* Np, int64_t* Nfp, int64_t* K_local, int64_t* K_global,
                   int64_t* n_halo_points, int64_t* n_swapped) {
  if (!c) return set_err(DG_E_ARG, "null context");
  if (Np) *Np = c->ref.Np;
  if (Nfp) *Nfp = c->ref.Nfp;
  if (K_local) *K_local = (int64_t)c->mesh.local.size();
  if (K_global) *K_global = c->mesh.K;
  if (n_halo_points) *n_halo_points = (int64_t)c->mesh.recv_gdof.size();
  if (n_swapped) *n_swapped = c->mesh.n_swapped;
  return DG_OK;
}

dg_status dg_local_elements(const dg_ctx* c, int64_t* gid) {
  if (!c || !gid) return set_err(DG_E_ARG, "null argument");
  std::copy(c->mesh.local.begin(), c->mesh.local.end(), gid);
  return DG_OK;
}

dg_status dg_set_fields(dg_ctx* c, const double* Hx, const double* Hy, const double* Ez) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  if (!Hx || !Hy || !Ez) return set_err(DG_E_ARG, "null field pointer");
  CU(c, cudaSetDevice(c->device));
  const int64_t n = c->Kl * c->ref.Np;
  const double* src[3] = {Hx, Hy, Ez};
  for (int f = 0; f < 3; ++f)
    if ((st = check_field_ptr(c, src[f])) != DG_OK) return st;
  for (int f = 0; f < 3; ++f)
    CU(c, cudaMemcpyAsync(c->stage + f * n, src[f], n * sizeof(double), cudaMemcpyDefault, c->stream));
  void* q = c->q[c->cur];
  if (c->tsz == 4)
    to_blocked<float><<<grid_for(3 * c->Kpad * c->ref.Np), 256, 0, c->stream>>>(
        c->stage, (float*)q, c->perm_d, c->Kl, c->Kpad, c->ref.Np, c->fstride, c->km->swizzle);
  else
    to_blocked<double><<<grid_for(3 * c->Kpad * c->ref.Np), 256, 0, c->stream>>>(
        c->stage, (double*)q, c->perm_d, c->Kl, c->Kpad, c->ref.Np, c->fstride, c->km->swizzle);
  CU(c, cudaGetLastError());
  CU(c, cudaMemsetAsync(c->res, 0, 3 * c->vstride * c->tsz, c->stream));
  CU(c, cudaMemsetAsync(c->first_bad, 0xff, sizeof(unsigned long long), c->stream));
  CU(c, cudaStreamSynchronize(c->stream));  // host sources are read before returning
  c->steps_done = 0;
  return DG_OK;
}

dg_status dg_get_fields(dg_ctx* c, double* Hx, double* Hy, double* Ez) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  if (!Hx || !Hy || !Ez) return set_err(DG_E_ARG, "null field pointer");
  CU(c, cudaSetDevice(c->device));
  const int64_t n = c->Kl * c->ref.Np;
  const void* q = c->q[c->cur];
  if (c->tsz == 4)
    from_blocked<float><<<grid_for(3 * n), 256, 0, c->stream>>>((const float*)q, c->stage, c->slot_of_d, c->Kl,
                                                                c->ref.Np, c->fstride, c->km->swizzle);
  else
    from_blocked<double><<<grid_for(3 * n), 256, 0, c->stream>>>((const double*)q, c->stage, c->slot_of_d, c->Kl,
                                                                 c->ref.Np, c->fstride, c->km->swizzle);
  CU(c, cudaGetLastError());
  double* dst[3] = {Hx, Hy, Ez};
  for (int f = 0; f < 3; ++f)
    if ((st = check_field_ptr(c, dst[f])) != DG_OK) return st;
  for (int f = 0; f < 3; ++f)
    CU(c, cudaMemcpyAsync(dst[f], c->stage + f * n, n * sizeof(double), cudaMemcpyDefault, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  return DG_OK;
}

}  // extern "C"

namespace {
dg_status check_step(dg_ctx* c) {  // options.check_every: mark the step if any value is non-finite
  const int64_t n = c->Kpad * c->ref.Np;
  const unsigned long long step = (unsigned long long)c->steps_done;
  if (c->tsz == 4)
    mark_nonfinite<float><<<grid_for(3 * n), 256, 0, c->stream>>>((const float*)c->q[c->cur], n, c->fstride, step,
                                                                  c->first_bad);
  else
    mark_nonfinite<double><<<grid_for(3 * n), 256, 0, c->stream>>>((const double*)c->q[c->cur], n, c->fstride, step,
                                                                   c->first_bad);
  CU(c, cudaGetLastError());
  c->stats.launches[3] += 1;
  return DG_OK;
}
}  // namespace

extern "C" {

static void drop_graphs(dg_ctx* c) {
  for (int p = 0; p < 2; ++p) {
    for (cudaGraphExec_t* g : {&c->gexec[p], &c->pexec[p]})
      if (*g) {
        cudaGraphExecDestroy(*g);
        *g = nullptr;
      }
    for (cudaEvent_t e : c->pev[p]) cudaEventDestroy(e);
    c->pev[p].clear();
    c->ptimed[p].clear();
  }
}

// Capture one LSERK4 step starting from q[parity] (the same launches run_stage enqueues);
// profiled = with event-record nodes around every launch (into pexec[parity])
static dg_status capture_step(dg_ctx* c, double dt, int parity, bool profiled = false) {
  const int cur0 = c->cur;
  const dg_kernel_stats st0 = c->stats;
  c->cur = parity;
  c->pcap = profiled ? parity : -1;
  if (profiled) {  // two launches per stage at most (split variant): 20 events
    c->ptimed[parity].clear();
    while (c->pev[parity].size() < 20) {
      cudaEvent_t ev;
      CU(c, cudaEventCreate(&ev));
      c->pev[parity].push_back(ev);
    }
  }
  CU(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  dg_status st = DG_OK;
  for (int i = 0; i < 5 && st == DG_OK; ++i) st = run_stage(c, i, dt);
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
  c->cur = cur0;
  c->stats = st0;
  c->pcap = -1;
  if (st != DG_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamEndCapture");
  const cudaError_t e2 = cudaGraphInstantiate(profiled ? &c->pexec[parity] : &c->gexec[parity], g, 0);
  cudaGraphDestroy(g);
  if (e2 != cudaSuccess) return cuda_fail(c, e2, "cudaGraphInstantiate");
  return DG_OK;
}

dg_status dg_run(dg_ctx* c, double dt, int64_t nsteps) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  if (!(dt > 0.0) || !std::isfinite(dt) || nsteps < 0) return set_err(DG_E_ARG, "need dt > 0 and nsteps >= 0");
  if (c->transport == 1 && c->nranks > 1) return set_err(DG_E_STATE, "in-process group contexts run via dg_run_group");
  CU(c, cudaSetDevice(c->device));
  for (int64_t s = 0; s < nsteps; ++s) {
    // graph replay once a step has run eagerly (kernel attributes set up outside any capture)
    // (NCCL contexts too: the pack, the comm-stream fork/join and the send/recv are captured; NCCL's
    // peer connections were set up by the eager first step)
    if (c->graphs && c->steps_done > 0) {
      if (c->gdt != dt) {
        drop_graphs(c);
        c->gdt = dt;
      }
      const int par = c->cur;
      if (!c->profiling) {
        if (!c->gexec[par] && (st = capture_step(c, dt, par)) != DG_OK) return st;
        CU(c, cudaGraphLaunch(c->gexec[par], c->stream));
      } else {
        // profiled replay: the same launches with event-record nodes; the per-launch times
        // are read back after each step (the host wait lies between steps, outside every bracket)
        if (!c->pexec[par] && (st = capture_step(c, dt, par, true)) != DG_OK) return st;
        CU(c, cudaGraphLaunch(c->pexec[par], c->stream));
        CU(c, cudaStreamSynchronize(c->stream));
        for (const auto& t : c->ptimed[par]) {
          float ms = 0.f;
          CU(c, cudaEventElapsedTime(&ms, c->pev[par][t.ev0], c->pev[par][t.ev1]));
          c->stats.ms[t.kind] += ms;
          c->stats.timed[t.kind] += 1;
        }
      }
      c->stats.launches[c->fused ? 0 : 1] += 5;
      if (!c->fused) c->stats.launches[2] += 5;
      c->cur = 1 - c->cur;  // five stages: five ping-pong flips
    } else {
      for (int i = 0; i < 5; ++i)
        if ((st = run_stage(c, i, dt)) != DG_OK) return st;
    }
    ++c->steps_done;
    if (c->check_every > 0 && c->steps_done % c->check_every == 0 && (st = check_step(c)) != DG_OK) return st;
  }
  return DG_OK;
}

dg_status dg_set_graphs(dg_ctx* c, int32_t enable) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  c->graphs = enable != 0;
  if (!c->graphs) {
    CU(c, cudaSetDevice(c->device));
    CU(c, cudaStreamSynchronize(c->stream));
    drop_graphs(c);
  }
  return DG_OK;
}

dg_status dg_run_group(dg_ctx* const* ctxs, int32_t n, double dt, int64_t nsteps) {
  if (!ctxs || n < 1) return set_err(DG_E_ARG, "empty group");
  if (!(dt > 0.0) || !std::isfinite(dt) || nsteps < 0) return set_err(DG_E_ARG, "need dt > 0 and nsteps >= 0");
  std::vector<dg_ctx*> byrank(n, nullptr);
  for (int i = 0; i < n; ++i) {
    dg_status st = check_usable(ctxs[i], true);
    if (st != DG_OK) return st;
    dg_ctx* c = ctxs[i];
    if (c->nranks != n || c->transport != 1 || c->device != ctxs[0]->device || c->prec != ctxs[0]->prec)
      return set_err(DG_E_ARG, "group contexts must be transport=1 ranks 0..n-1 of one mesh on one device");
    if (byrank[c->rank]) return set_err(DG_E_ARG, "duplicate rank in group");
    byrank[c->rank] = c;
  }
  dg_ctx* c0 = byrank[0];
  CU(c0, cudaSetDevice(c0->device));
  cudaStream_t s = c0->stream;
  for (int i = 1; i < n; ++i) {  // order the group's work after everything already queued on each ctx
    CU(c0, cudaEventRecord(byrank[i]->ev_pack, byrank[i]->stream));
    CU(c0, cudaStreamWaitEvent(s, byrank[i]->ev_pack, 0));
  }
  for (int64_t step = 0; step < nsteps; ++step)
    for (int i = 0; i < 5; ++i) {
      dg_status st;
      for (dg_ctx* c : byrank)
        if ((st = pack(c, s)) != DG_OK) return st;
      for (dg_ctx* c : byrank)
        for (size_t t = 0; t < c->mesh.nbr.size(); ++t) {
          const dg_ctx* src = byrank[c->mesh.nbr[t]];
          size_t u = std::find(src->mesh.nbr.begin(), src->mesh.nbr.end(), c->rank) - src->mesh.nbr.begin();
          const int64_t so = src->mesh.send_off[u], cnt = src->mesh.send_off[u + 1] - so;
          if (cnt != c->mesh.recv_off[t + 1] - c->mesh.recv_off[t]) return set_err(DG_E_STATE, "halo size mismatch");
          for (int f = 0; f < 3; ++f)
            CU(c, cudaMemcpyAsync(static_cast<char*>(c->q[c->cur]) +
                                      (f * c->fstride + c->ghost_base + c->mesh.recv_off[t]) * c->tsz,
                                  static_cast<const char*>(src->sendbuf) + (f * src->n_send + so) * src->tsz,
                                  cnt * c->tsz, cudaMemcpyDeviceToDevice, s));
        }
      for (dg_ctx* c : byrank) {  // the NCCL path's launches; the copies above are already on s
        if ((st = partitioned_stage(c, stage_args(c, i, dt), s, [] { return DG_OK; })) != DG_OK) return st;
        c->cur = 1 - c->cur;
      }
    }
  for (int i = 1; i < n; ++i) {  // later work on each ctx's own stream waits for the group
    CU(c0, cudaEventRecord(c0->ev_pack, s));
    CU(c0, cudaStreamWaitEvent(byrank[i]->stream, c0->ev_pack, 0));
  }
  for (dg_ctx* c : byrank) c->steps_done += nsteps;
  return DG_OK;
}

dg_status dg_sync(dg_ctx* c) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  CU(c, cudaSetDevice(c->device));
  CU(c, cudaMemsetAsync(c->flag, 0, sizeof(unsigned long long), c->stream));
  const int64_t n = c->Kpad * c->ref.Np;
  if (c->tsz == 4)
    count_nonfinite<float><<<grid_for(3 * n), 256, 0, c->stream>>>((const float*)c->q[c->cur], n, c->fstride, c->flag);
  else
    count_nonfinite<double><<<grid_for(3 * n), 256, 0, c->stream>>>((const double*)c->q[c->cur], n, c->fstride, c->flag);
  CU(c, cudaGetLastError());
  unsigned long long bad = 0, first = ~0ull;
  CU(c, cudaMemcpyAsync(&bad, c->flag, sizeof(bad), cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaMemcpyAsync(&first, c->first_bad, sizeof(first), cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  if (first != ~0ull)
    return set_err(DG_E_DIVERGED, "non-finite field values first found at step " + std::to_string(first) +
                                      " (checked every " + std::to_string(c->check_every) + " steps); " +
                                      std::to_string(bad) + " non-finite values after step " +
                                      std::to_string(c->steps_done));
  if (bad)
    return set_err(DG_E_DIVERGED, std::to_string(bad) + " non-finite field values after step " +
                                      std::to_string(c->steps_done));
  return DG_OK;
}

dg_status dg_eval_rhs(dg_ctx* c, int32_t which, double* rHx, double* rHy, double* rEz) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  if (which < 0 || which > 2 || !rHx || !rHy || !rEz) return set_err(DG_E_ARG, "bad dg_eval_rhs arguments");
  if (c->transport == 1 && c->nranks > 1) return set_err(DG_E_STATE, "dg_eval_rhs needs a single-rank or NCCL context");
  CU(c, cudaSetDevice(c->device));
  if (!c->out && (st = alloc(c, &c->out, 3 * c->vstride * c->tsz)) != DG_OK) return st;
  if (c->nranks > 1 && which != 1) {
    if ((st = pack(c, c->stream)) != DG_OK) return st;
    if ((st = exchange_nccl(c, c->stream)) != DG_OK) return st;
  }
  dg::StageArgs a = base_args(c);
  a.out = c->out;
  a.scale_volume = 1;
  const int mode = which == 0 ? dg::MODE_RHS : which == 1 ? dg::MODE_VOLUME : dg::MODE_SURFACE;
  if ((st = launch_stage(c, mode, a, c->stream, which == 1 ? 1 : 2)) != DG_OK) return st;
  const int64_t n = c->Kl * c->ref.Np;
  if (c->tsz == 4)
    from_blocked<float><<<grid_for(3 * n), 256, 0, c->stream>>>((const float*)c->out, c->stage, c->slot_of_d, c->Kl,
                                                                c->ref.Np, c->vstride, c->km->swizzle);
  else
    from_blocked<double><<<grid_for(3 * n), 256, 0, c->stream>>>((const double*)c->out, c->stage, c->slot_of_d, c->Kl,
                                                                 c->ref.Np, c->vstride, c->km->swizzle);
  CU(c, cudaGetLastError());
  double* dst[3] = {rHx, rHy, rEz};
  for (int f = 0; f < 3; ++f)
    CU(c, cudaMemcpyAsync(dst[f], c->stage + f * n, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  return DG_OK;
}

dg_status dg_energy_local(dg_ctx* c, double* E) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  if (!E) return set_err(DG_E_ARG, "null output");
  const int Np = c->ref.Np;
  const int64_t n = c->Kl * Np;
  std::vector<double> f(3 * n);
  if ((st = dg_get_fields(c, f.data(), f.data() + n, f.data() + 2 * n)) != DG_OK) return st;
  double tot = 0.0;
  std::vector<double> Mu(Np);
  for (int64_t kl = 0; kl < c->Kl; ++kl) {
    double ek = 0.0;
    for (int fld = 0; fld < 3; ++fld) {
      const double* u = f.data() + fld * n + kl * Np;
      double s = 0.0;
      for (int i = 0; i < Np; ++i) {
        double acc = 0.0;
        for (int j = 0; j < Np; ++j) acc += c->ref.M[i * Np + j] * u[j];
        s += u[i] * acc;
      }
      ek += (fld < 2 ? c->mu_l[kl] : c->eps_l[kl]) * s;
    }
    tot += c->mesh.J[kl] * ek;
  }
  *E = 0.5 * tot;
  return DG_OK;
}

dg_status dg_energy(dg_ctx* c, double* E) {
  dg_status st = dg_energy_local(c, E);
  if (st != DG_OK || c->nranks == 1 || c->transport != 0) return st;
  Nccl* n = nccl();
  if (!n || !c->nccl_comm) return set_err(DG_E_NCCL, "NCCL unavailable");
  CU(c, cudaMemcpyAsync(c->ebuf, E, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const ncclResult_t r = n->AllReduce(c->ebuf, c->ebuf, 1, ncclFloat64, ncclSum, c->nccl_comm, c->stream);
  if (r != ncclSuccess) {
    c->poisoned = true;
    return set_err(DG_E_NCCL, std::string("ncclAllReduce: ") + n->GetErrorString(r));
  }
  CU(c, cudaMemcpyAsync(E, c->ebuf, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  return DG_OK;
}

dg_status dg_get_operators(const dg_ctx* c, double* r, double* s, double* Dr, double* Ds, double* LIFT,
                           int32_t* Fmask) {
  if (!c) return set_err(DG_E_ARG, "null context");
  const auto& R = c->ref;
  if (r) std::copy(R.r.begin(), R.r.end(), r);
  if (s) std::copy(R.s.begin(), R.s.end(), s);
  if (Dr) std::copy(R.Dr.begin(), R.Dr.end(), Dr);
  if (Ds) std::copy(R.Ds.begin(), R.Ds.end(), Ds);
  if (LIFT) std::copy(R.LIFT.begin(), R.LIFT.end(), LIFT);
  if (Fmask)
    for (size_t i = 0; i < R.Fmask.size(); ++i) Fmask[i] = R.Fmask[i];
  return DG_OK;
}

dg_status dg_get_geometry(const dg_ctx* c, double* rx, double* sx, double* ry, double* sy, double* J, double* nx,
                          double* ny, double* sJ, double* Fsc) {
  if (!c) return set_err(DG_E_ARG, "null context");
  const auto& m = c->mesh;
  auto cp = [](const std::vector<double>& v, double* d) { if (d) std::copy(v.begin(), v.end(), d); };
  cp(m.rx, rx); cp(m.sx, sx); cp(m.ry, ry); cp(m.sy, sy); cp(m.J, J);
  cp(m.nx, nx); cp(m.ny, ny); cp(m.sJ, sJ); cp(m.Fsc, Fsc);
  return DG_OK;
}

dg_status dg_get_maps(const dg_ctx* c, int32_t* EToE, int8_t* EToF, int64_t* vmapM, int64_t* vmapP) {
  if (!c) return set_err(DG_E_ARG, "null context");
  const auto& m = c->mesh;
  const int64_t Kl = (int64_t)m.local.size();
  const int NF = 3 * c->ref.Nfp;
  for (int64_t kl = 0; kl < Kl; ++kl) {
    const int64_t k = m.local[kl];
    for (int f = 0; f < 3; ++f) {
      if (EToE) EToE[3 * kl + f] = (int32_t)m.EToE[3 * k + f];
      if (EToF) EToF[3 * kl + f] = m.EToF[3 * k + f];
    }
    if (vmapM || vmapP) dg::face_maps(c->ref, m, kl, vmapM ? vmapM + kl * NF : nullptr, vmapP ? vmapP + kl * NF : nullptr);
  }
  return DG_OK;
}

dg_status dg_get_nodes(const dg_ctx* c, double* x, double* y) {
  if (!c || !x || !y) return set_err(DG_E_ARG, "null argument");
  const int Np = c->ref.Np;
  for (size_t kl = 0; kl < c->mesh.local.size(); ++kl)
    dg::element_nodes(c->ref, c->mesh, c->mesh.local[kl], x + kl * Np, y + kl * Np);
  return DG_OK;
}

dg_status dg_halo_sizes(const dg_ctx* c, int32_t* n_nbr, int64_t* n_send, int64_t* n_recv) {
  if (!c) return set_err(DG_E_ARG, "null context");
  if (n_nbr) *n_nbr = (int32_t)c->mesh.nbr.size();
  if (n_send) *n_send = (int64_t)c->mesh.send_gdof.size();
  if (n_recv) *n_recv = (int64_t)c->mesh.recv_gdof.size();
  return DG_OK;
}

dg_status dg_get_halo(const dg_ctx* c, int32_t* nbr, int64_t* send_off, int64_t* send_gdof, int64_t* recv_off,
                      int64_t* recv_gdof, int64_t* recv_point) {
  if (!c) return set_err(DG_E_ARG, "null context");
  const auto& m = c->mesh;
  if (nbr) std::copy(m.nbr.begin(), m.nbr.end(), nbr);
  if (send_off) std::copy(m.send_off.begin(), m.send_off.end(), send_off);
  if (send_gdof) std::copy(m.send_gdof.begin(), m.send_gdof.end(), send_gdof);
  if (recv_off) std::copy(m.recv_off.begin(), m.recv_off.end(), recv_off);
  if (recv_gdof) std::copy(m.recv_gdof.begin(), m.recv_gdof.end(), recv_gdof);
  if (recv_point) std::copy(m.recv_point.begin(), m.recv_point.end(), recv_point);
  return DG_OK;
}

dg_status dg_stream(const dg_ctx* c, void** stream) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  if (!stream) return set_err(DG_E_ARG, "null output");
  *stream = c->stream;
  return DG_OK;
}

dg_status dg_profile(dg_ctx* c, int32_t enable) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  CU(c, cudaSetDevice(c->device));
  CU(c, cudaStreamSynchronize(c->stream));
  c->profiling = enable != 0;
  c->timed.clear();
  c->stats = dg_kernel_stats{};
  return DG_OK;
}

dg_status dg_get_kernel_stats(dg_ctx* c, dg_kernel_stats* out) {
  dg_status st = check_usable(c, true);
  if (st != DG_OK) return st;
  if (!out) return set_err(DG_E_ARG, "null output");
  CU(c, cudaSetDevice(c->device));
  if (!c->timed.empty()) {
    CU(c, cudaStreamSynchronize(c->stream));
    for (const auto& t : c->timed) {
      float ms = 0.f;
      CU(c, cudaEventElapsedTime(&ms, c->ev_pool[t.ev0], c->ev_pool[t.ev1]));
      c->stats.ms[t.kind] += ms;
      c->stats.timed[t.kind] += 1;
    }
    c->timed.clear();
  }
  *out = c->stats;
  return DG_OK;
}

dg_status dg_get_kernel_config(const dg_ctx* c, dg_kernel_config* out) {
  dg_status st = check_usable(c, false);
  if (st != DG_OK) return st;
  if (!out) return set_err(DG_E_ARG, "null output");
  const dg::KernelModule* km = c->km ? c->km : dg::find_module(c->N, c->prec, c->kernel_variant);  // host-only
  if (!km) return set_err(DG_E_DEGREE, "no kernel module compiled for N=" + std::to_string(c->N));
  const dg::KernelInfo k = km->info();
  out->contraction = k.contraction;
  out->threads = k.threads;
  out->slots = k.slots;
  out->residual_tma = k.residual_tma;
  out->teams_cap = k.teams_cap;
  out->flags = k.flags;
  out->smem_bytes = (int64_t)k.smem_bytes;
  return DG_OK;
}

void dg_destroy(dg_ctx* c) {
  if (!c) return;
  if (!c->host_only) {
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    drop_graphs(c);
    if (c->nccl_comm) {
      Nccl* n = nccl();
      if (n) (c->poisoned ? n->CommAbort : n->CommDestroy)(c->nccl_comm);
    }
    void* bufs[] = {c->q[0], c->q[1], c->res, c->rhsv, c->out, c->geo, c->ops, c->vmapP, c->send_idx,
                    c->sendbuf, c->stage, c->flag, c->first_bad, c->ebuf, c->tiles_int, c->tiles_bnd,
                    c->perm_d, c->slot_of_d};
    for (void* b : bufs)
      if (b) cudaFree(b);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    if (c->ev_pack) cudaEventDestroy(c->ev_pack);
    if (c->ev_comm) cudaEventDestroy(c->ev_comm);
    if (c->comm) cudaStreamDestroy(c->comm);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  }
  delete c;
}

}  // extern "C"
