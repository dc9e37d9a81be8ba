// C ABI of the 3D tetrahedral Maxwell path (include/dg3.h): context, device
// buffers (tile-blocked, Morton element order), the LSERK4 stage loop (volume kernel, then surface +
// LIFT + RK kernel; CUDA-graph replay per step), helper kernels, exports.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/dg3.h"
#include "kernel3_api.h"
#include "kernel_api.h"
#include "setup3d.h"

namespace dg {
#define DG_MODULE3(tag) KernelModule3 dg_module3_##tag();
#include "modules3.inc"
#undef DG_MODULE3

const KernelModule3* find_module3(int N, int prec) {
  static const std::vector<KernelModule3> mods = {
#define DG_MODULE3(tag) dg_module3_##tag(),
#include "modules3.inc"
#undef DG_MODULE3
  };
  for (const auto& m : mods)
    if (m.N == N && m.prec == prec) return &m;
  return nullptr;
}
}  // namespace dg

// dg_last_error is defined in runtime.cu; the 3D calls report through the same thread-local message
namespace dg {
void set_last_error(const std::string& m);
}

namespace {

const double kA[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                      -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double kB[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                      1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                      2277821191437.0 / 14882151754819.0};

dg_status err3(dg_status s, const std::string& m) {
  dg::set_last_error(m);
  return s;
}

// canonical fp64 [6][K][Np] <-> tile-blocked T [6][fstride]; slot d holds element perm[d] (-1: pad)
template <typename T>
__global__ void to_blocked6(const double* __restrict__ src, T* __restrict__ q, const int32_t* __restrict__ perm,
                            int64_t K, int64_t Kpad, int Np, int64_t fstride) {
  const int64_t total = Kpad * Np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 6 * total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / total);
    const int64_t o = i - c * total, tn = o >> 5, t = tn / Np;
    const int n = (int)(tn - t * Np);
    const int64_t k = perm[t * 32 + (o & 31)];
    q[c * fstride + o] = k >= 0 ? static_cast<T>(src[(c * K + k) * Np + n]) : T(0);
  }
}
template <typename T>
__global__ void from_blocked6(const T* __restrict__ q, double* __restrict__ dst, const int32_t* __restrict__ slot,
                              int64_t K, int Np, int64_t fstride) {
  const int64_t total = K * Np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 6 * total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / total);
    const int64_t o = i - c * total, k = o / Np;
    const int n = (int)(o - k * Np);
    const int64_t d = slot[k];
    dst[c * total + o] = static_cast<double>(q[c * fstride + ((d >> 5) * Np + n) * 32 + (d & 31)]);
  }
}
template <typename T>
__global__ void count_bad6(const T* __restrict__ q, int64_t n, int64_t fstride, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 6 * n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / n);
    if (!isfinite(q[c * fstride + (i - c * n)])) ++local;
  }
  if (local) atomicAdd(bad, local);
}
int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

// Morton (Z-order) sort of the element centroids: a 32-element tile is a compact cluster
std::vector<int64_t> morton_order3(const dg::Mesh3D& m) {
  const int64_t K = m.K;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  std::vector<double> c(3 * K);
  for (int64_t k = 0; k < K; ++k) {
    const double* V[3] = {m.VX.data(), m.VY.data(), m.VZ.data()};
    for (int d = 0; d < 3; ++d) {
      double s = 0.0;
      for (int v = 0; v < 4; ++v) s += V[d][m.EToV[4 * k + v]];
      c[3 * k + d] = s / 4.0;
      lo[d] = std::min(lo[d], s / 4.0);
      hi[d] = std::max(hi[d], s / 4.0);
    }
  }
  auto spread = [](uint64_t x) {  // 21 bits -> every third bit
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
  };
  std::vector<uint64_t> code(K);
  for (int64_t k = 0; k < K; ++k) {
    uint64_t q[3];
    for (int d = 0; d < 3; ++d) {
      const double w = hi[d] > lo[d] ? (c[3 * k + d] - lo[d]) / (hi[d] - lo[d]) : 0.0;
      q[d] = (uint64_t)std::min(2097151.0, std::max(0.0, w * 2097151.0));
    }
    code[k] = spread(q[0]) | spread(q[1]) << 1 | spread(q[2]) << 2;
  }
  std::vector<int64_t> perm(K);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return code[a] < code[b]; });
  return perm;
}

}  // namespace

struct dg3_ctx {
  int N = 0, prec = 8, device = -1, max_ctas = 0;
  bool fused = false;  // the fused stage kernel (dg_options.fused and the module has one)
  double alpha = 1.0;
  bool host_only = true, poisoned = false;
  dg::RefTet ref;
  dg::Mesh3D mesh;
  const dg::KernelModule3* km = nullptr;
  int64_t K = 0, ntiles = 0, Kpad = 0, fstride = 0, vstride = 0;
  size_t tsz = 8;
  std::vector<int64_t> perm, slot;
  void *q[2] = {nullptr, nullptr}, *res = nullptr, *rhsv = nullptr, *out = nullptr, *geo = nullptr, *ops = nullptr;
  int32_t *codes = nullptr, *perm_d = nullptr, *slot_d = nullptr;
  double* stage = nullptr;
  unsigned long long* flag = nullptr;
  int cur = 0;
  int64_t steps_done = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  double gdt = 0.0;
  bool profiling = false;
  std::vector<cudaEvent_t> ev;
  struct Timed { int kind, e0, e1; };
  std::vector<Timed> timed;
  dg_kernel_stats stats{};
};

namespace {

dg_status cuda3(dg3_ctx* c, cudaError_t e, const char* what) {
  if (c) c->poisoned = true;
  return err3(DG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CU3(ctx, x)                                          \
  do {                                                       \
    cudaError_t e__ = (x);                                   \
    if (e__ != cudaSuccess) return cuda3(ctx, e__, #x);      \
  } while (0)

dg_status usable(const dg3_ctx* c, bool device) {
  if (!c) return err3(DG_E_ARG, "null context");
  if (c->poisoned) return err3(DG_E_STATE, "context is poisoned by an earlier CUDA error");
  if (device && c->host_only) return err3(DG_E_STATE, "host-only context (device = -1) cannot compute");
  return DG_OK;
}

dg::StageArgs3 args(dg3_ctx* c) {
  dg::StageArgs3 a{};
  a.q_in = c->q[c->cur];
  a.q_out = c->q[1 - c->cur];
  a.res = c->res;
  a.rhsv = c->rhsv;
  a.out = c->out;
  a.geo = c->geo;
  a.vmapP = c->codes;
  a.ops = c->ops;
  a.fstride = c->fstride;
  a.vstride = c->vstride;
  a.ntiles = (int32_t)c->ntiles;
  a.write_res = 1;
  a.max_ctas = c->max_ctas;
  a.alpha = c->alpha;
  return a;
}

dg_status launch3(dg3_ctx* c, int mode, const dg::StageArgs3& a, int kind) {
  int e0 = -1;
  if (c->profiling) {
    if (c->ev.size() < c->timed.size() * 2 + 2)
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        CU3(c, cudaEventCreate(&e));
        c->ev.push_back(e);
      }
    e0 = (int)c->timed.size() * 2;
    CU3(c, cudaEventRecord(c->ev[e0], c->stream));
  }
  const cudaError_t e = c->km->launch(mode, a, c->stream);
  if (e != cudaSuccess) return cuda3(c, e, "3D stage kernel launch");
  c->stats.launches[kind] += 1;
  if (e0 >= 0) {
    CU3(c, cudaEventRecord(c->ev[e0 + 1], c->stream));
    c->timed.push_back({kind, e0, e0 + 1});
  }
  return DG_OK;
}

dg_status stage3(dg3_ctx* c, int i, double dt) {
  dg::StageArgs3 a = args(c);
  a.a = kA[i];
  a.b = kB[i];
  a.dt = dt;
  a.write_res = i == 4 ? 0 : 1;
  dg::StageArgs3 av = a;
  av.out = c->rhsv;
  dg_status st;
  if (c->fused) {  // volume + flux + LIFT + LSERK4 in one launch
    if ((st = launch3(c, dg::MODE_FUSED_RK, a, 0)) != DG_OK) return st;
  } else {
    if ((st = launch3(c, dg::MODE_VOLUME, av, 1)) != DG_OK) return st;
    if ((st = launch3(c, dg::MODE_SURFACE_RK, a, 2)) != DG_OK) return st;
  }
  c->cur = 1 - c->cur;
  return DG_OK;
}

dg_status alloc3(dg3_ctx* c, void** p, size_t bytes) {
  const cudaError_t e = cudaMalloc(p, bytes ? bytes : 256);
  if (e != cudaSuccess) {
    c->poisoned = true;
    return err3(e == cudaErrorMemoryAllocation ? DG_E_OOM : DG_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return DG_OK;
}

template <typename T>
void host_geometry(dg3_ctx* c, std::vector<T>& g, std::vector<int32_t>& codes) {
  const int Np = c->ref.Np, Nfp = c->ref.Nfp, NF = 4 * Nfp, NG = dg::NGEO3;
  const dg::Mesh3D& m = c->mesh;
  g.assign((size_t)c->ntiles * NG * 32, T(0));
  codes.assign((size_t)c->ntiles * NF * 32, 0);
  auto blk = [&](int64_t d, int n) { return ((d >> 5) * Np + n) * 32 + (d & 31); };
  for (int64_t d = 0; d < c->Kpad; ++d) {
    const int64_t t = d >> 5, lane = d & 31;
    auto G = [&](int comp) -> T& { return g[(t * NG + comp) * 32 + lane]; };
    if (d >= c->K) {  // padding: identity geometry, neighbour = itself
      G(0) = G(4) = G(8) = T(1);
      for (int f = 0; f < 4; ++f) G(25 + f) = T(1);
      for (int mm = 0; mm < NF; ++mm) codes[(t * NF + mm) * 32 + lane] = (int32_t)blk(d, c->ref.Fmask[mm]);
      continue;
    }
    const int64_t k = c->perm[d];
    const double gf[9] = {m.rx[k], m.ry[k], m.rz[k], m.sx[k], m.sy[k], m.sz[k], m.tx[k], m.ty[k], m.tz[k]};
    for (int i = 0; i < 9; ++i) G(i) = (T)gf[i];
    for (int f = 0; f < 4; ++f) {
      G(9 + 4 * f) = (T)m.nx[4 * k + f];
      G(10 + 4 * f) = (T)m.ny[4 * k + f];
      G(11 + 4 * f) = (T)m.nz[4 * k + f];
      G(12 + 4 * f) = (T)(0.5 * m.Fsc[4 * k + f]);
      const bool bnd = m.EToE[4 * k + f] == k && m.EToF[4 * k + f] == f;
      G(25 + f) = bnd ? T(-1) : T(1);
    }
    for (int mm = 0; mm < NF; ++mm) {
      const int64_t gp = m.vmapP[k * NF + mm];
      const int64_t k2 = gp / Np, d2 = c->slot[k2];
      const int n2 = (int)(gp - k2 * Np);
      codes[(t * NF + mm) * 32 + lane] =
          (c->km->staged && (d2 >> 5) == t) ? (int32_t)(-(1 + (int64_t)n2 * 32 + (d2 & 31))) : (int32_t)blk(d2, n2);
    }
  }
}

dg_status setup_device3(dg3_ctx* c, const dg_options* o) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return err3(DG_E_CUDA, std::string("no usable CUDA device: ") + cudaGetErrorString(e));
  if (c->device >= ndev) return err3(DG_E_ARG, "device ordinal out of range");
  CU3(c, cudaSetDevice(c->device));
  c->km = dg::find_module3(c->N, c->prec);
  if (c->km && !c->km->fused) c->fused = false;
  if (!c->km) return err3(DG_E_DEGREE, "no 3D kernel module for N=" + std::to_string(c->N) + " precision=" +
                                           std::to_string(c->prec));
  const int Np = c->ref.Np;
  c->tsz = (size_t)c->prec;
  c->ntiles = (c->K + 31) / 32;
  c->Kpad = c->ntiles * 32;
  c->fstride = c->vstride = c->Kpad * Np;
  if (6 * c->fstride >= ((int64_t)1 << 31)) return err3(DG_E_ARG, "mesh too large for 32-bit face codes");
  c->perm = morton_order3(c->mesh);
  c->slot.assign(c->K, 0);
  for (int64_t d = 0; d < c->K; ++d) c->slot[c->perm[d]] = d;
  dg_status st;
  {
    std::vector<int32_t> pd(c->Kpad, -1), sd(c->K);
    for (int64_t d = 0; d < c->K; ++d) pd[d] = (int32_t)c->perm[d];
    for (int64_t k = 0; k < c->K; ++k) sd[k] = (int32_t)c->slot[k];
    if ((st = alloc3(c, (void**)&c->perm_d, pd.size() * 4)) != DG_OK) return st;
    if ((st = alloc3(c, (void**)&c->slot_d, sd.size() * 4)) != DG_OK) return st;
    CU3(c, cudaMemcpy(c->perm_d, pd.data(), pd.size() * 4, cudaMemcpyHostToDevice));
    CU3(c, cudaMemcpy(c->slot_d, sd.data(), sd.size() * 4, cudaMemcpyHostToDevice));
  }
  const size_t fb = 6 * (size_t)c->fstride * c->tsz;
  for (int b = 0; b < 2; ++b)
    if ((st = alloc3(c, &c->q[b], fb)) != DG_OK) return st;
  if ((st = alloc3(c, &c->res, fb)) != DG_OK) return st;
  if ((st = alloc3(c, &c->rhsv, fb)) != DG_OK) return st;
  if ((st = alloc3(c, (void**)&c->stage, 6 * (size_t)c->K * Np * 8)) != DG_OK) return st;
  if ((st = alloc3(c, (void**)&c->flag, 8)) != DG_OK) return st;
  CU3(c, cudaMemset(c->q[0], 0, fb));
  CU3(c, cudaMemset(c->q[1], 0, fb));
  CU3(c, cudaMemset(c->res, 0, fb));
  {
    std::vector<unsigned char> ops(c->km->ops_bytes());
    c->km->pack_ops(c->ref.Dr.data(), c->ref.Ds.data(), c->ref.Dt.data(), c->ref.LIFT.data(), c->ref.Fmask.data(),
                    ops.data());
    if ((st = alloc3(c, &c->ops, ops.size())) != DG_OK) return st;
    CU3(c, cudaMemcpy(c->ops, ops.data(), ops.size(), cudaMemcpyHostToDevice));
  }
  std::vector<int32_t> codes;
  if (c->tsz == 4) {
    std::vector<float> g;
    host_geometry(c, g, codes);
    if ((st = alloc3(c, &c->geo, g.size() * 4)) != DG_OK) return st;
    CU3(c, cudaMemcpy(c->geo, g.data(), g.size() * 4, cudaMemcpyHostToDevice));
  } else {
    std::vector<double> g;
    host_geometry(c, g, codes);
    if ((st = alloc3(c, &c->geo, g.size() * 8)) != DG_OK) return st;
    CU3(c, cudaMemcpy(c->geo, g.data(), g.size() * 8, cudaMemcpyHostToDevice));
  }
  if ((st = alloc3(c, (void**)&c->codes, codes.size() * 4)) != DG_OK) return st;
  CU3(c, cudaMemcpy(c->codes, codes.data(), codes.size() * 4, cudaMemcpyHostToDevice));
  if (o->stream) {
    c->stream = static_cast<cudaStream_t>(o->stream);
  } else {
    CU3(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  CU3(c, cudaDeviceSynchronize());
  return DG_OK;
}

void drop3(dg3_ctx* c) {
  for (auto& g : c->gexec)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
}

}  // namespace

extern "C" {

dg_status dg3_setup(const dg_options* o, int64_t Nv, const double* VX, const double* VY, const double* VZ, int64_t K,
                    const int64_t* EToV, dg3_ctx** out) {
  if (!o || !out || !VX || !VY || !VZ || !EToV) return err3(DG_E_ARG, "null argument to dg3_setup");
  *out = nullptr;
  if (o->abi_version != DG_ABI_VERSION) return err3(DG_E_ARG, "ABI version mismatch");
  if (o->precision != 4 && o->precision != 8) return err3(DG_E_ARG, "precision must be 4 or 8");
  if (o->nranks != 1 || o->rank != 0) return err3(DG_E_ARG, "the 3D path is single-GPU (rank 0 of 1)");
  if (!(o->alpha >= 0.0) || o->max_ctas < 0) return err3(DG_E_ARG, "alpha and max_ctas must be >= 0");
  std::unique_ptr<dg3_ctx> c(new dg3_ctx());
  c->N = o->N;
  c->prec = o->precision;
  c->device = o->device;
  c->alpha = o->alpha;
  c->max_ctas = o->max_ctas;
  c->fused = o->fused != 0;  // effective only where the module has a fused kernel (setup_device3)
  try {
    c->ref = dg::build_reftet(o->N);
    dg::build_mesh3d(c->ref, Nv, VX, VY, VZ, K, EToV, c->mesh);
  } catch (const dg::SetupError& e) {
    return err3((dg_status)e.status, e.msg);
  } catch (const std::bad_alloc&) {
    return err3(DG_E_OOM, "host allocation failed in 3D setup");
  }
  c->K = K;
  c->host_only = o->device < 0;
  if (!c->host_only) {
    const dg_status st = setup_device3(c.get(), o);
    if (st != DG_OK) {
      dg3_destroy(c.release());
      return st;
    }
  }
  *out = c.release();
  return DG_OK;
}

dg_status dg3_sizes(const dg3_ctx* c, int64_t* Np, int64_t* Nfp, int64_t* K, int64_t* n_swapped) {
  if (!c) return err3(DG_E_ARG, "null context");
  if (Np) *Np = c->ref.Np;
  if (Nfp) *Nfp = c->ref.Nfp;
  if (K) *K = c->K;
  if (n_swapped) *n_swapped = c->mesh.n_swapped;
  return DG_OK;
}

dg_status dg3_set_fields(dg3_ctx* c, const double* const* f) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  if (!f) return err3(DG_E_ARG, "null fields");
  for (int i = 0; i < 6; ++i)
    if (!f[i]) return err3(DG_E_ARG, "null field pointer");
  CU3(c, cudaSetDevice(c->device));
  const int64_t n = c->K * c->ref.Np;
  for (int i = 0; i < 6; ++i)
    CU3(c, cudaMemcpyAsync(c->stage + i * n, f[i], n * 8, cudaMemcpyDefault, c->stream));
  if (c->tsz == 4)
    to_blocked6<float><<<grid_of(6 * c->Kpad * c->ref.Np), 256, 0, c->stream>>>(c->stage, (float*)c->q[c->cur], c->perm_d,
                                                                               c->K, c->Kpad, c->ref.Np, c->fstride);
  else
    to_blocked6<double><<<grid_of(6 * c->Kpad * c->ref.Np), 256, 0, c->stream>>>(c->stage, (double*)c->q[c->cur],
                                                                                c->perm_d, c->K, c->Kpad, c->ref.Np,
                                                                                c->fstride);
  CU3(c, cudaGetLastError());
  CU3(c, cudaMemsetAsync(c->res, 0, 6 * (size_t)c->vstride * c->tsz, c->stream));
  CU3(c, cudaStreamSynchronize(c->stream));
  c->steps_done = 0;
  return DG_OK;
}

static dg_status get_blocked(dg3_ctx* c, const void* src, int64_t stride, double* const* f) {
  const int64_t n = c->K * c->ref.Np;
  if (c->tsz == 4)
    from_blocked6<float><<<grid_of(6 * n), 256, 0, c->stream>>>((const float*)src, c->stage, c->slot_d, c->K,
                                                                c->ref.Np, stride);
  else
    from_blocked6<double><<<grid_of(6 * n), 256, 0, c->stream>>>((const double*)src, c->stage, c->slot_d, c->K,
                                                                 c->ref.Np, stride);
  CU3(c, cudaGetLastError());
  for (int i = 0; i < 6; ++i) CU3(c, cudaMemcpyAsync(f[i], c->stage + i * n, n * 8, cudaMemcpyDefault, c->stream));
  CU3(c, cudaStreamSynchronize(c->stream));
  return DG_OK;
}

dg_status dg3_get_fields(dg3_ctx* c, double* const* f) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  if (!f) return err3(DG_E_ARG, "null fields");
  for (int i = 0; i < 6; ++i)
    if (!f[i]) return err3(DG_E_ARG, "null field pointer");
  CU3(c, cudaSetDevice(c->device));
  return get_blocked(c, c->q[c->cur], c->fstride, f);
}

dg_status dg3_run(dg3_ctx* c, double dt, int64_t nsteps) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  if (!(dt > 0.0) || !std::isfinite(dt) || nsteps < 0) return err3(DG_E_ARG, "need dt > 0 and nsteps >= 0");
  CU3(c, cudaSetDevice(c->device));
  for (int64_t s = 0; s < nsteps; ++s) {
    if (c->steps_done > 0 && !c->profiling) {  // CUDA-graph replay of one step per ping-pong parity
      if (c->gdt != dt) {
        drop3(c);
        c->gdt = dt;
      }
      const int par = c->cur;
      if (!c->gexec[par]) {
        const dg_kernel_stats keep = c->stats;
        CU3(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < 5 && st == DG_OK; ++i) st = stage3(c, i, dt);
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        c->cur = par;
        c->stats = keep;
        if (st != DG_OK) {
          if (g) cudaGraphDestroy(g);
          return st;
        }
        if (e != cudaSuccess) return cuda3(c, e, "cudaStreamEndCapture");
        const cudaError_t e2 = cudaGraphInstantiate(&c->gexec[par], g, 0);
        cudaGraphDestroy(g);
        if (e2 != cudaSuccess) return cuda3(c, e2, "cudaGraphInstantiate");
      }
      CU3(c, cudaGraphLaunch(c->gexec[par], c->stream));
      if (c->fused) {
        c->stats.launches[0] += 5;
      } else {
        c->stats.launches[1] += 5;
        c->stats.launches[2] += 5;
      }
      c->cur = 1 - c->cur;
    } else {
      for (int i = 0; i < 5; ++i)
        if ((st = stage3(c, i, dt)) != DG_OK) return st;
    }
    ++c->steps_done;
  }
  return DG_OK;
}

dg_status dg3_sync(dg3_ctx* c) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  CU3(c, cudaSetDevice(c->device));
  CU3(c, cudaMemsetAsync(c->flag, 0, 8, c->stream));
  const int64_t n = c->Kpad * c->ref.Np;
  if (c->tsz == 4)
    count_bad6<float><<<grid_of(6 * n), 256, 0, c->stream>>>((const float*)c->q[c->cur], n, c->fstride, c->flag);
  else
    count_bad6<double><<<grid_of(6 * n), 256, 0, c->stream>>>((const double*)c->q[c->cur], n, c->fstride, c->flag);
  CU3(c, cudaGetLastError());
  unsigned long long bad = 0;
  CU3(c, cudaMemcpyAsync(&bad, c->flag, 8, cudaMemcpyDeviceToHost, c->stream));
  CU3(c, cudaStreamSynchronize(c->stream));
  if (bad) return err3(DG_E_DIVERGED, std::to_string(bad) + " non-finite field values after step " + std::to_string(c->steps_done));
  return DG_OK;
}

dg_status dg3_eval_rhs(dg3_ctx* c, int32_t which, double* const* f) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  if (which < 0 || which > 2 || !f) return err3(DG_E_ARG, "bad dg3_eval_rhs arguments");
  for (int i = 0; i < 6; ++i)
    if (!f[i]) return err3(DG_E_ARG, "null output pointer");
  CU3(c, cudaSetDevice(c->device));
  if (!c->out && (st = alloc3(c, &c->out, 6 * (size_t)c->vstride * c->tsz)) != DG_OK) return st;
  dg::StageArgs3 a = args(c);
  if (which != 2) {
    dg::StageArgs3 av = a;
    av.out = which == 1 ? c->out : c->rhsv;
    if ((st = launch3(c, dg::MODE_VOLUME, av, 1)) != DG_OK) return st;
  }
  if (which != 1 && (st = launch3(c, which == 0 ? dg::MODE_RHS : dg::MODE_SURFACE, a, 2)) != DG_OK) return st;
  return get_blocked(c, c->out, c->vstride, f);
}

dg_status dg3_energy(dg3_ctx* c, double* E) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  if (!E) return err3(DG_E_ARG, "null output");
  const int Np = c->ref.Np;
  const int64_t n = c->K * Np;
  std::vector<double> buf(6 * n);
  double* f[6];
  for (int i = 0; i < 6; ++i) f[i] = buf.data() + i * n;
  if ((st = dg3_get_fields(c, f)) != DG_OK) return st;
  double tot = 0.0;
  for (int64_t k = 0; k < c->K; ++k) {
    double ek = 0.0;
    for (int i = 0; i < 6; ++i) {
      const double* u = f[i] + k * Np;
      for (int a = 0; a < Np; ++a) {
        double acc = 0.0;
        for (int b = 0; b < Np; ++b) acc += c->ref.M[a * Np + b] * u[b];
        ek += u[a] * acc;
      }
    }
    tot += c->mesh.J[k] * ek;
  }
  *E = 0.5 * tot;
  return DG_OK;
}

dg_status dg3_get_operators(const dg3_ctx* c, double* r, double* s, double* t, double* Dr, double* Ds, double* Dt,
                            double* LIFT, int32_t* Fmask) {
  if (!c) return err3(DG_E_ARG, "null context");
  const auto& R = c->ref;
  auto cp = [](const std::vector<double>& v, double* d) { if (d) std::copy(v.begin(), v.end(), d); };
  cp(R.r, r); cp(R.s, s); cp(R.t, t); cp(R.Dr, Dr); cp(R.Ds, Ds); cp(R.Dt, Dt); cp(R.LIFT, LIFT);
  if (Fmask) std::copy(R.Fmask.begin(), R.Fmask.end(), Fmask);
  return DG_OK;
}

dg_status dg3_get_maps(const dg3_ctx* c, int32_t* EToE, int8_t* EToF, int64_t* vmapP) {
  if (!c) return err3(DG_E_ARG, "null context");
  const auto& m = c->mesh;
  for (int64_t i = 0; i < 4 * c->K; ++i) {
    if (EToE) EToE[i] = (int32_t)m.EToE[i];
    if (EToF) EToF[i] = m.EToF[i];
  }
  if (vmapP) std::copy(m.vmapP.begin(), m.vmapP.end(), vmapP);
  return DG_OK;
}

dg_status dg3_get_nodes(const dg3_ctx* c, double* x, double* y, double* z) {
  if (!c || !x || !y || !z) return err3(DG_E_ARG, "null argument");
  const int Np = c->ref.Np;
  for (int64_t k = 0; k < c->K; ++k) dg::element_nodes3d(c->ref, c->mesh, k, x + k * Np, y + k * Np, z + k * Np);
  return DG_OK;
}

dg_status dg3_get_geometry(const dg3_ctx* c, double* gfac, double* J, double* nx, double* ny, double* nz, double* sJ,
                           double* Fsc) {
  if (!c) return err3(DG_E_ARG, "null context");
  const auto& m = c->mesh;
  for (int64_t k = 0; k < c->K; ++k) {
    if (gfac) {
      const double v[9] = {m.rx[k], m.ry[k], m.rz[k], m.sx[k], m.sy[k], m.sz[k], m.tx[k], m.ty[k], m.tz[k]};
      std::copy(v, v + 9, gfac + 9 * k);
    }
    if (J) J[k] = m.J[k];
  }
  auto cp = [](const std::vector<double>& v, double* d) { if (d) std::copy(v.begin(), v.end(), d); };
  cp(m.nx, nx); cp(m.ny, ny); cp(m.nz, nz); cp(m.sJ, sJ); cp(m.Fsc, Fsc);
  return DG_OK;
}

dg_status dg3_stream(const dg3_ctx* c, void** s) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  if (!s) return err3(DG_E_ARG, "null output");
  *s = c->stream;
  return DG_OK;
}

dg_status dg3_profile(dg3_ctx* c, int32_t enable) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  CU3(c, cudaSetDevice(c->device));
  CU3(c, cudaStreamSynchronize(c->stream));
  c->profiling = enable != 0;
  c->timed.clear();
  c->stats = dg_kernel_stats{};
  return DG_OK;
}

dg_status dg3_get_kernel_stats(dg3_ctx* c, dg_kernel_stats* out) {
  dg_status st = usable(c, true);
  if (st != DG_OK) return st;
  if (!out) return err3(DG_E_ARG, "null output");
  if (!c->timed.empty()) {
    CU3(c, cudaStreamSynchronize(c->stream));
    for (const auto& t : c->timed) {
      float ms = 0.f;
      CU3(c, cudaEventElapsedTime(&ms, c->ev[t.e0], c->ev[t.e1]));
      c->stats.ms[t.kind] += ms;
      c->stats.timed[t.kind] += 1;
    }
    c->timed.clear();
  }
  *out = c->stats;
  return DG_OK;
}

void dg3_destroy(dg3_ctx* c) {
  if (!c) return;
  if (!c->host_only) {
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    drop3(c);
    void* bufs[] = {c->q[0], c->q[1], c->res, c->rhsv, c->out, c->geo, c->ops, c->codes, c->perm_d, c->slot_d,
                    c->stage, c->flag};
    for (void* b : bufs)
      if (b) cudaFree(b);
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  }
  delete c;
}

}  // extern "C"
