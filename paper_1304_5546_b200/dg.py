"""Thin ctypes binding of the C ABI in include/dg.h (argument marshalling only).

Every step of the hot path runs in libdg.so's CUDA kernels; there is no Python
or CPU compute path here.  If the library is missing, importing this module
raises ImportError -- build it with ``python -m paper_1304_5546_b200.build``.

The names follow the C ABI: ``dg_setup`` returns a :class:`Context` whose
methods are the remaining ``dg_*`` calls without the prefix (``ctx.run(dt, n)``
is ``dg_run``), plus module-level ``dg_run_group``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DG_LIB") or os.path.join(_HERE, "lib", "libdg.so")  # DG_LIB: dev override

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built; run `python -m paper_1304_5546_b200.build`")
_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

ABI_VERSION = 2
MAX_KERNEL_N = 9

STATUS = {0: "DG_OK", 1: "DG_E_ARG", 2: "DG_E_DEGREE", 3: "DG_E_MESH_DEGENERATE",
          4: "DG_E_MESH_NONMANIFOLD", 5: "DG_E_MESH_NONCONFORMING", 6: "DG_E_UNSUPPORTED_BC",
          7: "DG_E_CUDA", 8: "DG_E_NCCL", 9: "DG_E_OOM", 10: "DG_E_DIVERGED", 11: "DG_E_STATE"}

EXPORTS = ["dg_options_default", "dg_setup", "dg_sizes", "dg_local_elements", "dg_set_fields",
           "dg_get_fields", "dg_run", "dg_run_group", "dg_sync", "dg_eval_rhs", "dg_energy", "dg_energy_local",
           "dg_get_operators", "dg_get_geometry", "dg_get_maps", "dg_get_nodes", "dg_halo_sizes",
           "dg_get_halo", "dg_stream", "dg_profile", "dg_get_kernel_stats", "dg_get_kernel_config", "dg_set_graphs",
           "dg_destroy", "dg_last_error"]


class DGError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Options(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("N", C.c_int32), ("precision", C.c_int32),
                ("device", C.c_int32), ("alpha", C.c_double), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("fused", C.c_int32), ("transport", C.c_int32),
                ("nccl_id", C.c_void_p), ("part", C.c_void_p), ("stream", C.c_void_p),
                ("max_ctas", C.c_int32), ("tile_order", C.c_int32), ("check_every", C.c_int32),
                ("kernel_variant", C.c_int32)]


class KernelStats(C.Structure):
    _fields_ = [("launches", C.c_int64 * 4), ("ms", C.c_double * 4), ("timed", C.c_int64 * 4)]


KIND = ("fused", "volume", "surface", "helper")


class KernelConfig(C.Structure):
    _fields_ = [("contraction", C.c_int32), ("threads", C.c_int32), ("slots", C.c_int32),
                ("residual_tma", C.c_int32), ("teams_cap", C.c_int32), ("flags", C.c_int32),
                ("smem_bytes", C.c_int64)]


CONTRACTION = ("fma", "dmma_fp64", "3xtf32", "tcgen05_3xtf32")

_vp = C.c_void_p
_i64 = C.c_int64
_P = C.POINTER
_sig = {
    "dg_options_default": [_vp],
    "dg_setup": [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _P(_vp)],
    "dg_sizes": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "dg_local_elements": [_vp, _vp],
    "dg_set_fields": [_vp, _vp, _vp, _vp],
    "dg_get_fields": [_vp, _vp, _vp, _vp],
    "dg_run": [_vp, C.c_double, _i64],
    "dg_run_group": [_vp, C.c_int32, C.c_double, _i64],
    "dg_sync": [_vp],
    "dg_eval_rhs": [_vp, C.c_int32, _vp, _vp, _vp],
    "dg_energy": [_vp, _vp],
    "dg_energy_local": [_vp, _vp],
    "dg_get_operators": [_vp] * 7,
    "dg_get_geometry": [_vp] * 10,
    "dg_get_maps": [_vp] * 5,
    "dg_get_nodes": [_vp] * 3,
    "dg_halo_sizes": [_vp] * 4,
    "dg_get_halo": [_vp] * 7,
    "dg_stream": [_vp, _P(_vp)],
    "dg_profile": [_vp, C.c_int32],
    "dg_get_kernel_stats": [_vp, _vp],
    "dg_get_kernel_config": [_vp, _vp],
    "dg_set_graphs": [_vp, C.c_int32],
}
for _name, _args in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
_lib.dg_destroy.argtypes = [_vp]
_lib.dg_destroy.restype = None
_lib.dg_last_error.argtypes = []
_lib.dg_last_error.restype = C.c_char_p


def last_error():
    return _lib.dg_last_error().decode()


def _check(st):
    if st != 0:
        raise DGError(st, last_error())


def _ptr(a):
    """Pointer of a C-contiguous numpy array or a (CPU or CUDA) torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


def _as(a, dtype, n=None):
    arr = np.ascontiguousarray(a, dtype=dtype)
    if n is not None and arr.size != n:
        raise ValueError(f"expected {n} values, got {arr.size}")
    return arr


def dg_options_default():
    o = Options()
    _check(_lib.dg_options_default(C.byref(o)))
    return o


class Context:
    """A dg_ctx (one rank's partition).  Create with :func:`dg_setup`."""

    def __init__(self, handle, N, precision):
        self._h = handle
        self.N = N
        self.precision = precision
        np_, nfp, kl, kg, nh, nsw = (C.c_int64() for _ in range(6))
        _check(_lib.dg_sizes(self._h, C.byref(np_), C.byref(nfp), C.byref(kl), C.byref(kg),
                             C.byref(nh), C.byref(nsw)))
        self.Np, self.Nfp, self.K_local, self.K_global = np_.value, nfp.value, kl.value, kg.value
        self.n_halo_points, self.n_swapped = nh.value, nsw.value

    # -- lifecycle
    def destroy(self):
        if self._h:
            _lib.dg_destroy(self._h)
            self._h = None

    close = destroy

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.destroy()

    @property
    def handle(self):
        return self._h

    # -- fields
    def _fields_io(self, fields, writable=False):
        """Validate field buffers: numpy arrays (converted to contiguous fp64 on input) or torch
        tensors (fp64, contiguous, CPU or this context's CUDA device -- dg_set_fields /
        dg_get_fields copy with cudaMemcpyDefault), each of K_local * Np values."""
        n = self.K_local * self.Np
        out = []
        for a in fields:
            if isinstance(a, np.ndarray):
                if writable:
                    if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or a.size != n \
                            or not a.flags["WRITEABLE"]:
                        raise ValueError(f"output arrays must be writable C-contiguous float64 of {n} values")
                else:
                    a = _as(a, np.float64, n)
            else:  # torch tensor
                if str(a.dtype) != "torch.float64" or not a.is_contiguous() or a.numel() != n:
                    raise ValueError(f"field tensors must be contiguous torch.float64 of {n} values")
                if a.device.type not in ("cpu", "cuda"):
                    raise ValueError(f"unsupported tensor device {a.device}")
            out.append(a)
        return out

    def local_elements(self):
        g = np.empty(self.K_local, dtype=np.int64)
        _check(_lib.dg_local_elements(self._h, _ptr(g)))
        return g

    def set_fields(self, Hx, Hy, Ez):
        a = self._fields_io((Hx, Hy, Ez))
        _check(_lib.dg_set_fields(self._h, _ptr(a[0]), _ptr(a[1]), _ptr(a[2])))

    def get_fields(self, out=None):
        if out is None:
            out = tuple(np.empty((self.K_local, self.Np)) for _ in range(3))
        self._fields_io(out, writable=True)
        _check(_lib.dg_get_fields(self._h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    def run(self, dt, nsteps):
        _check(_lib.dg_run(self._h, float(dt), int(nsteps)))

    def sync(self):
        _check(_lib.dg_sync(self._h))

    def eval_rhs(self, which=0):
        which = {"full": 0, "volume": 1, "surface": 2}.get(which, which)
        out = tuple(np.empty((self.K_local, self.Np)) for _ in range(3))
        _check(_lib.dg_eval_rhs(self._h, int(which), _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    def energy(self):
        """dg_energy: the whole mesh's energy (all-reduced over an NCCL communicator: collective)."""
        e = C.c_double()
        _check(_lib.dg_energy(self._h, C.byref(e)))
        return e.value

    def energy_local(self):
        """dg_energy_local: this partition's share of the energy (no communication)."""
        e = C.c_double()
        _check(_lib.dg_energy_local(self._h, C.byref(e)))
        return e.value

    # -- verification exports
    def operators(self):
        Np, Nfp = self.Np, self.Nfp
        r, s = np.empty(Np), np.empty(Np)
        Dr, Ds = np.empty((Np, Np)), np.empty((Np, Np))
        LIFT = np.empty((Np, 3 * Nfp))
        Fmask = np.empty((3, Nfp), dtype=np.int32)
        _check(_lib.dg_get_operators(self._h, *(_ptr(x) for x in (r, s, Dr, Ds, LIFT, Fmask))))
        return dict(r=r, s=s, Dr=Dr, Ds=Ds, LIFT=LIFT, Fmask=Fmask)

    def geometry(self):
        K = self.K_local
        names1 = ("rx", "sx", "ry", "sy", "J")
        names3 = ("nx", "ny", "sJ", "Fsc")
        d = {n: np.empty(K) for n in names1}
        d.update({n: np.empty((K, 3)) for n in names3})
        _check(_lib.dg_get_geometry(self._h, *(_ptr(d[n]) for n in names1 + names3)))
        return d

    def maps(self):
        K, Nfp = self.K_local, self.Nfp
        EToE = np.empty((K, 3), dtype=np.int32)
        EToF = np.empty((K, 3), dtype=np.int8)
        vmapM = np.empty((K, 3, Nfp), dtype=np.int64)
        vmapP = np.empty((K, 3, Nfp), dtype=np.int64)
        _check(_lib.dg_get_maps(self._h, *(_ptr(x) for x in (EToE, EToF, vmapM, vmapP))))
        return dict(EToE=EToE, EToF=EToF, vmapM=vmapM, vmapP=vmapP)

    def nodes(self):
        x = np.empty((self.K_local, self.Np))
        y = np.empty((self.K_local, self.Np))
        _check(_lib.dg_get_nodes(self._h, _ptr(x), _ptr(y)))
        return x, y

    def halo(self):
        nn, ns, nr = C.c_int32(), C.c_int64(), C.c_int64()
        _check(_lib.dg_halo_sizes(self._h, C.byref(nn), C.byref(ns), C.byref(nr)))
        nbr = np.empty(nn.value, dtype=np.int32)
        so = np.empty(nn.value + 1, dtype=np.int64)
        ro = np.empty(nn.value + 1, dtype=np.int64)
        sg = np.empty(ns.value, dtype=np.int64)
        rg = np.empty(nr.value, dtype=np.int64)
        rp = np.empty(nr.value, dtype=np.int64)
        _check(_lib.dg_get_halo(self._h, *(_ptr(x) for x in (nbr, so, sg, ro, rg, rp))))
        return dict(nbr=nbr, send_off=so, send_gdof=sg, recv_off=ro, recv_gdof=rg, recv_point=rp)

    # -- measurement
    def stream(self):
        s = C.c_void_p()
        _check(_lib.dg_stream(self._h, C.byref(s)))
        return s.value

    def set_graphs(self, enable=True):
        """dg_set_graphs: replay dg_run's steps as CUDA graphs (default on)."""
        _check(_lib.dg_set_graphs(self._h, 1 if enable else 0))

    def profile(self, enable=True):
        _check(_lib.dg_profile(self._h, 1 if enable else 0))

    def kernel_config(self):
        """dg_get_kernel_config: the compiled stage-kernel configuration of this (N, precision)."""
        k = KernelConfig()
        _check(_lib.dg_get_kernel_config(self._h, C.byref(k)))
        return dict(contraction=CONTRACTION[k.contraction], threads=k.threads, slots=k.slots,
                    residual_tma=bool(k.residual_tma), teams_cap=k.teams_cap, smem_bytes=k.smem_bytes,
                    flux_first=bool(k.flags & 1), ops_global=bool(k.flags & 2),
                    flux_in_fragments=bool(k.flags & 4), pass_interleave=bool(k.flags & 8),
                    compressed_connectivity=bool(k.flags & 16), compressed_geometry=bool(k.flags & 48),
                    w_precomputed=bool(k.flags & 64), dmma_units=bool(k.flags & 128),
                    warp_specialised=bool(k.flags & 256))

    def kernel_stats(self):
        st = KernelStats()
        _check(_lib.dg_get_kernel_stats(self._h, C.byref(st)))
        return {k: dict(launches=st.launches[i], ms=st.ms[i], timed=st.timed[i]) for i, k in enumerate(KIND)}


def dg_setup(N, VX, VY, EToV, eps=None, mu=None, bctag=None, precision=8, device=0, alpha=1.0,
             rank=0, nranks=1, fused=True, transport=0, nccl_id=None, part=None, stream=None,
             max_ctas=0, tile_order=0, check_every=0, kernel_variant=0):
    """dg_setup: build a context for ``rank`` of ``nranks`` on the GLOBAL mesh (VX, VY, EToV)."""
    VX = _as(VX, np.float64)
    VY = _as(VY, np.float64)
    EToV = _as(EToV, np.int64)
    K = EToV.shape[0]
    if EToV.shape != (K, 3) or VX.shape != VY.shape:
        raise ValueError("bad mesh arrays")
    eps_a = None if eps is None else _as(eps, np.float64, K)
    mu_a = None if mu is None else _as(mu, np.float64, K)
    bc_a = None if bctag is None else _as(bctag, np.int8, 3 * K)
    part_a = None if part is None else _as(part, np.int32, K)
    o = dg_options_default()
    o.N, o.precision, o.device, o.alpha = int(N), int(precision), int(device), float(alpha)
    o.rank, o.nranks, o.fused, o.transport = int(rank), int(nranks), 1 if fused else 0, int(transport)
    idbuf = None
    if nccl_id is not None:
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        o.nccl_id = C.cast(idbuf, C.c_void_p)
    o.part = _ptr(part_a)
    o.stream = stream
    o.max_ctas, o.tile_order, o.check_every = int(max_ctas), int(tile_order), int(check_every)
    o.kernel_variant = {"tuned": 0, "tcgen05": 1}.get(kernel_variant, kernel_variant)
    h = C.c_void_p()
    _check(_lib.dg_setup(C.byref(o), VX.size, _ptr(VX), _ptr(VY), K, _ptr(EToV), _ptr(eps_a), _ptr(mu_a),
                         _ptr(bc_a), C.byref(h)))
    return Context(h.value, int(N), int(precision))


def dg_run_group(ctxs, dt, nsteps):
    """dg_run_group: advance in-process partitions (transport=1) in lock step on one device."""
    arr = (C.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
    _check(_lib.dg_run_group(arr, len(ctxs), float(dt), int(nsteps)))


def nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (rank 0 calls this and broadcasts the bytes)."""
    h = None
    for name in ("libnccl.so.2", "libnccl.so"):
        try:
            h = C.CDLL(name, mode=C.RTLD_GLOBAL)
            break
        except OSError:
            continue
    if h is None:
        raise DGError(8, "libnccl not found")
    buf = C.create_string_buffer(128)
    st = h.ncclGetUniqueId(buf)
    if st != 0:
        raise DGError(8, f"ncclGetUniqueId failed ({st})")
    return buf.raw
