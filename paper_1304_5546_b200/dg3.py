"""Thin ctypes binding of the 3D C ABI in include/dg3.h (argument marshalling only; SURVEY.md §8(f)
row 4).  Every step runs in libdg.so's CUDA kernels; no Python or CPU compute path exists.

``dg3_setup`` returns a :class:`Context3` whose methods are the remaining ``dg3_*`` calls without the
prefix.  Fields are the 6-tuple (Hx, Hy, Hz, Ex, Ey, Ez), each [K][Np] fp64.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import dg as _dg

_lib = _dg._lib
_vp = C.c_void_p
_i64 = C.c_int64
_P = C.POINTER
EXPORTS3 = ["dg3_setup", "dg3_sizes", "dg3_set_fields", "dg3_get_fields", "dg3_run", "dg3_sync", "dg3_eval_rhs",
            "dg3_energy", "dg3_get_operators", "dg3_get_maps", "dg3_get_nodes", "dg3_get_geometry", "dg3_stream",
            "dg3_profile", "dg3_get_kernel_stats", "dg3_destroy"]
MAX_KERNEL_N3 = 5
_sig = {
    "dg3_setup": [_vp, _i64, _vp, _vp, _vp, _i64, _vp, _P(_vp)],
    "dg3_sizes": [_vp] * 5,
    "dg3_set_fields": [_vp, _vp],
    "dg3_get_fields": [_vp, _vp],
    "dg3_run": [_vp, C.c_double, _i64],
    "dg3_sync": [_vp],
    "dg3_eval_rhs": [_vp, C.c_int32, _vp],
    "dg3_energy": [_vp, _vp],
    "dg3_get_operators": [_vp] * 9,
    "dg3_get_maps": [_vp] * 4,
    "dg3_get_nodes": [_vp] * 4,
    "dg3_get_geometry": [_vp] * 8,
    "dg3_stream": [_vp, _P(_vp)],
    "dg3_profile": [_vp, C.c_int32],
    "dg3_get_kernel_stats": [_vp, _vp],
}
for _name, _args in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
_lib.dg3_destroy.argtypes = [_vp]
_lib.dg3_destroy.restype = None
_check = _dg._check
_ptr = _dg._ptr


def _six(arrays, n, writable=False):
    """Six fp64 C-contiguous buffers of n values each -> (kept arrays, void*[6])."""
    if len(arrays) != 6:
        raise ValueError("six fields (Hx, Hy, Hz, Ex, Ey, Ez)")
    keep = []
    for a in arrays:
        if isinstance(a, np.ndarray):
            if writable:
                if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or a.size != n:
                    raise ValueError(f"output arrays must be C-contiguous float64 of {n} values")
            else:
                a = _dg._as(a, np.float64, n)
        elif str(getattr(a, "dtype", "")) != "torch.float64" or not a.is_contiguous() or a.numel() != n:
            raise ValueError(f"field tensors must be contiguous torch.float64 of {n} values")
        keep.append(a)
    arr = (C.c_void_p * 6)(*[_ptr(a) for a in keep])
    return keep, arr


class Context3:
    def __init__(self, handle, N, precision):
        self._h = handle
        self.N, self.precision = N, precision
        np_, nfp, k, nsw = (C.c_int64() for _ in range(4))
        _check(_lib.dg3_sizes(self._h, C.byref(np_), C.byref(nfp), C.byref(k), C.byref(nsw)))
        self.Np, self.Nfp, self.K, self.n_swapped = np_.value, nfp.value, k.value, nsw.value

    def destroy(self):
        if self._h:
            _lib.dg3_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def _out(self):
        return tuple(np.empty((self.K, self.Np)) for _ in range(6))

    def set_fields(self, *fields):
        keep, arr = _six(fields, self.K * self.Np)
        _check(_lib.dg3_set_fields(self._h, arr))

    def get_fields(self, out=None):
        out = self._out() if out is None else out
        keep, arr = _six(out, self.K * self.Np, writable=True)
        _check(_lib.dg3_get_fields(self._h, arr))
        return out

    def run(self, dt, nsteps):
        _check(_lib.dg3_run(self._h, float(dt), int(nsteps)))

    def sync(self):
        _check(_lib.dg3_sync(self._h))

    def eval_rhs(self, which=0):
        which = {"full": 0, "volume": 1, "surface": 2}.get(which, which)
        out = self._out()
        keep, arr = _six(out, self.K * self.Np, writable=True)
        _check(_lib.dg3_eval_rhs(self._h, int(which), arr))
        return out

    def energy(self):
        e = C.c_double()
        _check(_lib.dg3_energy(self._h, C.byref(e)))
        return e.value

    def operators(self):
        Np, NF = self.Np, 4 * self.Nfp
        d = dict(r=np.empty(Np), s=np.empty(Np), t=np.empty(Np), Dr=np.empty((Np, Np)), Ds=np.empty((Np, Np)),
                 Dt=np.empty((Np, Np)), LIFT=np.empty((Np, NF)), Fmask=np.empty((4, self.Nfp), dtype=np.int32))
        _check(_lib.dg3_get_operators(self._h, *(_ptr(d[k]) for k in ("r", "s", "t", "Dr", "Ds", "Dt", "LIFT", "Fmask"))))
        return d

    def maps(self):
        K = self.K
        d = dict(EToE=np.empty((K, 4), dtype=np.int32), EToF=np.empty((K, 4), dtype=np.int8),
                 vmapP=np.empty((K, 4, self.Nfp), dtype=np.int64))
        _check(_lib.dg3_get_maps(self._h, _ptr(d["EToE"]), _ptr(d["EToF"]), _ptr(d["vmapP"])))
        return d

    def nodes(self):
        x, y, z = (np.empty((self.K, self.Np)) for _ in range(3))
        _check(_lib.dg3_get_nodes(self._h, _ptr(x), _ptr(y), _ptr(z)))
        return x, y, z

    def geometry(self):
        K = self.K
        d = dict(gfac=np.empty((K, 9)), J=np.empty(K), nx=np.empty((K, 4)), ny=np.empty((K, 4)),
                 nz=np.empty((K, 4)), sJ=np.empty((K, 4)), Fsc=np.empty((K, 4)))
        _check(_lib.dg3_get_geometry(self._h, *(_ptr(d[k]) for k in ("gfac", "J", "nx", "ny", "nz", "sJ", "Fsc"))))
        return d

    def stream(self):
        s = C.c_void_p()
        _check(_lib.dg3_stream(self._h, C.byref(s)))
        return s.value

    def profile(self, enable=True):
        _check(_lib.dg3_profile(self._h, 1 if enable else 0))

    def kernel_stats(self):
        st = _dg.KernelStats()
        _check(_lib.dg3_get_kernel_stats(self._h, C.byref(st)))
        return {k: dict(launches=st.launches[i], ms=st.ms[i], timed=st.timed[i]) for i, k in enumerate(_dg.KIND)}


def dg3_setup(N, VX, VY, VZ, EToV, precision=8, device=0, alpha=1.0, stream=None, max_ctas=0, fused=True):
    """dg3_setup: a single-GPU 3D context on the tetrahedral mesh (VX, VY, VZ, EToV [K][4]);
    fused: one fused stage kernel per LSERK4 stage where compiled, else volume + surface kernels."""
    VX, VY, VZ = (_dg._as(a, np.float64) for a in (VX, VY, VZ))
    EToV = _dg._as(EToV, np.int64)
    K = EToV.shape[0]
    if EToV.shape != (K, 4) or not (VX.shape == VY.shape == VZ.shape):
        raise ValueError("bad 3D mesh arrays")
    o = _dg.dg_options_default()
    o.N, o.precision, o.device, o.alpha = int(N), int(precision), int(device), float(alpha)
    o.stream = stream
    o.max_ctas = int(max_ctas)
    o.fused = 1 if fused else 0
    h = C.c_void_p()
    _check(_lib.dg3_setup(C.byref(o), VX.size, _ptr(VX), _ptr(VY), _ptr(VZ), K, _ptr(EToV), C.byref(h)))
    return Context3(h.value, int(N), int(precision))
