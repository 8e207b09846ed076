"""Thin Python binding of the C ABI in include/bnf.h (argument marshalling
only: every step of the hot path runs in libbnf.so's CUDA kernels).

The package deliberately has NO fallback: if libbnf.so is missing or fails
to load, importing this module raises.  Build it with
``python paper_1806_10284_b200/build.py`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbnf.so")

if not os.path.exists(LIB_PATH):
    raise ImportError("libbnf.so not built (%s); run python paper_1806_10284_b200/build.py" % LIB_PATH)
_lib = C.CDLL(LIB_PATH)

OK, EINVAL, EGEOM, ENOMEM, ECUDA, ENCCL, ENOCONV, ESTATE = range(8)
MEM_HOST, MEM_DEVICE = 0, 1
OP_AR, OP_M = 0, 1
VEC_Y, VEC_E, VEC_H = 0, 1, 2


class BnfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("bnf error %d: %s" % (code, msg))
        self.code = code


class LatticeInfo(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("perm", C.c_int * 3), ("sign3", C.c_int), ("m", C.c_int * 3),
                ("rho", C.c_int * 3), ("category", C.c_int), ("lengths", C.c_double * 3),
                ("cos_raw", C.c_double * 3), ("cos_snap", C.c_double * 3), ("a", C.c_double * 9),
                ("a_canon", C.c_double * 9), ("l", C.c_double * 3), ("delta", C.c_double * 3),
                ("Ag", C.c_longlong * 9)]


class Opts(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("tol_outer", C.c_double),
                ("tol_inner", C.c_double), ("max_outer", C.c_int), ("max_inner", C.c_int),
                ("block", C.c_int), ("guard", C.c_int), ("seed", C.c_ulonglong), ("refine", C.c_int),
                ("profile", C.c_int), ("warm", C.c_int), ("reorth_once_ok", C.c_int),
                ("res_tol", C.c_double), ("max_polish", C.c_int), ("slabs", C.c_int),
                ("relax_inner", C.c_int), ("method", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("outer_steps", C.c_int), ("converged", C.c_int), ("inner_iters", C.c_longlong),
                ("matvecs", C.c_longlong), ("kernel_launches", C.c_longlong),
                ("max_ritz_residual", C.c_double), ("max_residual", C.c_double), ("seconds", C.c_double),
                ("polish_steps", C.c_int), ("polish_failed", C.c_int),
                ("active_matvecs", C.c_longlong)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = C.c_void_p
_D3 = C.c_double * 3
_lib.bnf_last_error.restype = C.c_char_p
_lib.bnf_version.restype = C.c_int
_sigs = {
    "bnf_lattice_create": [C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(_P)],
    "bnf_lattice_query": [_P, C.POINTER(LatticeInfo)],
    "bnf_kvec_reduce": [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "bnf_kappa_canonical": [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "bnf_cg_solve": [_P, _P, _P, C.c_int, C.c_int, C.POINTER(C.c_int)],
    "bnf_yee_points": [_P, C.c_int, C.c_int, C.POINTER(C.c_double)],
    "bnf_solver_create": [_P, C.POINTER(Opts), C.POINTER(_P)],
    "bnf_nccl_unique_id": [C.c_char_p],
    "bnf_solver_create_dist": [_P, C.POINTER(Opts), C.c_int, C.c_int, C.c_char_p, C.POINTER(_P)],
    "bnf_set_epsilon": [_P, _P, C.c_int],
    "bnf_set_kappa": [_P, C.POINTER(C.c_double)],
    "bnf_apply_Ar": [_P, _P, _P, C.c_int, C.c_int],
    "bnf_solve": [_P, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double), C.POINTER(Stats)],
    "bnf_eigvecs": [_P, C.c_int, _P, C.c_int],
    "bnf_kernel_times": [_P, C.POINTER(C.c_char_p), C.POINTER(C.c_double), C.POINTER(C.c_longlong), C.c_int,
                         C.POINTER(C.c_int)],
    "bnf_kernel_times_reset": [_P],
    "bnf_set_profile": [_P, C.c_int],
    "bnf_phase_counters": [_P, _P, C.c_int],
    "bnf_host_herm_eig": [C.c_int, _P, _P, _P],
}
for _name, _args in _sigs.items():
    getattr(_lib, _name).argtypes = _args
    getattr(_lib, _name).restype = C.c_int
_lib.bnf_lattice_destroy.argtypes = [_P]
_lib.bnf_lattice_destroy.restype = None
_lib.bnf_solver_destroy.argtypes = [_P]
_lib.bnf_solver_destroy.restype = None
_lib.bnf_opts_default.argtypes = [C.POINTER(Opts)]
_lib.bnf_opts_default.restype = None

FRAME_SNAPPED, FRAME_ORIGINAL = 0, 1

EXPORTS = ["bnf_lattice_create", "bnf_lattice_query", "bnf_lattice_destroy", "bnf_kvec_reduce",
           "bnf_nccl_unique_id", "bnf_solver_create_dist",
           "bnf_kappa_canonical", "bnf_cg_solve", "bnf_yee_points",
           "bnf_opts_default", "bnf_solver_create", "bnf_solver_destroy", "bnf_set_epsilon", "bnf_set_kappa",
           "bnf_apply_Ar", "bnf_solve", "bnf_eigvecs", "bnf_kernel_times", "bnf_kernel_times_reset", "bnf_set_profile", "bnf_phase_counters",
           "bnf_last_error", "bnf_version", "bnf_host_herm_eig"]


def _check(rc, allow=()):
    if rc != OK and rc not in allow:
        raise BnfError(rc, _lib.bnf_last_error().decode())
    return rc


def version():
    return _lib.bnf_version()


def _ptr(x):
    """Device pointer of a torch tensor, or host pointer of a numpy array."""
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    return x.ctypes.data_as(C.c_void_p)


class Lattice:
    def __init__(self, a_raw, n):
        a = np.ascontiguousarray(np.asarray(a_raw, dtype=np.float64).T)   # columns -> a[3*l + r]
        nn = (C.c_int * 3)(*[int(v) for v in n])
        h = _P()
        _check(_lib.bnf_lattice_create(a.ctypes.data_as(C.POINTER(C.c_double)), nn, C.byref(h)))
        self._h = h
        info = LatticeInfo()
        _check(_lib.bnf_lattice_query(h, C.byref(info)))
        self.info = info
        self.n = tuple(info.n)
        self.nn = self.n[0] * self.n[1] * self.n[2]
        self.m = tuple(info.m)
        self.rho = tuple(info.rho)
        self.perm = tuple(info.perm)
        self.sign3 = info.sign3
        self.category = info.category
        self.delta = tuple(info.delta)
        self.l = tuple(info.l)
        self.cos = tuple(info.cos_snap)
        self.a = np.array(info.a).reshape(3, 3).T           # columns
        self.a_canon = np.array(info.a_canon).reshape(3, 3).T
        self.Ag = np.array(info.Ag, dtype=np.int64).reshape(3, 3).T

    def kvec_reduce(self, K):
        out = _D3()
        _check(_lib.bnf_kvec_reduce(self._h, _D3(*[float(x) for x in K]), out))
        return tuple(out)

    def yee_points(self, comp, frame=0):
        """(n, 3) float64 Yee points of component comp: frame 0 = snapped
        (transformed) frame, 1 = original frame (bnf_yee_points)."""
        out = np.empty((self.nn, 3), dtype=np.float64)
        _check(_lib.bnf_yee_points(self._h, int(comp), int(frame), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def kappa_from_raw(self, kappa_raw):
        out = _D3()
        _check(_lib.bnf_kappa_canonical(self._h, _D3(*[float(x) for x in kappa_raw]), out))
        return tuple(out)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.bnf_lattice_destroy(self._h)
            self._h = None


def nccl_unique_id():
    """NCCL unique id (128 bytes) for bnf_solver_create_dist; broadcast it to every rank."""
    buf = C.create_string_buffer(128)
    _check(_lib.bnf_nccl_unique_id(buf))
    return buf.raw


class Solver:
    def __init__(self, lattice: Lattice, device=0, stream=None, dist=None, **kw):
        """dist = (nranks, rank, nccl_id): distributed slab mode (bnf_solver_create_dist)."""
        o = Opts()
        _lib.bnf_opts_default(C.byref(o))
        o.device = int(device)
        o.stream = C.c_void_p(stream) if stream else None
        for k, v in kw.items():
            setattr(o, k, v)
        h = _P()
        if dist is not None:
            nranks, rank, uid = dist
            _check(_lib.bnf_solver_create_dist(lattice._h, C.byref(o), int(nranks), int(rank), bytes(uid), C.byref(h)))
        else:
            _check(_lib.bnf_solver_create(lattice._h, C.byref(o), C.byref(h)))
        self._h = h
        self.lattice = lattice
        self.n = lattice.nn
        self.opts = o

    def set_epsilon(self, eps):
        """eps: numpy (3n,) float64 (host) or a CUDA torch float64 tensor."""
        if hasattr(eps, "data_ptr"):
            assert eps.is_cuda and eps.numel() == 3 * self.n and eps.is_contiguous()
            _check(_lib.bnf_set_epsilon(self._h, C.c_void_p(eps.data_ptr()), MEM_DEVICE))
        else:
            e = np.ascontiguousarray(eps, dtype=np.float64).ravel()
            assert e.size == 3 * self.n
            _check(_lib.bnf_set_epsilon(self._h, e.ctypes.data_as(C.c_void_p), MEM_HOST))

    def set_kappa(self, kappa):
        _check(_lib.bnf_set_kappa(self._h, _D3(*[float(k) for k in kappa])))

    def apply_Ar(self, y, out, b, op=OP_AR):
        """y, out: CUDA complex128 torch tensors of b*2n elements."""
        _check(_lib.bnf_apply_Ar(self._h, _ptr(y), _ptr(out), int(b), int(op)))

    def cg_solve(self, c, x, b, max_iter):
        """x = M^{-1} c by the solver's CG (c, x: CUDA complex128 tensors of b*2n)."""
        it = C.c_int()
        _check(_lib.bnf_cg_solve(self._h, _ptr(c), _ptr(x), int(b), int(max_iter), C.byref(it)))
        return it.value

    def solve(self, kappa, nev, allow_noconv=False):
        lam = np.zeros(nev)
        st = Stats()
        rc = _check(_lib.bnf_solve(self._h, _D3(*[float(k) for k in kappa]), int(nev),
                                   lam.ctypes.data_as(C.POINTER(C.c_double)), C.byref(st)),
                    allow=(ENOCONV,) if allow_noconv else ())
        d = st.as_dict()
        d["rc"] = rc
        return lam, d

    def eigvecs(self, kind, out, nev=None):
        mem = MEM_DEVICE if hasattr(out, "data_ptr") else MEM_HOST
        _check(_lib.bnf_eigvecs(self._h, int(kind), _ptr(out), mem))
        return out

    def kernel_times(self, reset=False):
        cap = 64
        names = (C.c_char_p * cap)()
        ms = (C.c_double * cap)()
        cnt = (C.c_longlong * cap)()
        k = C.c_int()
        _check(_lib.bnf_kernel_times(self._h, names, ms, cnt, cap, C.byref(k)))
        out = {names[i].decode(): (ms[i], cnt[i]) for i in range(min(k.value, cap))}
        if reset:
            _check(_lib.bnf_kernel_times_reset(self._h))
        return out

    def set_profile(self, on):
        """Per-kernel CUDA-event timing on/off (off: CG loop as one CUDA graph)."""
        _check(_lib.bnf_set_profile(self._h, int(bool(on))))

    def phase_counters(self):
        """Plane-pass per-phase cycle sums (BNF_PHASE_PROF set at creation); resets them."""
        out = np.zeros(16, dtype=np.uint64)
        _check(_lib.bnf_phase_counters(self._h, out.ctypes.data_as(C.c_void_p), 16))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib.bnf_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def host_herm_eig(a):
    """Testing hook: the library's host Hermitian eigensolver."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    n = a.shape[0]
    w = np.zeros(n)
    z = np.zeros((n, n), dtype=np.complex128)
    _check(_lib.bnf_host_herm_eig(n, a.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p),
                                  z.ctypes.data_as(C.c_void_p)))
    return w, z
