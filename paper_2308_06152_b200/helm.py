"""Thin ctypes binding of libhelm.so (include/helm.h).  Argument marshalling only: every
step of the hot path runs in the CUDA kernels of the library.  Fields are torch
complex128 CUDA tensors of shape (ny, nx) (row-major, x contiguous); PyTorch provides
device memory and streams, nothing else.  There is no CPU fallback: if the library or a
CUDA device is missing, construction raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("HELM_LIB") or os.path.join(_HERE, "libhelm.so")

HELM_BC_DIRICHLET = 0
HELM_BC_SOMMERFELD = 1
COARSE_OPS = {"galerkin": 0, "red_o2": 1, "red_o4": 2, "red_glk1": 3, "red_glk2": 4, "red_o6": 5, "red_cmpo4": 6, "red_9pto2": 7}
VECTORS = {"bilinear": 0, "high_order": 1}
OUTER = {"fgmres": 0, "gcr": 1}
PRECOND = {"adef1": 0, "tlkm": 1}
BCS = {"dirichlet": HELM_BC_DIRICHLET, "sommerfeld": HELM_BC_SOMMERFELD}


class helm_grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("h", ctypes.c_double), ("bc", ctypes.c_int)]


class helm_params(ctypes.Structure):
    _fields_ = [("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("omega", ctypes.c_double),
                ("nu_pre", ctypes.c_int), ("nu_post", ctypes.c_int), ("coarse_op", ctypes.c_int),
                ("inner_tol", ctypes.c_double), ("inner_maxit", ctypes.c_int), ("max_levels", ctypes.c_int),
                ("restart", ctypes.c_int), ("max_coarsest", ctypes.c_int), ("vectors", ctypes.c_int),
                ("graph", ctypes.c_int), ("tail_max_n", ctypes.c_int), ("pdl", ctypes.c_int),
                ("coarsest_n", ctypes.c_int), ("coop", ctypes.c_int), ("outer", ctypes.c_int),
                ("col_min_n", ctypes.c_int), ("dist_levels", ctypes.c_int), ("dist_min_rows", ctypes.c_int),
                ("col_pipe", ctypes.c_int), ("fuse_dots", ctypes.c_int), ("precond", ctypes.c_int),
                ("gamma", ctypes.c_double), ("tail_cluster", ctypes.c_int),
                ("lag_stepb", ctypes.c_int), ("dots_cluster", ctypes.c_int), ("inner_restart", ctypes.c_int),
                ("e_stream", ctypes.c_int), ("tma", ctypes.c_int), ("sstep", ctypes.c_int),
                ("sstep_passes", ctypes.c_int), ("sstep_shift", ctypes.c_double)]


class helm_dist(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
                ("group", ctypes.c_void_p), ("nccl_id", ctypes.c_void_p),
                ("flags", ctypes.c_int)]


HELM_COMM_THREADS = 0
HELM_COMM_NCCL = 1
HELM_COMM_PEER = 2
HELM_DIST_EXCHANGE_AT_ONE_RANK = 1


class helm_report(ctypes.Structure):
    _fields_ = [("outer_iterations", ctypes.c_int), ("converged", ctypes.c_int), ("relres", ctypes.c_double),
                ("inner_solves", ctypes.c_int), ("inner_iterations_total", ctypes.c_longlong),
                ("inner_iterations_max", ctypes.c_int), ("restarts", ctypes.c_int), ("seconds", ctypes.c_double),
                ("kernels", ctypes.c_longlong), ("inner_restarts", ctypes.c_longlong)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
EXPORTS = {
    "helm_default_params": (None, [ctypes.POINTER(helm_params)]),
    "helm_setup": (_I, [ctypes.POINTER(_P), ctypes.POINTER(helm_grid), _P, _I, ctypes.POINTER(helm_params), _P]),
    "helm_destroy": (None, [_P]),
    "helm_num_levels": (_I, [_P]),
    "helm_level_info": (_I, [_P, _I, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_D)]),
    "helm_apply_A": (_I, [_P, _P, _P]),
    "helm_apply_M": (_I, [_P, _I, _P, _P]),
    "helm_restrict": (_I, [_P, _I, _P, _P]),
    "helm_prolong": (_I, [_P, _I, _P, _P]),
    "helm_apply_E": (_I, [_P, _P, _P]),
    "helm_apply_Zt": (_I, [_P, _P, _P]),
    "helm_apply_Z": (_I, [_P, _P, _P]),
    "helm_vcycle": (_I, [_P, _I, _P, _P]),
    "helm_deflate": (_I, [_P, _P, _P, ctypes.POINTER(_I)]),
    "helm_solve": (_I, [_P, _P, _P, _D, _I, ctypes.POINTER(helm_report)]),
    "helm_solve_host": (_I, [_P, _P, _P, _D, _I, ctypes.POINTER(helm_report)]),
    "helm_flush_l2": (_I, [_P, ctypes.c_size_t]),
    "helm_launch_count": (ctypes.c_longlong, [_P]),
    "helm_bench_kernel": (_I, [_P, _I, _I, _I, _I, ctypes.POINTER(_D), ctypes.POINTER(_D)]),
    "helm_bench_graph": (_I, [_P, _I, _I, _I, ctypes.POINTER(_D)]),
    "helm_group_create": (_I, [_I, ctypes.POINTER(_P)]),
    "helm_group_destroy": (None, [_P]),
    "helm_nccl_unique_id": (_I, [ctypes.c_char_p]),
    "helm_setup_dist": (_I, [ctypes.POINTER(_P), ctypes.POINTER(helm_grid), _P, _I, ctypes.POINTER(helm_params), _P,
                             ctypes.POINTER(helm_dist)]),
    "helm_dist_rows": (_I, [_P, _I, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "helm_peer_handle": (_I, [_P, ctypes.c_char_p]),
    "helm_peer_connect": (_I, [_P, ctypes.c_char_p]),
    "helm_peer_error": (_I, [_P]),
    "helm_peer_layout": (_I, [ctypes.POINTER(helm_grid), ctypes.POINTER(helm_params), _I,
                              ctypes.POINTER(ctypes.c_size_t), _I]),
    "helm_dist_plan": (_I, [ctypes.POINTER(helm_grid), ctypes.POINTER(helm_params), _I, ctypes.POINTER(_I),
                            ctypes.POINTER(_I), _I]),
    "helm_last_error": (ctypes.c_char_p, []),
    "helm_build_info": (ctypes.c_char_p, []),
}

_lib = None


def load_library(path: str = _LIB_PATH):
    """Load libhelm.so and bind every symbol of include/helm.h (raises if any is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class HelmError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise HelmError(f"libhelm error {rc}: {_lib.helm_last_error().decode()}")


def default_params(**overrides) -> helm_params:
    lib = load_library()
    p = helm_params()
    lib.helm_default_params(ctypes.byref(p))
    for key, val in overrides.items():
        if key == "coarse_op" and isinstance(val, str):
            val = COARSE_OPS[val]
        if key == "vectors" and isinstance(val, str):
            val = VECTORS[val]
        if key == "outer" and isinstance(val, str):
            val = OUTER[val]
        if key == "precond" and isinstance(val, str):
            val = PRECOND[val]
        if key == "beta":
            p.beta1, p.beta2 = val
            continue
        if not hasattr(p, key):
            raise KeyError(key)
        setattr(p, key, val)
    return p


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class Helm:
    """One solver context (helm_setup ... helm_destroy)."""

    def __init__(self, nx: int, ny: int, h: float, bc: str, k, params: helm_params | dict | None = None,
                 stream=None):
        import torch
        self.torch = torch
        lib = load_library()
        if not torch.cuda.is_available():
            raise HelmError("no CUDA device: libhelm has no CPU fallback")
        self.lib = lib
        self.nx, self.ny, self.h, self.bc = int(nx), int(ny), float(h), bc
        if isinstance(params, dict) or params is None:
            params = default_params(**(params or {}))
        self.params = params
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        kt = torch.as_tensor(np.ascontiguousarray(k, dtype=np.float64)) if not isinstance(k, torch.Tensor) else k
        kt = kt.to(device="cuda", dtype=torch.float64).contiguous()
        assert kt.shape == (self.ny, self.nx)
        g = helm_grid(self.nx, self.ny, self.h, BCS[bc])
        ctx = ctypes.c_void_p()
        _check(lib.helm_setup(ctypes.byref(ctx), ctypes.byref(g), _ptr(kt), 1, ctypes.byref(params),
                              ctypes.c_void_p(self.stream.cuda_stream)))
        self.ctx = ctx
        self.levels = [self.level_info(l) for l in range(lib.helm_num_levels(ctx))]

    # -- helpers --------------------------------------------------------------------
    def level_info(self, l):
        nx, ny, h = _I(), _I(), _D()
        _check(self.lib.helm_level_info(self.ctx, l, ctypes.byref(nx), ctypes.byref(ny), ctypes.byref(h)))
        return (ny.value, nx.value, h.value)

    def field(self, level=0):
        ny, nx, _ = self.levels[level]
        return self.torch.zeros((ny, nx), dtype=self.torch.complex128, device="cuda")

    def _in(self, x, level=0):
        t = self.torch
        x = t.as_tensor(x).to(device="cuda", dtype=t.complex128).contiguous()
        assert tuple(x.shape) == self.levels[level][:2], (x.shape, self.levels[level])
        return x

    # -- the C ABI, one method per entry point -----------------------------------------
    def helm_apply_A(self, x, y=None):
        x = self._in(x)
        y = self.field(0) if y is None else y
        _check(self.lib.helm_apply_A(self.ctx, _ptr(x), _ptr(y)))
        return y

    def helm_apply_M(self, level, x, y=None):
        x = self._in(x, level)
        y = self.field(level) if y is None else y
        _check(self.lib.helm_apply_M(self.ctx, level, _ptr(x), _ptr(y)))
        return y

    def helm_restrict(self, level, v):
        v = self._in(v, level)
        y = self.field(level + 1)
        _check(self.lib.helm_restrict(self.ctx, level, _ptr(v), _ptr(y)))
        return y

    def helm_prolong(self, level, e):
        e = self._in(e, level + 1)
        y = self.field(level)
        _check(self.lib.helm_prolong(self.ctx, level, _ptr(e), _ptr(y)))
        return y

    def helm_apply_Zt(self, v):
        v = self._in(v, 0)
        y = self.field(1)
        _check(self.lib.helm_apply_Zt(self.ctx, _ptr(v), _ptr(y)))
        return y

    def helm_apply_Z(self, e):
        e = self._in(e, 1)
        y = self.field(0)
        _check(self.lib.helm_apply_Z(self.ctx, _ptr(e), _ptr(y)))
        return y

    def helm_apply_E(self, x):
        x = self._in(x, 1)
        y = self.field(1)
        _check(self.lib.helm_apply_E(self.ctx, _ptr(x), _ptr(y)))
        return y

    def helm_vcycle(self, level, f, u=None):
        f = self._in(f, level)
        u = self.field(level) if u is None else u
        _check(self.lib.helm_vcycle(self.ctx, level, _ptr(f), _ptr(u)))
        return u

    def helm_deflate(self, v, z=None):
        v = self._in(v)
        z = self.field(0) if z is None else z
        its = _I()
        _check(self.lib.helm_deflate(self.ctx, _ptr(v), _ptr(z), ctypes.byref(its)))
        return z, its.value

    def helm_solve(self, b, tol=1e-6, maxit=600, x=None):
        b = self._in(b)
        x = self.field(0) if x is None else x
        rep = helm_report()
        _check(self.lib.helm_solve(self.ctx, _ptr(b), _ptr(x), float(tol), int(maxit), ctypes.byref(rep)))
        return x, rep.as_dict()

    def helm_solve_host(self, b_host: np.ndarray, x_host: np.ndarray | None = None, tol=1e-6, maxit=600):
        """End-to-end: b and x are host (numpy complex128, ideally pinned) arrays."""
        b_host = np.ascontiguousarray(b_host, dtype=np.complex128)
        x_host = np.empty_like(b_host) if x_host is None else x_host
        rep = helm_report()
        _check(self.lib.helm_solve_host(self.ctx, b_host.ctypes.data_as(_P), x_host.ctypes.data_as(_P),
                                        float(tol), int(maxit), ctypes.byref(rep)))
        return x_host, rep.as_dict()

    def helm_flush_l2(self, nbytes=256 << 20):
        _check(self.lib.helm_flush_l2(self.ctx, nbytes))

    KERNELS = {"apply_A": 0, "vc_down": 1, "vc_up": 2, "apply_E": 3, "gs_dots": 4, "gs_update": 5}

    def helm_bench_kernel(self, which, arg=1, reps=20, flush=True):
        """(mean us per launch, algorithmic bytes per launch) of one kernel at this context's sizes."""
        us, nb = _D(), _D()
        _check(self.lib.helm_bench_kernel(self.ctx, self.KERNELS.get(which, which), int(arg), int(reps), int(flush),
                                          ctypes.byref(us), ctypes.byref(nb)))
        return us.value, nb.value

    REGIONS = {"vcycle": 0, "apply_E": 1, "apply_A": 2, "dcgs": 3, "inner_iter": 4, "e_dots": 5, "dcgs_reduce": 6,
               "dcgs_update": 7, "dcgs_dots": 8, "vc_down": 9, "vc_up": 10, "ss_dots": 11, "ss_reduce": 12,
               "ss_update": 13, "ss_power": 14, "ss_e": 15, "outer_dcgs": 16}

    def helm_bench_graph(self, which, arg=0, reps=50):
        """Mean in-graph device time (us) of one instance of a region (warm, back-to-back)."""
        us = _D()
        _check(self.lib.helm_bench_graph(self.ctx, self.REGIONS.get(which, which), int(arg), int(reps),
                                         ctypes.byref(us)))
        return us.value

    def helm_launch_count(self):
        return int(self.lib.helm_launch_count(self.ctx))

    # short aliases
    apply_A = helm_apply_A
    apply_M = helm_apply_M
    restrict = helm_restrict
    prolong = helm_prolong
    apply_E = helm_apply_E
    apply_Z = helm_apply_Z
    apply_Zt = helm_apply_Zt
    vcycle = helm_vcycle
    deflate = helm_deflate
    solve = helm_solve
    solve_host = helm_solve_host

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.helm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def helm_setup(problem, params=None, stream=None) -> Helm:
    """Build a context from a workloads.Problem-like object (k, h, bc, nx, ny)."""
    return Helm(problem.nx, problem.ny, problem.h, problem.bc, problem.k, params, stream)


# ---------------------------------------------------------------------- decomposed solves
def peer_layout(nx, ny, h, bc, nranks, params=None):
    """Host-only peer-arena layout (helm_peer_layout): [bytes, flags, red, gat, gat_n, up0, dn0, ...]."""
    lib = load_library()
    p = params if isinstance(params, helm_params) else default_params(**(params or {}))
    g = helm_grid(int(nx), int(ny), float(h), BCS[bc])
    out = (ctypes.c_size_t * 256)()
    n = lib.helm_peer_layout(ctypes.byref(g), ctypes.byref(p), int(nranks), out, 256)
    if n < 0:
        _check(n)
    return [int(out[i]) for i in range(n)]


def dist_plan(nx, ny, h, bc, nranks, params=None):
    """Host-only row-strip plan (helm_dist_plan): (D, table[l][q] = (a, b, s, e))."""
    lib = load_library()
    p = params if isinstance(params, helm_params) else default_params(**(params or {}))
    g = helm_grid(int(nx), int(ny), float(h), BCS[bc])
    cap = 64
    table = (_I * (cap * nranks * 4))()
    D = _I()
    nl = lib.helm_dist_plan(ctypes.byref(g), ctypes.byref(p), int(nranks), ctypes.byref(D), table, cap)
    if nl < 0:
        _check(nl)
    rows = [[tuple(table[(l * nranks + q) * 4 + i] for i in range(4)) for q in range(nranks)] for l in range(nl)]
    return D.value, rows


class ThreadGroup:
    """helm_group_create: nranks ranks living as host threads of this process (one device)."""

    def __init__(self, nranks):
        lib = load_library()
        self.lib = lib
        self.nranks = int(nranks)
        g = ctypes.c_void_p()
        _check(lib.helm_group_create(self.nranks, ctypes.byref(g)))
        self.handle = g

    def close(self):
        if getattr(self, "handle", None):
            self.lib.helm_group_destroy(self.handle)
            self.handle = None


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.helm_nccl_unique_id(buf))
    return buf.raw


class HelmDist(Helm):
    """One rank of a row-strip decomposed solver (helm_setup_dist).  Level-0 fields passed to
    and returned by the entry points are this rank's owned rows, shape (nrows, nx)."""

    def __init__(self, nx, ny, h, bc, k, rank, nranks, group: ThreadGroup | None = None, nccl_id: bytes | None = None,
                 params=None, stream=None, peer_exchange=None, exchange_at_one_rank=False):
        """Transport: a ThreadGroup (ranks as threads on one GPU), an NCCL unique id, or
        peer_exchange = callable(bytes) -> list of every rank's bytes (e.g. through
        torch.distributed.all_gather_object) for the NVLink peer-memory transport.
        exchange_at_one_rank: with the peer transport and nranks == 1, run the exchange kernels
        against the rank's own arena (HELM_DIST_EXCHANGE_AT_ONE_RANK; tests)."""
        import torch
        self.torch = torch
        lib = load_library()
        if not torch.cuda.is_available():
            raise HelmError("no CUDA device: libhelm has no CPU fallback")
        self.lib = lib
        self.nx, self.ny, self.h, self.bc = int(nx), int(ny), float(h), bc
        if isinstance(params, dict) or params is None:
            params = default_params(**(params or {}))
        self.params = params
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        kt = torch.as_tensor(np.ascontiguousarray(k, dtype=np.float64)) if not isinstance(k, torch.Tensor) else k
        kt = kt.to(device="cuda", dtype=torch.float64).contiguous()
        assert kt.shape == (self.ny, self.nx)
        g = helm_grid(self.nx, self.ny, self.h, BCS[bc])
        self._id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        kind = HELM_COMM_NCCL if nccl_id is not None else (HELM_COMM_PEER if peer_exchange is not None else
                                                           HELM_COMM_THREADS)
        d = helm_dist(kind, int(rank), int(nranks),
                      group.handle if group is not None else None,
                      ctypes.cast(self._id, ctypes.c_void_p) if self._id is not None else None,
                      HELM_DIST_EXCHANGE_AT_ONE_RANK if exchange_at_one_rank else 0)
        ctx = ctypes.c_void_p()
        _check(lib.helm_setup_dist(ctypes.byref(ctx), ctypes.byref(g), _ptr(kt), 1, ctypes.byref(params),
                                   ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(d)))
        self.ctx = ctx
        self.rank, self.nranks = int(rank), int(nranks)
        if kind == HELM_COMM_PEER:
            hbuf = ctypes.create_string_buffer(64)
            _check(lib.helm_peer_handle(ctx, hbuf))
            handles = peer_exchange(hbuf.raw)
            assert len(handles) == self.nranks and all(len(x) == 64 for x in handles)
            _check(lib.helm_peer_connect(ctx, b"".join(handles)))
        self.levels = [self.level_info(l) for l in range(lib.helm_num_levels(ctx))]
        self.row0, self.nrows = self.dist_rows(0)

    def dist_rows(self, level=0):
        r0, nr = _I(), _I()
        _check(self.lib.helm_dist_rows(self.ctx, int(level), ctypes.byref(r0), ctypes.byref(nr)))
        return r0.value, nr.value

    def field(self, level=0):
        assert level == 0
        return self.torch.zeros((self.nrows, self.nx), dtype=self.torch.complex128, device="cuda")

    def _in(self, x, level=0):
        t = self.torch
        assert level == 0
        x = t.as_tensor(x).to(device="cuda", dtype=t.complex128).contiguous()
        assert tuple(x.shape) == (self.nrows, self.nx), (x.shape, (self.nrows, self.nx))
        return x
