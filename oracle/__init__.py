"""Python binding of the CPU oracle (oracle/oracle.h) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
leg import this module.  It is the parity checker, never the product path.
The oracle restates the reference solve path (SerialBackend + templates,
ParallelBackend over in-process ranks); see oracle.h for the file:line map.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = _HERE / "_build" / "liboracle.so"
_lib = None

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


def _load():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            from paper_1804_02539_b200 import build
            build.build_oracle()
        lib = C.CDLL(str(_LIB))
        from paper_1804_02539_b200._native import PmgHierarchyDesc
        lib.oracle_create.argtypes = [C.POINTER(PmgHierarchyDesc), C.POINTER(_vp)]
        lib.oracle_create.restype = C.c_int
        lib.oracle_destroy.argtypes = [_vp]
        lib.oracle_destroy.restype = None
        lib.oracle_last_error.restype = C.c_char_p
        lib.oracle_num_dofs.argtypes = [_vp, C.c_int]
        lib.oracle_num_dofs.restype = C.c_int64
        for name, args in [
            ("oracle_apply_op", [_vp, C.c_int, _dp, _dp]),
            ("oracle_residual", [_vp, C.c_int, _dp, _dp, _dp]),
            ("oracle_smooth", [_vp, C.c_int, _dp, _dp]),
            ("oracle_restrict", [_vp, C.c_int, _dp, _dp]),
            ("oracle_add_prolonged", [_vp, C.c_int, _dp, C.c_double, _dp]),
            ("oracle_coarse_solve", [_vp, _dp, _dp]),
            ("oracle_set_coarse_mode", [_vp, C.c_int]),
            ("oracle_mg_cycle", [_vp, C.c_int, _dp, _dp]),
            ("oracle_precondition", [_vp, _dp, _dp]),
            ("oracle_pcg_solve", [_vp, _dp, C.c_double, C.c_int, C.c_int, _dp, _dp, C.POINTER(C.c_int), _dp]),
            ("oracle_parallel_pcg_solve", [_vp, C.c_int, _dp, C.c_double, C.c_int, C.c_int, _dp, _dp,
                                           C.POINTER(C.c_int), _dp, C.POINTER(C.c_uint64)]),
        ]:
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Oracle:
    """SerialBackend semantics on global dof vectors of a Hierarchy."""

    def __init__(self, hierarchy):
        self.h = hierarchy  # keeps the descriptor's memory alive
        lib = _load()
        ctx = C.c_void_p()
        self._check(lib.oracle_create(C.byref(hierarchy.desc), C.byref(ctx)))
        self._ctx = ctx

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, _load().oracle_last_error().decode())

    def __del__(self):
        try:
            if self._ctx:
                _load().oracle_destroy(self._ctx)
        except Exception:
            pass

    def n(self, level):
        return int(_load().oracle_num_dofs(self._ctx, level))

    def _vec(self, x, n):
        x = np.ascontiguousarray(x, dtype=np.float64)
        assert x.size == n, (x.size, n)
        return x

    def apply_op(self, level, u):
        out = np.empty(self.n(level))
        self._check(_load().oracle_apply_op(self._ctx, level, _p(self._vec(u, self.n(level))), _p(out)))
        return out

    def residual(self, level, f, u):
        out = np.empty(self.n(level))
        self._check(_load().oracle_residual(self._ctx, level, _p(self._vec(f, self.n(level))),
                                            _p(self._vec(u, self.n(level))), _p(out)))
        return out

    def smooth(self, level, r):
        out = np.empty(self.n(level))
        self._check(_load().oracle_smooth(self._ctx, level, _p(self._vec(r, self.n(level))), _p(out)))
        return out

    def restrict(self, level, r):
        out = np.empty(self.n(level - 1))
        self._check(_load().oracle_restrict(self._ctx, level, _p(self._vec(r, self.n(level))), _p(out)))
        return out

    def add_prolonged(self, level, coarse, c, u):
        u = self._vec(u, self.n(level)).copy()
        self._check(_load().oracle_add_prolonged(self._ctx, level, _p(self._vec(coarse, self.n(level - 1))), c, _p(u)))
        return u

    def set_coarse_mode(self, mode: int):
        """0: dense LLT substitution (default); 1: explicit inverse GEMV."""
        self._check(_load().oracle_set_coarse_mode(self._ctx, mode))

    def coarse_solve(self, r):
        out = np.empty(self.n(0))
        self._check(_load().oracle_coarse_solve(self._ctx, _p(self._vec(r, self.n(0))), _p(out)))
        return out

    def mg_cycle(self, level, u, f):
        u = self._vec(u, self.n(level)).copy()
        self._check(_load().oracle_mg_cycle(self._ctx, level, _p(u), _p(self._vec(f, self.n(level)))))
        return u

    def precondition(self, r):
        L = self.h.finest_level
        z = np.empty(self.n(L))
        self._check(_load().oracle_precondition(self._ctx, _p(self._vec(r, self.n(L))), _p(z)))
        return z

    def pcg_solve(self, f, tol=1e-8, max_iter=500, allow_cap=False, ranks=0):
        """ranks == 0: SerialBackend pcg_solve; ranks >= 1: parallel_pcg_solve
        over that many in-process ranks.  Returns (u, history, t_solve, comm_bytes)."""
        L = self.h.finest_level
        f = self._vec(f, self.n(L))
        u = np.empty(self.n(L))
        hist = np.zeros(max_iter + 1)
        it = C.c_int(0)
        ts = C.c_double(0.0)
        lib = _load()
        if ranks == 0:
            self._check(lib.oracle_pcg_solve(self._ctx, _p(f), tol, max_iter, 1 if allow_cap else 0, _p(u), _p(hist),
                                             C.byref(it), C.byref(ts)))
            return u, hist[: it.value + 1].copy(), ts.value, 0
        cb = C.c_uint64(0)
        self._check(lib.oracle_parallel_pcg_solve(self._ctx, ranks, _p(f), tol, max_iter, 1 if allow_cap else 0, _p(u),
                                                  _p(hist), C.byref(it), C.byref(ts), C.byref(cb)))
        return u, hist[: it.value + 1].copy(), ts.value, cb.value
