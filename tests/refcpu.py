"""ctypes binding of the refcpu CPU oracle (oracle/build/librefcpu.so).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs use this as the checker / the reference CPU arm. The product
(paper_2101_11649_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "build", "librefcpu.so")
PINS = os.path.join(ORACLE_DIR, "build", "pins")

_I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_set_dot_order.argtypes = [C.c_int]
        L.ref_spmv.argtypes = [C.c_int, C.c_int, _I32P, _I32P, _F64P, _F64P, _F64P]
        L.ref_setup.argtypes = [C.c_int, _I32P, _I32P, _F64P, _I32P, C.c_int, C.POINTER(C.c_char_p),
                                vp, C.c_char_p, C.POINTER(vp)]
        L.ref_setup_seconds.argtypes = [vp]
        L.ref_setup_seconds.restype = C.c_double
        L.ref_apply.argtypes = [vp, _F64P, _F64P]
        L.ref_solve.argtypes = [vp, _F64P, _F64P, C.c_int, C.c_int, C.c_double, C.c_double,
                                C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double), _F64P,
                                C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_solve_op.argtypes = [vp, C.c_int, _I32P, _I32P, _F64P, _F64P, _F64P, C.c_int, C.c_int,
                                   C.c_double, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_double), _F64P, C.c_int, C.POINTER(C.c_int)]
        L.ref_dump.argtypes = [vp, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_int), C.POINTER(C.c_longlong), vp, vp, vp]
        L.ref_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]
        L.ref_free.argtypes = [vp]
        L.ref_amg_info.argtypes = [vp, C.c_int, C.POINTER(C.c_int), vp, C.c_int, C.POINTER(C.c_longlong),
                                   C.POINTER(C.c_int)]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _chk(code):
    if code in (0, 1):
        return code
    raise RefError(code, lib().ref_last_error().decode())


def set_threads(n: int):
    lib().ref_set_threads(n)


DOT_ORDERS = {"canonical": 0, "sequential": 1, "eigen_sse2": 2}


def set_dot_order(name: str):
    """Inner-product order of the oracle GMRES: "canonical" (the device's fixed
    592x256 tree), "sequential" (one accumulator, left to right) or
    "eigen_sse2" (Eigen's 2-packet SSE2 redux order, restated; unpinned)."""
    lib().ref_set_dot_order(DOT_ORDERS[name])


def spmv(ptr, col, val, x, ncols=None):
    ptr = np.ascontiguousarray(ptr, np.int32)
    n = ptr.size - 1
    y = np.empty(n)
    _chk(lib().ref_spmv(n, ncols or n, ptr, np.ascontiguousarray(col, np.int32),
                        np.ascontiguousarray(val, np.float64), np.ascontiguousarray(x, np.float64), y))
    return y


class RefHierarchy:
    def __init__(self, ptr, col, val, fields, labels, strategy_json, unknown_map=None):
        self.ptr = np.ascontiguousarray(ptr, np.int32)
        self.col = np.ascontiguousarray(col, np.int32)
        self.val = np.ascontiguousarray(val, np.float64)
        self.n = self.ptr.size - 1
        lab = np.ascontiguousarray(labels, np.int32)
        names = (C.c_char_p * len(fields))(*[f.encode() for f in fields])
        um = None if unknown_map is None else np.ascontiguousarray(unknown_map, np.int32)
        self._um = um
        self._h = C.c_void_p()
        _chk(lib().ref_setup(self.n, self.ptr, self.col, self.val, lab, len(fields), names,
                             None if um is None else C.c_void_p(um.ctypes.data),
                             strategy_json.encode(), C.byref(self._h)))
        self.setup_s = lib().ref_setup_seconds(self._h)

    def apply(self, v):
        z = np.empty(self.n)
        _chk(lib().ref_apply(self._h, np.ascontiguousarray(v, np.float64), z))
        return z

    def solve(self, b, restart=30, max_iters=500, rel_tol=1e-6, abs_tol=0.0, x0=None, cap=4096):
        x = np.zeros(self.n) if x0 is None else np.array(x0, dtype=np.float64)
        conv, it, fr, hl, ss = C.c_int(), C.c_int(), C.c_double(), C.c_int(), C.c_double()
        hist = np.zeros(cap)
        _chk(lib().ref_solve(self._h, np.ascontiguousarray(b, np.float64), x, restart, max_iters, rel_tol,
                             abs_tol, C.byref(conv), C.byref(it), C.byref(fr), hist, cap, C.byref(hl),
                             C.byref(ss)))
        return x, {"converged": bool(conv.value), "iterations": it.value, "final_residual": fr.value,
                   "history": hist[:min(hl.value, cap)].tolist(), "solve_s": ss.value}

    def solve_op(self, ptr, col, val, b, restart=30, max_iters=500, rel_tol=1e-6, abs_tol=0.0, x0=None,
                 cap=4096):
        """gmres(A', b, x, cfg, mgr_preconditioner(H)): another operator, this hierarchy as M."""
        x = np.zeros(self.n) if x0 is None else np.array(x0, dtype=np.float64)
        conv, it, fr, hl = C.c_int(), C.c_int(), C.c_double(), C.c_int()
        hist = np.zeros(cap)
        ptr = np.ascontiguousarray(ptr, np.int32)
        _chk(lib().ref_solve_op(self._h, ptr.size - 1, ptr, np.ascontiguousarray(col, np.int32),
                                np.ascontiguousarray(val, np.float64), np.ascontiguousarray(b, np.float64), x,
                                restart, max_iters, rel_tol, abs_tol, C.byref(conv), C.byref(it),
                                C.byref(fr), hist, cap, C.byref(hl)))
        return x, {"converged": bool(conv.value), "iterations": it.value, "final_residual": fr.value,
                   "history": hist[:min(hl.value, cap)].tolist()}

    def info(self):
        m, c = C.c_int(), C.c_int()
        fr = (C.c_int * 64)()
        lib().ref_info(self._h, C.byref(m), C.byref(c), fr, 64)
        return {"mgr_levels": m.value, "coarse_amg_levels": c.value,
                "frelax_amg_levels": [fr[i] for i in range(m.value)]}

    def amg_info(self, which=-1):
        nl, fb, tr = C.c_int(), C.c_longlong(), C.c_int()
        sizes = np.zeros(64, np.int32)
        _chk(lib().ref_amg_info(self._h, which, C.byref(nl), C.c_void_p(sizes.ctypes.data), 64, C.byref(fb),
                                C.byref(tr)))
        return {"level_sizes": sizes[:min(nl.value, 64)].tolist(), "interp_fallback_rows": fb.value,
                "truncated": bool(tr.value)}

    def dump(self, path):
        kind, rows, cols, nnz = C.c_int(), C.c_int(), C.c_int(), C.c_longlong()
        L = lib()
        _chk(L.ref_dump(self._h, path.encode(), C.byref(kind), C.byref(rows), C.byref(cols), C.byref(nnz),
                        None, None, None))
        if kind.value == 0:
            ptr = np.empty(rows.value + 1, np.int32)
            col = np.empty(max(nnz.value, 1), np.int32)
            val = np.empty(max(nnz.value, 1), np.float64)
            _chk(L.ref_dump(self._h, path.encode(), C.byref(kind), C.byref(rows), C.byref(cols),
                            C.byref(nnz), C.c_void_p(ptr.ctypes.data), C.c_void_p(col.ctypes.data),
                            C.c_void_p(val.ctypes.data)))
            return ptr, col[:nnz.value], val[:nnz.value], (rows.value, cols.value)
        if kind.value == 1:
            col = np.empty(max(nnz.value, 1), np.int32)
            _chk(L.ref_dump(self._h, path.encode(), C.byref(kind), C.byref(rows), C.byref(cols),
                            C.byref(nnz), None, C.c_void_p(col.ctypes.data), None))
            return col[:nnz.value]
        val = np.empty(max(nnz.value, 1), np.float64)
        _chk(L.ref_dump(self._h, path.encode(), C.byref(kind), C.byref(rows), C.byref(cols), C.byref(nnz),
                        None, None, C.c_void_p(val.ctypes.data)))
        return val[:nnz.value]

    def __del__(self):
        try:
            if self._h:
                lib().ref_free(self._h)
        except Exception:
            pass


def dump_paths(info: dict) -> list:
    """Every dump path of a hierarchy shape (same grammar for GPU and oracle)."""
    paths = []
    for l in range(info["mgr_levels"]):
        paths += [f"mgr.{l}.{w}" for w in ("A", "P", "R", "F", "C")]
        for k in range(info["frelax_amg_levels"][l]):
            paths += [f"mgr.{l}.frelax.amg.{k}.A"]
            if k + 1 < info["frelax_amg_levels"][l]:
                paths += [f"mgr.{l}.frelax.amg.{k}.{w}" for w in ("P", "R", "C", "F")]
    paths.append("mgr.coarse.A")
    for k in range(info["coarse_amg_levels"]):
        paths.append(f"mgr.coarse.amg.{k}.A")
        if k + 1 < info["coarse_amg_levels"]:
            paths += [f"mgr.coarse.amg.{k}.{w}" for w in ("P", "R", "C", "F")]
    return paths
