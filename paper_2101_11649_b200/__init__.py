"""paper_2101_11649_b200 — B200-native MGR-preconditioned GMRES.

Python host mirror of the reference's C++ API for the hot path
(/root/reference/proj/include/mgrkit/{mgr,krylov,strategy_json}.hpp), bound
over the C ABI of ``libmgrx.so`` (include/mgrx.h). Names follow the
reference: ``mgr_setup`` builds an MGR hierarchy from a CSR matrix, a
DofPartition (field names + per-dof labels), an optional unknown map and a
strategy (JSON text in the reference schema); ``mgr_apply`` applies one
V-cycle; ``gmres`` solves with the hierarchy as right preconditioner.

All numerics run in CUDA kernels on the GPU. There is no CPU fallback: if
``libmgrx.so`` is missing or no B200 is visible, every call raises.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("MGRX_LIB") or os.path.join(_HERE, "libmgrx.so")
_GEN_PATH = os.path.join(_HERE, "libmgrx_problems.so")

OK, NOT_CONVERGED, INVALID_ARGUMENT, RUNTIME = 0, 1, 2, 3


class MgrxError(RuntimeError):
    """Raised for status RUNTIME (std::runtime_error in the reference)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class MgrxInvalidArgument(MgrxError, ValueError):
    """Raised for status INVALID_ARGUMENT (std::invalid_argument)."""


class _Krylov(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iters", C.c_int), ("rel_tol", C.c_double),
                ("abs_tol", C.c_double), ("ortho", C.c_int)]


_ORTHO = {"default": 0, "mgs": 1, "cgs2": 2}


def _krylov(cfg) -> "_Krylov":
    if cfg.ortho not in _ORTHO:
        raise MgrxInvalidArgument(INVALID_ARGUMENT, f"gmres: unknown orthogonalisation '{cfg.ortho}'")
    return _Krylov(cfg.restart, cfg.max_iters, cfg.rel_tol, cfg.abs_tol, _ORTHO[cfg.ortho])


class _Report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("final_residual", C.c_double),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int),
                ("history_len", C.c_int), ("setup_s", C.c_double), ("solve_s", C.c_double),
                ("gpu_launches", C.c_longlong)]


_lib = None
_gen = None

_I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def lib() -> C.CDLL:
    """Load libmgrx.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise MgrxError(RUNTIME, f"libmgrx.so not built at {_LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(_LIB_PATH)
        vp = C.c_void_p
        L.mgrx_last_error.restype = C.c_char_p
        L.mgrx_create.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
        L.mgrx_destroy.argtypes = [vp]
        L.mgrx_matrix_csr.argtypes = [vp, C.c_int, C.c_int, _I32P, _I32P, _F64P, C.POINTER(vp)]
        L.mgrx_matrix_csr_device.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, C.POINTER(vp)]
        L.mgrx_matrix_destroy.argtypes = [vp]
        L.mgrx_spmv.argtypes = [vp, vp, vp, C.c_int]
        L.mgrx_setup.argtypes = [vp, vp, _I32P, C.c_int, C.POINTER(C.c_char_p), vp, C.c_char_p,
                                 C.POINTER(vp)]
        L.mgrx_hier_destroy.argtypes = [vp]
        L.mgrx_apply.argtypes = [vp, vp, vp, C.c_int]
        L.mgrx_solve.argtypes = [vp, vp, vp, C.POINTER(_Krylov), C.POINTER(_Report), C.c_int]
        L.mgrx_solve_op.argtypes = [vp, vp, vp, vp, C.POINTER(_Krylov), C.POINTER(_Report), C.c_int]
        L.mgrx_dump.argtypes = [vp, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_int), C.POINTER(C.c_longlong), vp, vp, vp]
        L.mgrx_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]
        L.mgrx_amg_info.argtypes = [vp, C.c_int, C.POINTER(C.c_int), vp, C.c_int, C.POINTER(C.c_longlong),
                                    C.POINTER(C.c_int)]
        L.mgrx_corrupt_transfer.argtypes = [vp, C.c_int, C.c_double]
        L.mgrx_time_kernel.argtypes = [vp, C.c_char_p, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]
        L.mgrx_nccl_unique_id.argtypes = [C.c_char_p]
        L.mgrx_local_group_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.mgrx_local_group_destroy.argtypes = [vp]
        L.mgrx_transport_group_create.argtypes = [C.c_int, vp, C.POINTER(vp)]
        L.mgrx_shard_create.argtypes = [vp, C.c_int, C.c_int, vp, C.c_char_p, vp, C.POINTER(vp)]
        L.mgrx_device_memory.argtypes = [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                         C.POINTER(C.c_longlong)]
        L.mgrx_hier_bytes.argtypes = [vp, C.POINTER(C.c_longlong)]
        L.mgrx_shard_bytes.argtypes = [vp, C.POINTER(C.c_longlong)]
        L.mgrx_shard_create_scatter.argtypes = [vp, vp, C.c_int, C.c_int, vp, C.c_char_p, vp, C.POINTER(vp)]
        L.mgrx_shard_rows.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.mgrx_shard_fused.argtypes = [vp, C.POINTER(C.c_int)]
        L.mgrx_shard_apply.argtypes = [vp, vp, vp, C.c_int]
        L.mgrx_shard_solve.argtypes = [vp, vp, vp, C.POINTER(_Krylov), C.POINTER(_Report), C.c_int]
        L.mgrx_shard_destroy.argtypes = [vp]
        _lib = L
    return _lib


def _check(code: int) -> int:
    if code in (OK, NOT_CONVERGED):
        return code
    msg = lib().mgrx_last_error().decode()
    if code == INVALID_ARGUMENT:
        raise MgrxInvalidArgument(code, msg)
    raise MgrxError(code, msg)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class Context:
    """One CUDA stream on one GPU (one process per GPU)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        dev = (C.c_int * 1)(device)
        _check(lib().mgrx_create(dev, 1, C.byref(self._h)))
        self.device = device

    def memory(self) -> dict:
        """libmgrx's device memory on this GPU (stream-ordered pool): bytes in
        use, reserved, and the in-use high-water mark."""
        u, r, h = C.c_longlong(), C.c_longlong(), C.c_longlong()
        _check(lib().mgrx_device_memory(self._h, C.byref(u), C.byref(r), C.byref(h)))
        return {"used": u.value, "reserved": r.value, "high": h.value}

    def close(self):
        if self._h:
            lib().mgrx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")))
    return _default_ctx


class Matrix:
    """Device-resident CSR (fp64 values, int32 indices); validated like
    proj/src/sparse.cpp:24-41."""

    def __init__(self, ptr, col, val, shape=None, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        ptr = np.ascontiguousarray(ptr, dtype=np.int32)
        col = np.ascontiguousarray(col, dtype=np.int32)
        val = np.ascontiguousarray(val, dtype=np.float64)
        rows = ptr.size - 1
        cols = shape[1] if shape is not None else rows
        self.shape = (rows, cols)
        self.nnz = int(ptr[-1])
        self._h = C.c_void_p()
        _check(lib().mgrx_matrix_csr(self.ctx._h, rows, cols, ptr, col, val, C.byref(self._h)))

    @classmethod
    def from_device(cls, rows, cols, d_ptr: int, d_col: int, d_val: int, ctx=None):
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.shape = (rows, cols)
        self._h = C.c_void_p()
        _check(lib().mgrx_matrix_csr_device(self.ctx._h, rows, cols, C.c_void_p(d_ptr),
                                            C.c_void_p(d_col), C.c_void_p(d_val), C.byref(self._h)))
        return self

    def spmv(self, x: np.ndarray, team_sums: bool = False) -> np.ndarray:
        """y = A x. team_sums: allow the tolerance-level team-sum kernel the
        default solve uses (MGRX_TEAM_SUMS); otherwise bitwise row sums."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.size != self.shape[1]:
            raise MgrxInvalidArgument(INVALID_ARGUMENT, "spmv: dimension mismatch")
        y = np.empty(self.shape[0], dtype=np.float64)
        _check(lib().mgrx_spmv(self._h, _ptr(x), _ptr(y), 4 if team_sums else 0))
        return y

    def spmv_device(self, x_ptr: int, y_ptr: int):
        _check(lib().mgrx_spmv(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), 1))

    def close(self):
        if getattr(self, "_h", None):
            lib().mgrx_matrix_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class KrylovConfig:
    """proj/include/mgrkit/krylov.hpp:14-19 (same defaults), plus `ortho`:
    "default"/"cgs2" the low-synchronisation lagged CGS2 Arnoldi (north_star
    tolerance parity), "mgs" the reference's modified Gram-Schmidt (bitwise
    against the oracle)."""
    restart: int = 50
    max_iters: int = 500
    rel_tol: float = 1e-7
    abs_tol: float = 0.0
    ortho: str = "default"


@dataclass
class SolveReport:
    """proj/include/mgrkit/krylov.hpp:21-28 plus device timings."""
    converged: bool = False
    iterations: int = 0
    final_residual: float = 0.0
    residual_history: list = field(default_factory=list)
    setup_s: float = 0.0
    solve_s: float = 0.0
    gpu_launches: int = 0


@dataclass
class DofPartition:
    """proj/include/mgrkit/mgr.hpp:20-28."""
    field_order: list
    labels: np.ndarray

    @staticmethod
    def from_names(field_order: Sequence[str], names: Sequence[str]) -> "DofPartition":
        idx = {f: k for k, f in enumerate(field_order)}
        try:
            lab = np.array([idx[n] for n in names], dtype=np.int32)
        except KeyError as e:
            raise MgrxInvalidArgument(INVALID_ARGUMENT, f"unknown field name: {e.args[0]}")
        return DofPartition(list(field_order), lab)


class Hierarchy:
    """MgrHierarchy built on the GPU (proj/include/mgrkit/mgr.hpp:79-100)."""

    def __init__(self, A: Matrix, partition: DofPartition, strategy, unknown_map=None):
        self.A = A
        self.ctx = A.ctx
        text = strategy if isinstance(strategy, str) else json.dumps(strategy)
        labels = np.ascontiguousarray(partition.labels, dtype=np.int32)
        if labels.size != A.shape[0]:
            raise MgrxInvalidArgument(INVALID_ARGUMENT, "mgr_setup: partition size does not match the matrix")
        names = (C.c_char_p * len(partition.field_order))(*[f.encode() for f in partition.field_order])
        umap = None
        if unknown_map is not None:
            umap = np.ascontiguousarray(unknown_map, dtype=np.int32)
        self._umap = umap
        self._h = C.c_void_p()
        _check(lib().mgrx_setup(self.ctx._h, A._h, labels, len(partition.field_order), names,
                                _ptr(umap) if umap is not None else None, text.encode(),
                                C.byref(self._h)))
        self.n = A.shape[0]

    def apply(self, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.size != self.n:
            raise MgrxInvalidArgument(INVALID_ARGUMENT, "mgr_apply: size mismatch")
        z = np.empty(self.n, dtype=np.float64)
        _check(lib().mgrx_apply(self._h, _ptr(v), _ptr(z), 0))
        return z

    def apply_device(self, v_ptr: int, z_ptr: int):
        _check(lib().mgrx_apply(self._h, C.c_void_p(v_ptr), C.c_void_p(z_ptr), 1))

    def solve(self, b: np.ndarray, x: Optional[np.ndarray] = None, cfg: Optional[KrylovConfig] = None,
              history_cap: int = 4096, out: Optional[np.ndarray] = None) -> tuple:
        """gmres(A, b, x0, cfg, M) with host arrays. x (initial guess) is not
        modified; None means a zero guess (nothing copied to the device). The
        solution goes to `out` when given (contiguous float64 of size n, e.g.
        pinned memory), else to a new array."""
        cfg = cfg or KrylovConfig()
        b = np.ascontiguousarray(b, dtype=np.float64)
        if out is None:
            out = np.empty(self.n)
        elif out.dtype != np.float64 or out.size != self.n or not out.flags.c_contiguous:
            raise MgrxError(INVALID_ARGUMENT, "solve: out must be a contiguous float64 array of size n")
        flags = 0
        if x is None:
            flags |= 2  # MGRX_ZERO_GUESS
        else:
            np.copyto(out, np.asarray(x, dtype=np.float64).reshape(-1))
        rep, hist = self._report(history_cap)
        k = _krylov(cfg)
        _check(lib().mgrx_solve(self._h, _ptr(b), _ptr(out), C.byref(k), C.byref(rep), flags))
        return out, self._to_report(rep, hist)

    def solve_device(self, b_ptr: int, x_ptr: int, cfg: Optional[KrylovConfig] = None,
                     history_cap: int = 4096) -> SolveReport:
        cfg = cfg or KrylovConfig()
        rep, hist = self._report(history_cap)
        k = _krylov(cfg)
        _check(lib().mgrx_solve(self._h, C.c_void_p(b_ptr), C.c_void_p(x_ptr), C.byref(k), C.byref(rep), 1))
        return self._to_report(rep, hist)

    def solve_op(self, A: "Matrix", b: np.ndarray, x: Optional[np.ndarray] = None,
                 cfg: Optional[KrylovConfig] = None, history_cap: int = 4096) -> tuple:
        """gmres(A, b, x0, cfg, mgr_preconditioner(self)) with an operator A
        other than the one this hierarchy was built from (a hierarchy kept
        across Newton steps; mgrx_solve_op)."""
        cfg = cfg or KrylovConfig()
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty(self.n)
        flags = 0
        if x is None:
            flags |= 2  # MGRX_ZERO_GUESS
        else:
            np.copyto(out, np.asarray(x, dtype=np.float64).reshape(-1))
        rep, hist = self._report(history_cap)
        k = _krylov(cfg)
        _check(lib().mgrx_solve_op(self._h, A._h, _ptr(b), _ptr(out), C.byref(k), C.byref(rep), flags))
        return out, self._to_report(rep, hist)

    @staticmethod
    def _report(cap):
        hist = np.zeros(cap, dtype=np.float64)
        rep = _Report()
        rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_cap = cap
        return rep, hist

    @staticmethod
    def _to_report(rep, hist) -> SolveReport:
        n = min(rep.history_len, hist.size)
        return SolveReport(bool(rep.converged), rep.iterations, rep.final_residual, hist[:n].tolist(),
                           rep.setup_s, rep.solve_s, rep.gpu_launches)

    def info(self) -> dict:
        m, c = C.c_int(), C.c_int()
        fr = (C.c_int * 64)()
        _check(lib().mgrx_info(self._h, C.byref(m), C.byref(c), fr, 64))
        return {"mgr_levels": m.value, "coarse_amg_levels": c.value,
                "frelax_amg_levels": [fr[i] for i in range(m.value)]}

    def device_bytes(self) -> int:
        """Device bytes the setup allocated (matrix copy + hierarchy)."""
        v = C.c_longlong()
        _check(lib().mgrx_hier_bytes(self._h, C.byref(v)))
        return v.value

    def amg_info(self, which: int = -1) -> dict:
        """AmgSetupInfo (proj/include/mgrkit/amg.hpp:35-39) of the MGR coarse
        AMG (which=-1) or of MGR level `which`'s F-relaxation AMG."""
        nl, fb, tr = C.c_int(), C.c_longlong(), C.c_int()
        sizes = np.zeros(64, np.int32)
        _check(lib().mgrx_amg_info(self._h, which, C.byref(nl), _ptr(sizes), 64, C.byref(fb), C.byref(tr)))
        return {"level_sizes": sizes[:min(nl.value, 64)].tolist(), "interp_fallback_rows": fb.value,
                "truncated": bool(tr.value)}

    def corrupt_transfer(self, level: int = 0, factor: float = 1.01) -> None:
        """Negative control of proj/src/verify.cpp:115 (`verify
        --corrupt-transfer`): scale P of MGR level `level` in place."""
        _check(lib().mgrx_corrupt_transfer(self._h, int(level), float(factor)))

    def dump(self, path: str):
        """CSR -> (ptr, col, val, shape); int list -> int32 array; vector -> float64 array."""
        kind, rows, cols, nnz = C.c_int(), C.c_int(), C.c_int(), C.c_longlong()
        _check(lib().mgrx_dump(self._h, path.encode(), C.byref(kind), C.byref(rows), C.byref(cols),
                               C.byref(nnz), None, None, None))
        if kind.value == 0:
            ptr = np.empty(rows.value + 1, np.int32)
            col = np.empty(max(nnz.value, 1), np.int32)
            val = np.empty(max(nnz.value, 1), np.float64)
            _check(lib().mgrx_dump(self._h, path.encode(), C.byref(kind), C.byref(rows), C.byref(cols),
                                   C.byref(nnz), _ptr(ptr), _ptr(col), _ptr(val)))
            return ptr, col[:nnz.value], val[:nnz.value], (rows.value, cols.value)
        if kind.value == 1:
            col = np.empty(max(nnz.value, 1), np.int32)
            _check(lib().mgrx_dump(self._h, path.encode(), C.byref(kind), C.byref(rows), C.byref(cols),
                                   C.byref(nnz), None, _ptr(col), None))
            return col[:nnz.value]
        val = np.empty(max(nnz.value, 1), np.float64)
        _check(lib().mgrx_dump(self._h, path.encode(), C.byref(kind), C.byref(rows), C.byref(cols),
                               C.byref(nnz), None, None, _ptr(val)))
        return val[:nnz.value]

    def time_kernel(self, which: str, reps: int = 20) -> tuple:
        """(average device ms, algorithmic bytes) of one hot kernel."""
        ms, by = C.c_double(), C.c_double()
        _check(lib().mgrx_time_kernel(self._h, which.encode(), reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def close(self):
        if getattr(self, "_h", None):
            lib().mgrx_hier_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- row-slab sharded solve -----------------------------------
def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it and distributes it)."""
    buf = C.create_string_buffer(128)
    _check(lib().mgrx_nccl_unique_id(buf))
    return buf.raw


class LocalGroup:
    """Ranks that are threads of this process on one device (parity tests)."""

    def __init__(self, size: int):
        self.size = size
        self._h = C.c_void_p()
        _check(lib().mgrx_local_group_create(size, C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().mgrx_local_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p), C.POINTER(C.c_int),
                           C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p), C.POINTER(C.c_int))
_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int)


class _Transport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("exchange", _EXCHANGE_FN), ("allgather", _ALLGATHER_FN)]


def _host_array(ptr, count):
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(count,)) if count > 0 else np.empty(0)


class TransportGroup:
    """mgrx_transport_group_create: ranks are processes connected by the
    caller's own communicator (MPI, gloo, ...), host-staged. `exchange(sends,
    recvs)` gets lists of (peer, float64 host array) -- send each array to its
    peer, fill each receive array from its peer -- and `allgather(src, dst)`
    fills dst (size * len(src)) with every rank's src in rank order; both
    block until done. Use as the `group` of a Shard in every process."""

    def __init__(self, size: int, exchange, allgather):
        self.size = size

        def _xchg(_user, ns, sp, sb, sc, nr, rp, rb, rc):
            try:
                exchange([(sp[i], _host_array(sb[i], sc[i])) for i in range(ns)],
                         [(rp[j], _host_array(rb[j], rc[j])) for j in range(nr)])
                return 0
            except Exception:  # the library reports the failure as its own error
                import traceback
                traceback.print_exc()
                return 1

        def _gather(_user, src, dst, count):
            try:
                allgather(_host_array(src, count), _host_array(dst, count * size))
                return 0
            except Exception:
                import traceback
                traceback.print_exc()
                return 1

        self._cb = (_EXCHANGE_FN(_xchg), _ALLGATHER_FN(_gather))  # keep the thunks alive
        self._t = _Transport(None, self._cb[0], self._cb[1])
        self._h = C.c_void_p()
        _check(lib().mgrx_transport_group_create(size, C.byref(self._t), C.byref(self._h)))

    @staticmethod
    def torch_distributed(pg=None) -> "TransportGroup":
        """Transport over an initialised torch.distributed process group
        (gloo: host tensors; isend / irecv for the halos, all_gather)."""
        import torch
        import torch.distributed as dist
        size = dist.get_world_size(pg)

        def exchange(sends, recvs):
            ops = [dist.irecv(torch.from_numpy(a), src=p, group=pg) for p, a in recvs]
            ops += [dist.isend(torch.from_numpy(a), dst=p, group=pg) for p, a in sends]
            for o in ops:
                o.wait()

        def allgather(src, dst):
            dist.all_gather_into_tensor(torch.from_numpy(dst), torch.from_numpy(src), group=pg)

        return TransportGroup(size, exchange, allgather)

    def close(self):
        if getattr(self, "_h", None):
            lib().mgrx_local_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Shard:
    """This rank's slab of a hierarchy (every rank builds the same Hierarchy):
    owned fine rows [row_begin, row_end); apply / solve on owned slices.
    Collective: every rank of the group makes the same sequence of calls."""

    def __init__(self, H: Optional[Hierarchy], rank: int, size: int, row_starts=None,
                 nccl_id: Optional[bytes] = None, group: Optional[LocalGroup] = None, scatter: bool = False,
                 ctx: Optional[Context] = None):
        """scatter=False: every rank passes its replica of the global Hierarchy.
        scatter=True (mgrx_shard_create_scatter): rank 0 passes the global
        Hierarchy, the other ranks pass None (and a Context); rank 0 sends
        every rank its slab plan, no other rank holds a global operator, and
        rank 0 may drop H afterwards."""
        self.H = H if not scatter else None
        st = None
        if row_starts is not None:
            st = np.ascontiguousarray(row_starts, dtype=np.int32)
            if st.size != size + 1:
                raise MgrxInvalidArgument(INVALID_ARGUMENT, "row_starts must have size+1 entries")
        self._st = st
        self._h = C.c_void_p()
        g = group._h if group is not None else None
        if scatter:
            if st is None:
                raise MgrxInvalidArgument(INVALID_ARGUMENT, "scatter: row_starts are required")
            cx = ctx or (H.ctx if H is not None else default_context())
            self._ctx = cx
            _check(lib().mgrx_shard_create_scatter(cx._h, H._h if H is not None else None, rank, size, _ptr(st),
                                                   nccl_id, g, C.byref(self._h)))
        else:
            _check(lib().mgrx_shard_create(H._h, rank, size, _ptr(st) if st is not None else None,
                                           nccl_id, g, C.byref(self._h)))
        b, e = C.c_int(), C.c_int()
        _check(lib().mgrx_shard_rows(self._h, C.byref(b), C.byref(e)))
        self.row_begin, self.row_end = b.value, e.value
        self.n = self.row_end - self.row_begin
        f = C.c_int()
        _check(lib().mgrx_shard_fused(self._h, C.byref(f)))
        self.fused = bool(f.value)  # fused sharded Arnoldi in use (one GPU per rank)

    def device_bytes(self) -> int:
        """Device bytes of this rank's shard (slabs, halo plans, replicated
        small parts, work vectors), as allocated by the creating thread."""
        v = C.c_longlong()
        _check(lib().mgrx_shard_bytes(self._h, C.byref(v)))
        return v.value

    def apply(self, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        z = np.empty(self.n)
        _check(lib().mgrx_shard_apply(self._h, _ptr(v), _ptr(z), 0))
        return z

    def solve(self, b: np.ndarray, x: Optional[np.ndarray] = None, cfg: Optional[KrylovConfig] = None,
              history_cap: int = 4096, out: Optional[np.ndarray] = None) -> tuple:
        cfg = cfg or KrylovConfig()
        b = np.ascontiguousarray(b, dtype=np.float64)
        if out is None:
            out = np.empty(self.n)
        flags = 0
        if x is None:
            flags |= 2
        else:
            np.copyto(out, np.asarray(x, dtype=np.float64).reshape(-1))
        rep, hist = Hierarchy._report(history_cap)
        k = _krylov(cfg)
        _check(lib().mgrx_shard_solve(self._h, _ptr(b), _ptr(out), C.byref(k), C.byref(rep), flags))
        return out, Hierarchy._to_report(rep, hist)

    def solve_device(self, b_ptr: int, x_ptr: int, cfg: Optional[KrylovConfig] = None, zero_guess=False,
                     history_cap: int = 4096) -> SolveReport:
        cfg = cfg or KrylovConfig()
        rep, hist = Hierarchy._report(history_cap)
        k = _krylov(cfg)
        _check(lib().mgrx_shard_solve(self._h, C.c_void_p(b_ptr), C.c_void_p(x_ptr), C.byref(k), C.byref(rep),
                                      1 | (2 if zero_guess else 0)))
        return Hierarchy._to_report(rep, hist)

    def close(self):
        if getattr(self, "_h", None):
            lib().mgrx_shard_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_row_starts(problem: "Problem", size: int) -> np.ndarray:
    """Fine-row offsets for `size` ranks cut at z-slab boundaries of a
    generated bundle (slab-major numbering): ranks own whole
    z-layers; falls back to an even split for bundles without slab metadata."""
    n = problem.n
    meta = problem.meta or {}
    slabs = None
    if meta.get("problem") == "mfd" and meta.get("numbering") == "slab-major-z":
        nx, ny, nz = meta["dims"]
        per = nx * ny + (nx + 1) * ny + nx * (ny + 1) + nx * ny
        slabs = [k * per for k in range(nz)]
    elif meta.get("problem") == "comp":
        nx, ny, nz = meta["dims"]
        per = nx * ny * meta.get("dofs_per_cell", 4)
        slabs = [k * per for k in range(nz)]  # wells are numbered last: the last rank owns them
    if not slabs or len(slabs) < size:
        return np.array([n * q // size for q in range(size + 1)], np.int32)
    k = len(slabs)
    return np.array([slabs[(q * k) // size] for q in range(size)] + [n], np.int32)


# ---- reference-named entry points -----------------------------------------
def mgr_setup(A: Matrix, partition: DofPartition, strategy, unknown_map=None) -> Hierarchy:
    """proj/include/mgrkit/mgr.hpp:105-106"""
    return Hierarchy(A, partition, strategy, unknown_map)


def mgr_apply(H: Hierarchy, v: np.ndarray) -> np.ndarray:
    """proj/include/mgrkit/mgr.hpp:111"""
    return H.apply(v)


def gmres(A: Matrix, b: np.ndarray, x: np.ndarray, cfg: KrylovConfig, H: Hierarchy):
    """gmres(A, b, x, cfg, mgr_preconditioner(H)) — proj/include/mgrkit/krylov.hpp:33-34.
    With the matrix H was built from, the hierarchy's copy of A is the
    operator; any other matrix goes through mgrx_solve_op (H as a lagged
    preconditioner). Returns (x, SolveReport)."""
    if A is not H.A:
        return H.solve_op(A, b, x, cfg)
    return H.solve(b, x, cfg)


# ---- problem generators (BASELINE configs) --------------------------------
def _genlib() -> C.CDLL:
    global _gen
    if _gen is None:
        if not os.path.exists(_GEN_PATH):
            raise MgrxError(RUNTIME, f"libmgrx_problems.so not built at {_GEN_PATH}")
        G = C.CDLL(_GEN_PATH)
        G.mgrx_gen_mfd.restype = C.c_void_p
        G.mgrx_gen_mfd.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint, C.c_double]
        G.mgrx_gen_comp.restype = C.c_void_p
        G.mgrx_gen_comp.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint]
        G.mgrx_gen_frac.restype = C.c_void_p
        G.mgrx_gen_frac.argtypes = [C.c_int, C.c_double, C.c_uint]
        for f in ("mgrx_gen_n", "mgrx_gen_nfields", "mgrx_gen_has_unknown_map"):
            getattr(G, f).argtypes = [C.c_void_p]
        G.mgrx_gen_nnz.argtypes = [C.c_void_p]
        G.mgrx_gen_nnz.restype = C.c_longlong
        G.mgrx_gen_field.argtypes = [C.c_void_p, C.c_int]
        G.mgrx_gen_field.restype = C.c_char_p
        G.mgrx_gen_meta.argtypes = [C.c_void_p]
        G.mgrx_gen_meta.restype = C.c_char_p
        G.mgrx_gen_last_error.restype = C.c_char_p
        G.mgrx_gen_copy.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        G.mgrx_gen_free.argtypes = [C.c_void_p]
        _gen = G
    return _gen


@dataclass
class Problem:
    """A bundle: matrix (CSR), rhs, DofPartition, optional unknown map, meta."""
    ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    rhs: np.ndarray
    partition: DofPartition
    unknown_map: Optional[np.ndarray]
    meta: dict

    @property
    def n(self) -> int:
        return self.ptr.size - 1


def _take(h) -> Problem:
    G = _genlib()
    if not h:
        raise MgrxInvalidArgument(INVALID_ARGUMENT, G.mgrx_gen_last_error().decode())
    try:
        n, nnz = G.mgrx_gen_n(h), G.mgrx_gen_nnz(h)
        ptr = np.empty(n + 1, np.int32)
        col = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        lab = np.empty(n, np.int32)
        rhs = np.empty(n, np.float64)
        umap = np.empty(n, np.int32) if G.mgrx_gen_has_unknown_map(h) else None
        G.mgrx_gen_copy(h, _ptr(ptr), _ptr(col), _ptr(val), _ptr(lab), _ptr(rhs),
                        _ptr(umap) if umap is not None else None)
        fields = [G.mgrx_gen_field(h, k).decode() for k in range(G.mgrx_gen_nfields(h))]
        meta = json.loads(G.mgrx_gen_meta(h).decode())
        return Problem(ptr, col, val, rhs, DofPartition(fields, lab), umap, meta)
    finally:
        G.mgrx_gen_free(h)


def mfd_problem(nx: int, ny: int, nz: int, field: str = "iid", sigma: float = 1.5,
                seed: int = 20210128, accumulation: float = 1e-3) -> Problem:
    """Hybrid-MFD [p, pi] condensed system (BASELINE cfg1: 20x20x10 iid;
    cfg2: 128x128x64 layered)."""
    kind = {"iid": 0, "layered": 1}[field]
    return _take(_genlib().mgrx_gen_mfd(nx, ny, nz, kind, sigma, seed, accumulation))


def comp_problem(nx: int, ny: int, nz: int, wells: int = 8, sigma_t: float = 2.0,
                 seed: int = 20210130) -> Problem:
    """Compositional [p, rho1, rho2, rho3] + wells (BASELINE cfg3: 100x100x50,
    8 wells; cfg5: weak-scaled)."""
    return _take(_genlib().mgrx_gen_comp(nx, ny, nz, wells, sigma_t, seed))


def frac_problem(nodes_per_side: int = 64, sigma_e: float = 0.5, seed: int = 20210131) -> Problem:
    """3-D Q1 elasticity + planar-fracture lubrication, fields {u, p} with a
    displacement-component unknown map (BASELINE cfg4: 64^3 nodes)."""
    return _take(_genlib().mgrx_gen_frac(nodes_per_side, sigma_e, seed))


STRATEGY_DIR =os.path.join(os.path.dirname(_HERE), "strategies")


def load_strategy(name: str) -> str:
    """Strategy JSON text from strategies/<name>.json (reference schema)."""
    path = name if os.path.exists(name) else os.path.join(STRATEGY_DIR, name + ".json")
    with open(path) as f:
        return f.read()
