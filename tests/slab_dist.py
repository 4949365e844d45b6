"""TEST SCAFFOLDING (not the product): a Python/NumPy restatement of the
row-slab distributed MGR-GMRES, used by the world-size-2
gloo tests to check the slab algorithm's host logic (partition, halo plans,
rank-order reductions) on CPU. The product's sharded path is csrc/shard.cu
(C ABI mgrx_shard_*); it never imports this module.

One process per GPU. The slab-major dof numbering (generators)
makes every operator of every level a contiguous row block per rank: MGR C/F
sets are ascending subsets (proj/src/mgr.cpp:27-35) and AMG coarse order
follows fine order (proj/src/amg.cpp:209-222), so a rank's coarse rows are
the C points inside its fine range.

Setup: every rank builds the same global hierarchy (bit-exact kernels, so
all ranks hold identical operators) and keeps its row slab of each operator,
with columns renumbered [owned | halo] and a halo exchange plan per index
space. Solve: halo exchange (batched point-to-point: NCCL on GPUs, gloo on
CPU) before every SpMV-type product, a deterministic reduction for inner
products (all-gather of per-rank partials, summed in rank order), the
coarsest dense solve replicated (all-gather of the coarse vector).

Smoothers: jacobi and l1_jacobi shard exactly (pointwise + halo'd SpMV). The
reference's hybrid Gauss-Seidel with one range is a sequential sweep over
the whole matrix; across ranks it would be a distributed triangular solve,
which this layer does not implement (raises NotImplementedError) — sharded
runs use the Jacobi-family strategies of the same schema.

Local compute goes through a backend: ``NumpyBackend`` (CPU tests) or
``DeviceBackend`` (libmgrx kernels on the rank's GPU, torch for plumbing).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

try:
    import torch
    import torch.distributed as tdist
except Exception:  # pragma: no cover
    torch = None
    tdist = None


# ----------------------------------------------------------------------------
# communication
# ----------------------------------------------------------------------------
class Comm:
    """Thin wrapper over torch.distributed (or a single-rank stand-in)."""

    def __init__(self, device: str = "cpu"):
        self.dist = tdist is not None and tdist.is_available() and tdist.is_initialized()
        self.rank = tdist.get_rank() if self.dist else 0
        self.size = tdist.get_world_size() if self.dist else 1
        self.device = device

    def allgather_obj(self, obj):
        if not self.dist:
            return [obj]
        out = [None] * self.size
        tdist.all_gather_object(out, obj)
        return out

    def exchange(self, sends: Dict[int, "torch.Tensor"], recvs: Dict[int, "torch.Tensor"]):
        """Batched point-to-point: sends[q] -> rank q, recvs[q] <- rank q."""
        if not self.dist or (not sends and not recvs):
            return
        ops = []
        for q, t in recvs.items():
            ops.append(tdist.P2POp(tdist.irecv, t, q))
        for q, t in sends.items():
            ops.append(tdist.P2POp(tdist.isend, t, q))
        for w in tdist.batch_isend_irecv(ops):
            w.wait()

    def allgather_vec(self, t: "torch.Tensor", counts: List[int]) -> "torch.Tensor":
        if not self.dist:
            return t
        mx = max(counts)
        buf = torch.zeros(mx, dtype=t.dtype, device=t.device)
        buf[: t.numel()] = t
        parts = [torch.zeros(mx, dtype=t.dtype, device=t.device) for _ in range(self.size)]
        tdist.all_gather(parts, buf)
        return torch.cat([p[:c] for p, c in zip(parts, counts)])

    def sum_scalars(self, vals: "torch.Tensor") -> "torch.Tensor":
        """Deterministic sum over ranks of a small vector of partials: every
        rank all-gathers the partials and adds them in rank order."""
        if not self.dist:
            return vals
        parts = [torch.zeros_like(vals) for _ in range(self.size)]
        tdist.all_gather(parts, vals)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc = acc + p
        return acc


# ----------------------------------------------------------------------------
# partitioned operators
# ----------------------------------------------------------------------------
def ranges_from_flags(flags: np.ndarray, parent: List[Tuple[int, int]]) -> List[Tuple[int, int]]:
    """Sub-index-space ranges: the flagged points inside each parent range,
    numbered in order (contiguous per rank)."""
    pre = np.concatenate([[0], np.cumsum(flags.astype(np.int64))])
    return [(int(pre[a]), int(pre[b])) for a, b in parent]


@dataclass
class HaloPlan:
    """Local columns = [owned (0..m) | halo (m..m+h)], halo sorted by global id."""
    m: int
    halo_global: np.ndarray
    recv: Dict[int, np.ndarray]   # rank -> positions in the halo array
    send: Dict[int, np.ndarray]   # rank -> local owned indices to send


def build_plan(comm: Comm, col_ranges: List[Tuple[int, int]], needed_global: np.ndarray) -> HaloPlan:
    me = comm.rank
    c0, c1 = col_ranges[me]
    halo = np.unique(needed_global[(needed_global < c0) | (needed_global >= c1)])
    owner = np.searchsorted([b for _, b in col_ranges], halo, side="right")
    recv = {int(q): np.nonzero(owner == q)[0] for q in np.unique(owner)}
    # tell every rank which of its entries I need
    req = {int(q): halo[idx] for q, idx in recv.items()}
    all_req = comm.allgather_obj(req)
    send = {}
    for q in range(comm.size):
        if q == me:
            continue
        want = all_req[q].get(me)
        if want is not None and len(want):
            send[q] = (np.asarray(want) - c0).astype(np.int64)
    return HaloPlan(c1 - c0, halo, recv, send)


@dataclass
class SlabCsr:
    """Rows [r0, r1) of a global CSR with columns renumbered through a plan."""
    rows: int
    ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    plan: HaloPlan


def slab(comm: Comm, csr: Tuple, row_ranges, col_ranges) -> SlabCsr:
    ptr, col, val = csr[0], csr[1], csr[2]
    r0, r1 = row_ranges[comm.rank]
    lo, hi = int(ptr[r0]), int(ptr[r1])
    lcol_g = col[lo:hi].astype(np.int64)
    plan = build_plan(comm, col_ranges, lcol_g)
    c0, c1 = col_ranges[comm.rank]
    owned = (lcol_g >= c0) & (lcol_g < c1)
    lcol = np.empty_like(lcol_g)
    lcol[owned] = lcol_g[owned] - c0
    lcol[~owned] = plan.m + np.searchsorted(plan.halo_global, lcol_g[~owned])
    lptr = (ptr[r0:r1 + 1] - lo).astype(np.int32)
    return SlabCsr(r1 - r0, lptr, lcol.astype(np.int32), val[lo:hi].copy(), plan)


# ----------------------------------------------------------------------------
# local compute backends
# ----------------------------------------------------------------------------
class NumpyBackend:
    """CPU reference backend (tests): sequential per-row sums, no FMA."""
    device = "cpu"

    def vec(self, a):
        return torch.as_tensor(np.asarray(a, dtype=np.float64)).clone()

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def matrix(self, s: SlabCsr):
        return s

    def spmv(self, M: SlabCsr, xfull: "torch.Tensor") -> "torch.Tensor":
        x = xfull.numpy()
        y = np.zeros(M.rows)
        for i in range(M.rows):
            acc = 0.0
            for k in range(M.ptr[i], M.ptr[i + 1]):
                acc += M.val[k] * x[M.col[k]]
            y[i] = 0.0 + acc
        return torch.from_numpy(y)

    def dot(self, a, b):
        return float(np.dot(a.numpy(), b.numpy()))


class DeviceBackend:
    """libmgrx kernels on this rank's GPU (local slab SpMV); torch tensors
    carry vectors (plumbing)."""

    def __init__(self, ctx):
        import paper_2101_11649_b200 as mx
        self.mx = mx
        self.ctx = ctx
        self.device = f"cuda:{ctx.device}"

    def vec(self, a):
        return torch.as_tensor(np.asarray(a, dtype=np.float64), device=self.device).clone()

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64, device=self.device)

    def matrix(self, s: SlabCsr):
        ncols = s.plan.m + len(s.plan.halo_global)
        M = self.mx.Matrix(s.ptr, s.col, s.val, shape=(s.rows, max(ncols, 1)), ctx=self.ctx)
        M.slab = s
        return M

    def spmv(self, M, xfull):
        y = torch.empty(M.shape[0], dtype=torch.float64, device=self.device)
        if M.shape[0]:
            M.spmv_device(xfull.data_ptr(), y.data_ptr())
        return y

    def dot(self, a, b):
        return float(torch.dot(a, b).item())


# ----------------------------------------------------------------------------
# distributed hierarchy
# ----------------------------------------------------------------------------
class DistOperator:
    def __init__(self, comm, be, csr, row_ranges, col_ranges):
        self.comm, self.be = comm, be
        s = slab(comm, csr, row_ranges, col_ranges)
        self.plan = s.plan
        self.M = be.matrix(s)
        self.rows = s.rows

    def halo(self, x_owned: "torch.Tensor") -> "torch.Tensor":
        p = self.plan
        h = torch.zeros(len(p.halo_global), dtype=x_owned.dtype, device=x_owned.device)
        recvs = {q: torch.zeros(len(idx), dtype=x_owned.dtype, device=x_owned.device) for q, idx in p.recv.items()}
        sends = {q: x_owned[torch.as_tensor(idx, device=x_owned.device)].contiguous() for q, idx in p.send.items()}
        self.comm.exchange(sends, recvs)
        for q, idx in p.recv.items():
            h[torch.as_tensor(idx, device=x_owned.device)] = recvs[q]
        return torch.cat([x_owned, h])

    def apply(self, x_owned):
        return self.be.spmv(self.M, self.halo(x_owned))


@dataclass
class DistSmoother:
    kind: str
    sweeps: int
    weight: float
    dinv: "torch.Tensor"
    A: Optional[DistOperator]

    def apply(self, r):
        w = self.weight
        z = w * (self.dinv * r)
        for _ in range(1, self.sweeps):
            d = r - (0.0 + self.A.apply(z))
            z = z + w * (self.dinv * d)
        return z


def _smoother(comm, be, spec, A_csr, rr, dump_diag):
    kind = spec.get("kind", "jacobi")
    if kind not in ("jacobi", "l1_jacobi"):
        raise NotImplementedError(
            f"sharded smoother '{kind}': only jacobi / l1_jacobi shard exactly across slabs")
    r0, r1 = rr[comm.rank]
    dinv = be.vec(dump_diag[r0:r1])
    sweeps = int(spec.get("sweeps", 1))
    A = DistOperator(comm, be, A_csr, rr, rr) if sweeps > 1 else None
    return DistSmoother(kind, sweeps, float(spec.get("weight", 1.0)), dinv, A)


def _inv_diag(csr, l1: bool):
    ptr, col, val = csr[0], csr[1], csr[2]
    n = ptr.size - 1
    d = np.zeros(n)
    for i in range(n):
        s = 0.0
        for k in range(ptr[i], ptr[i + 1]):
            if col[k] == i:
                s += val[k]
            elif l1:
                s += abs(val[k])
        d[i] = s
    return 1.0 / d


class DistAmg:
    def __init__(self, comm, be, dump, prefix, nlev, spec, row_ranges):
        self.comm, self.be = comm, be
        self.levels = []
        rr = row_ranges
        pre = spec.get("pre_smoother", {"kind": "hybrid_l1_gs_forward"})
        post = spec.get("post_smoother", {"kind": "hybrid_l1_gs_backward"})
        for k in range(nlev):
            A = dump(f"{prefix}.{k}.A")
            if k == nlev - 1:
                n = A[0].size - 1
                dense = np.zeros((n, n))
                for i in range(n):
                    dense[i, A[1][A[0][i]:A[0][i + 1]]] = A[2][A[0][i]:A[0][i + 1]]
                self.coarse = (dense, rr)
                break
            C = dump(f"{prefix}.{k}.C")
            flags = np.zeros(A[0].size - 1, bool)
            flags[C] = True
            cr = ranges_from_flags(flags, rr)
            L = {"A": DistOperator(comm, be, A, rr, rr),
                 "P": DistOperator(comm, be, dump(f"{prefix}.{k}.P"), rr, cr),
                 "R": DistOperator(comm, be, dump(f"{prefix}.{k}.R"), cr, rr),
                 "pre": _smoother(comm, be, pre, A, rr, _inv_diag(A, pre.get("kind") == "l1_jacobi")),
                 "post": _smoother(comm, be, post, A, rr, _inv_diag(A, post.get("kind") == "l1_jacobi")),
                 "rows": rr}
            self.levels.append(L)
            rr = cr

    def vcycle(self, r, l=0):
        if l == len(self.levels):
            dense, rr = self.coarse
            full = self.comm.allgather_vec(r, [b - a for a, b in rr])
            z = np.linalg.solve(dense, full.cpu().numpy()) if dense.size else full.cpu().numpy()
            a, b = rr[self.comm.rank]
            return self.be.vec(z[a:b])
        L = self.levels[l]
        z = L["pre"].apply(r)
        t = r - (0.0 + L["A"].apply(z))
        rc = 0.0 + L["R"].apply(t)
        ec = self.vcycle(rc, l + 1)
        z = z + L["P"].apply(ec)
        t = r - (0.0 + L["A"].apply(z))
        return z + L["post"].apply(t)


class DistMgr:
    """Sharded MGR preconditioner built from a replicated hierarchy's dumps.
    `dump(path)` returns the same objects as Hierarchy.dump / RefHierarchy.dump."""

    def __init__(self, comm, be, dump, info, strategy: dict, row_ranges):
        self.comm, self.be = comm, be
        self.levels = []
        rr = row_ranges
        for l, spec in enumerate(strategy.get("levels", [])):
            if spec.get("restrict", "injection") != "injection" or spec.get("global_relax"):
                raise NotImplementedError("sharded MGR levels use injection restriction, no global relax")
            A = dump(f"mgr.{l}.A")
            F = dump(f"mgr.{l}.F")
            n = A[0].size - 1
            isf = np.zeros(n, bool)
            isf[F] = True
            fr = ranges_from_flags(isf, rr)
            cr = ranges_from_flags(~isf, rr)
            P = dump(f"mgr.{l}.P")
            # restricted-residual operator A_CF (rows C, cols F-index) and A_FF
            Cidx = np.nonzero(~isf)[0]
            fpos = np.cumsum(isf) - 1
            Acf = _extract(A, Cidx, isf, fpos)
            Aff = _extract(A, F, isf, fpos)
            relax = spec.get("f_relax", {"kind": "jacobi"})
            L = {"F_local": None, "rows": rr, "fr": fr, "cr": cr,
                 "Acf": DistOperator(comm, be, Acf, cr, fr),
                 "P": DistOperator(comm, be, P, rr, cr),
                 "relax": _smoother(comm, be, relax, Aff, fr,
                                    _inv_diag(Aff, relax.get("kind") == "l1_jacobi")),
                 "isf_local": None}
            a, b = rr[comm.rank]
            L["isf_local"] = torch.as_tensor(isf[a:b], device=be.device)
            self.levels.append(L)
            rr = cr
        coarse = strategy.get("coarse", {"kind": "dense_lu"})
        if coarse.get("kind") != "amg_vcycle":
            raise NotImplementedError("sharded coarse solver: amg_vcycle")
        self.cycles = int(coarse.get("cycles", 1))
        self.Ac = DistOperator(comm, be, dump("mgr.coarse.A"), rr, rr)
        self.amg = DistAmg(comm, be, dump, "mgr.coarse.amg", info["coarse_amg_levels"], coarse.get("amg", {}), rr)

    def apply(self, v, l=0):
        if l == len(self.levels):
            z = self.amg.vcycle(v)
            for _ in range(1, self.cycles):
                z = z + self.amg.vcycle(v - (0.0 + self.Ac.apply(z)))
            return z
        L = self.levels[l]
        isf = L["isf_local"]
        vF = v[isf]
        zF = L["relax"].apply(vF)
        rc = v[~isf] - (0.0 + L["Acf"].apply(zF))
        e = self.apply(rc, l + 1)
        z = torch.zeros_like(v)
        z[isf] = 0.0 + zF
        return z + L["P"].apply(e)


def _extract(A, rows, isf, fpos):
    ptr, col, val = A[0], A[1], A[2]
    optr, ocol, oval = [0], [], []
    for r in rows:
        for k in range(ptr[r], ptr[r + 1]):
            if isf[col[k]]:
                ocol.append(fpos[col[k]])
                oval.append(val[k])
        optr.append(len(ocol))
    return np.array(optr, np.int32), np.array(ocol, np.int32), np.array(oval, np.float64)


def slab_ranges(n: int, slab_starts: List[int], size: int) -> List[Tuple[int, int]]:
    """Contiguous row ranges for `size` ranks, cut at slab boundaries
    (slab_starts: first dof of each z-slab, ascending)."""
    k = len(slab_starts)
    cuts = [slab_starts[(r * k) // size] for r in range(size)] + [n]
    return [(cuts[r], cuts[r + 1]) for r in range(size)]


def gmres(comm, be, A: DistOperator, M, b, x, restart=30, max_iters=500, rel_tol=1e-6):
    """Right-preconditioned restarted GMRES (proj/src/krylov.cpp:37-147) on
    slab-distributed vectors; inner products reduced deterministically."""
    def dot(a, c):
        return float(comm.sum_scalars(torch.tensor([be.dot(a, c)], dtype=torch.float64,
                                                    device=a.device))[0])

    bnorm = dot(b, b) ** 0.5
    hist = []
    if bnorm == 0.0:
        return torch.zeros_like(b), {"converged": True, "iterations": 0, "history": hist}
    target = rel_tol * bnorm
    its = 0
    m = restart
    while its < max_iters:
        r = b - (0.0 + A.apply(x))
        rn = dot(r, r) ** 0.5
        if rn <= target:
            hist.append(rn / bnorm)
            return x, {"converged": True, "iterations": its, "history": hist}
        V = [r / rn]
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = rn
        k = 0
        happy = False
        while k < m and its < max_iters:
            w = 0.0 + A.apply(M(V[k]))
            w0 = dot(w, w) ** 0.5
            for i in range(k + 1):
                h = dot(V[i], w)
                H[i, k] = h
                w = w - h * V[i]
            if dot(w, w) ** 0.5 < w0 / np.sqrt(2.0):
                for i in range(k + 1):
                    h = dot(V[i], w)
                    H[i, k] += h
                    w = w - h * V[i]
            H[k + 1, k] = dot(w, w) ** 0.5
            happy = H[k + 1, k] < 1e-300
            if not happy:
                V.append(w / H[k + 1, k])
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            a, c = H[k, k], H[k + 1, k]
            rr = float(np.hypot(a, c))
            cs[k], sn[k] = (1.0, 0.0) if rr == 0.0 else (a / rr, c / rr)
            H[k, k], H[k + 1, k] = rr, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            its += 1
            k += 1
            hist.append(abs(g[k]) / bnorm)
            if happy or abs(g[k]) <= target:
                break
        y = np.linalg.solve(np.triu(H[:k, :k]), g[:k]) if k else np.zeros(0)
        upd = torch.zeros_like(b)
        for j in range(k):
            upd = upd + V[j] * float(y[j])
        x = x + M(upd)
        rt = b - (0.0 + A.apply(x))
        tn = dot(rt, rt) ** 0.5
        hist.append(tn / bnorm)
        if tn <= target:
            return x, {"converged": True, "iterations": its, "history": hist}
        if happy:
            raise RuntimeError("gmres: Arnoldi breakdown before reaching tolerance")
    return x, {"converged": False, "iterations": its, "history": hist}
