"""Compulsory-traffic byte model of one whole MGR-GMRES solve.

The whole-solve roofline fraction the north_star asks for is
    frac = model_bytes(solve) / (t_solve * peak HBM GB/s).
The model counts each array an operation must read or write once (perfect
x-vector reuse), from the hierarchy's sizes only, so it is the same number
for this library, the CPU oracle and a reader recomputing it:

* CSR SpMV y = A x:      12 nnz + 4 (m+1) + 8 min(ncols, nnz) + 8 m
* residual b - A x:      SpMV + 8 m
* Jacobi / l1-Jacobi:    sweep 0 from zero 24 m; later sweeps SpMV + 16 m
* Gauss-Seidel sweep:    12 nnz + 4 (m+1) + 24 m (from zero); later sweeps
                         SpMV + 16 m
* AMG level (V-cycle):   pre + post smoother + 2 residuals + R SpMV +
                         P-add (SpMV + 16 m); coarsest: dense 8 m^2 + 24 m
* coarse AMG, c cycles:  c V-cycles + (c - 1) (residual + 16 m)
* MGR level, injection R: F-relax on A_FF + restricted residual
                         (12 nnz(A_CF) + 4(|C|+1) + 8|F| + 16|C|) +
                         prolongation (16|C| + 12 nnz(P_F) + 4(|F|+1) + 8|C|
                         + 16|F|); other R kinds: residual + R SpMV + P-add
* dense LU solve:        8 s^2 + 24 s per diagonal block s (block diagonal
                         coarse systems: the connected components)
* GMRES step k:          SpMV(A) + M^-1 + orthogonalisation:
                         MGS (ortho "mgs"): 24 n (k+1) + 32 n;
                         lagged CGS2 (ortho "cgs2", lowsync.cu): two sweeps
                         each reading V_0..V_{k-1}, U and w, the second
                         writing v_k and U: 16 n (k+3)
* per restart cycle:     initial residual + norm + scale (SpMV + 8n + 8n
                         + 16n; cgs2: no scale, r is U), V y (8 n k + 16 n),
                         M^-1, x += z (24 n)

Used by bench.py (`solve_roofline`). Walks the hierarchy through the public
dump API (sizes, plus the level operator pattern for nnz(A_CF))."""
from __future__ import annotations

import json

import numpy as np


def _spmv(nnz, m, ncols):
    return 12.0 * nnz + 4.0 * (m + 1) + 8.0 * min(ncols, nnz) + 8.0 * m


def _shape(H, path):
    d = H.dump(path)
    if isinstance(d, tuple):
        ptr, col, val, (rows, cols) = d
        return rows, cols, int(ptr[-1]), d
    return len(d), None, None, d


class SolveModel:
    def __init__(self, H, strategy_text: str):
        self.H = H
        self.st = json.loads(strategy_text)
        self.info = H.info()
        self._cache = {}
        self.m_prec = self._mgr_bytes()

    def _csr(self, path):
        if path not in self._cache:
            self._cache[path] = _shape(self.H, path)
        return self._cache[path]

    # -- smoothers ------------------------------------------------------
    def _smoother(self, spec, nnz, m, ncols, amg_prefix=None, amg_levels=0):
        kind = spec.get("kind", "jacobi")
        sweeps = int(spec.get("sweeps", 1))
        if kind in ("jacobi", "l1_jacobi"):
            return 24.0 * m + (sweeps - 1) * (_spmv(nnz, m, ncols) + 16.0 * m)
        if kind.startswith("hybrid_l1_gs") or kind == "gauss_seidel":
            first = 12.0 * nnz + 4.0 * (m + 1) + 24.0 * m
            return first + (sweeps - 1) * (_spmv(nnz, m, ncols) + 16.0 * m)
        if kind == "amg_vcycle" and amg_prefix is not None:
            v = self._vcycle(amg_prefix, amg_levels, spec.get("amg", {}))
            return sweeps * v + (sweeps - 1) * (_spmv(nnz, m, ncols) + 24.0 * m)
        # block-Jacobi / dense: a pass over the vectors plus the factors
        return 24.0 * m

    def _vcycle(self, prefix, nlev, amg):
        pre = amg.get("pre_smoother", {"kind": "hybrid_l1_gs", "sweeps": 1})
        post = amg.get("post_smoother", {"kind": "hybrid_l1_gs", "sweeps": 1})
        total = 0.0
        for k in range(nlev):
            m, nc, nnz, _ = self._csr(f"{prefix}.{k}.A")
            if k + 1 == nlev:
                total += 8.0 * m * m + 24.0 * m
                break
            pr, pc, pnnz, _ = self._csr(f"{prefix}.{k}.P")
            rr, rc, rnnz, _ = self._csr(f"{prefix}.{k}.R")
            total += self._smoother(pre, nnz, m, nc) + self._smoother(post, nnz, m, nc)
            total += 2.0 * (_spmv(nnz, m, nc) + 8.0 * m)
            total += _spmv(rnnz, rr, rc) + _spmv(pnnz, pr, pc) + 16.0 * m
        return total

    def _dense(self, path):
        m, _, _, (ptr, col, _, _) = self._csr(path)
        if m == 0:
            return 0.0
        try:
            import scipy.sparse as sp
            from scipy.sparse.csgraph import connected_components
            G = sp.csr_matrix((np.ones(len(col)), col, ptr), shape=(m, m))
            _, lab = connected_components(G, directed=False)
            sizes = np.bincount(lab).astype(np.float64)
        except Exception:
            sizes = np.array([float(m)])
        return float(np.sum(8.0 * sizes * sizes)) + 24.0 * m

    # -- MGR ------------------------------------------------------------
    def _mgr_bytes(self):
        levels = self.st.get("levels", [])
        total = 0.0
        for l, lv in enumerate(levels[: self.info["mgr_levels"]]):
            m, nc, nnz, (ptr, col, _, _) = self._csr(f"mgr.{l}.A")
            F = self.H.dump(f"mgr.{l}.F")
            C = self.H.dump(f"mgr.{l}.C")
            nf, ncc = len(F), len(C)
            isf = np.zeros(m, bool)
            isf[F] = True
            # A_FF pattern size (F-relax) and A_CF (restricted residual)
            rowf = np.repeat(isf, np.diff(ptr))
            colf = isf[col]
            nnz_ff = int(np.count_nonzero(rowf & colf))
            nnz_cf = int(np.count_nonzero(~rowf & colf))
            fr = lv.get("f_relax", {"kind": "jacobi", "sweeps": 1})
            total += self._smoother(fr, nnz_ff, nf, nf, f"mgr.{l}.frelax.amg",
                                    self.info["frelax_amg_levels"][l])
            pr, pc, pnnz, _ = self._csr(f"mgr.{l}.P")
            if lv.get("restrict", "injection") == "injection":
                total += 12.0 * nnz_cf + 4.0 * (ncc + 1) + 8.0 * nf + 16.0 * ncc
                total += 16.0 * ncc + 12.0 * (pnnz - ncc) + 4.0 * (nf + 1) + 8.0 * ncc + 16.0 * nf
            else:
                rr, rc, rnnz, _ = self._csr(f"mgr.{l}.R")
                total += _spmv(nnz, m, nc) + 8.0 * m + _spmv(rnnz, rr, rc)
                total += _spmv(pnnz, pr, pc) + 16.0 * m
        co = self.st.get("coarse", {"kind": "dense_lu"})
        if co.get("kind") == "amg_vcycle":
            c = int(co.get("cycles", 1))
            m, nc, nnz, _ = self._csr("mgr.coarse.A")
            v = self._vcycle("mgr.coarse.amg", self.info["coarse_amg_levels"], co.get("amg", {}))
            total += c * v + (c - 1) * (_spmv(nnz, m, nc) + 24.0 * m)
        else:
            total += self._dense("mgr.coarse.A")
        return total

    # -- GMRES ----------------------------------------------------------
    def solve_bytes(self, A_nnz: int, n: int, iterations: int, restart: int, ortho: str = "mgs") -> dict:
        spmv_a = _spmv(A_nnz, n, n)
        steps, cycles, left = 0.0, 0, iterations
        while left > 0:
            ks = min(left, restart)
            for k in range(ks):
                orth = 16.0 * n * (k + 3) if ortho == "cgs2" else 24.0 * n * (k + 1) + 32.0 * n
                steps += spmv_a + self.m_prec + orth
            cycles += 1
            steps += spmv_a + 8.0 * n + 8.0 * n + (0.0 if ortho == "cgs2" else 16.0 * n)  # r0, norm, v0
            steps += 8.0 * n * ks + 16.0 * n + self.m_prec + 24.0 * n  # x += M^-1 V y
            left -= ks
        steps += spmv_a + 8.0 * n + 8.0 * n  # final true residual
        return {"bytes": steps, "precond_bytes_per_apply": self.m_prec, "spmv_bytes": spmv_a,
                "restart_cycles": cycles, "ortho": ortho}
