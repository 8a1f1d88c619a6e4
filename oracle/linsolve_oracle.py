"""CPU oracle of the MG-GMRES / Vanka path (test infrastructure only).

Restates, in numpy/scipy, the reference's
  * gmres ............................. linsolve.py:41-115
  * patch_factorize ................... linsolve.py:120-134
  * VankaSmoother (weights, sweep) ..... linsolve.py:137-178
  * MgSolver (V-cycle, transfers) ...... linsolve.py:229-270
on the operators of a ``workloads.Case``.  The operator is taken as the
scalar CSR of the assembled Jacobian (like the reference's
``bsr.tocsr()``); patch blocks are gathered from it independently of the
device code.
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

CHUNK = 512


class OracleSolverError(Exception):
    def __init__(self, message, stats=None):
        super().__init__(message)
        self.stats = stats


@dataclass
class Stats:
    iterations: int = 0
    initial_residual: float = 0.0
    final_residual: float = 0.0
    elapsed: float = 0.0
    converged: bool = True
    residuals: list = field(default_factory=list)


def gmres(A, b, M=None, rel_tol=1e-4, abs_tol=0.0, max_iter=200):
    """Right-preconditioned unrestarted GMRES, classical Gram-Schmidt with
    the conditional second pass and Givens rotations (linsolve.py:41-115)."""
    t0 = time.perf_counter()
    Aop = A.dot if hasattr(A, "dot") else A
    Mop = (M.dot if hasattr(M, "dot") else M) if M is not None else (lambda v: v)
    b = np.asarray(b, dtype=float).ravel()
    beta = np.linalg.norm(b)
    st = Stats(initial_residual=beta, residuals=[beta])
    tol = max(rel_tol * beta, abs_tol)
    if beta == 0.0 or beta <= tol:
        st.final_residual = beta
        return np.zeros_like(b), st
    m = max_iter
    H = np.zeros((m + 1, m))
    cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
    g[0] = beta
    V = np.empty((m + 1, len(b)))
    V[0] = b / beta
    k = 0
    for k in range(m):
        w = Aop(Mop(V[k]))
        nb = np.linalg.norm(w)
        h = V[:k + 1] @ w
        w -= V[:k + 1].T @ h
        H[:k + 1, k] = h
        if np.linalg.norm(w) < 0.7071 * nb:
            h2 = V[:k + 1] @ w
            w -= V[:k + 1].T @ h2
            H[:k + 1, k] += h2
        H[k + 1, k] = np.linalg.norm(w)
        if H[k + 1, k] > 0:
            V[k + 1] = w / H[k + 1, k]
        for i in range(k):
            t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
            H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
            H[i, k] = t
        r = np.hypot(H[k, k], H[k + 1, k])
        cs[k], sn[k] = H[k, k] / r, H[k + 1, k] / r
        H[k, k] = r
        H[k + 1, k] = 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        res = abs(g[k + 1])
        st.residuals.append(res)
        if res <= tol:
            break
    st.iterations = k + 1
    st.final_residual = st.residuals[-1]
    y = np.linalg.solve(np.triu(H[:k + 1, :k + 1]), g[:k + 1])
    x = Mop(V[:k + 1].T @ y)
    st.elapsed = time.perf_counter() - t0
    if st.final_residual > tol:
        st.converged = False
        raise OracleSolverError(f"GMRES stalled at {st.final_residual:.3e}", st)
    return x, st


def _block_keys(pattern):
    rows = np.repeat(np.arange(pattern.n_nodes, dtype=np.int64), np.diff(pattern.indptr))
    return rows * pattern.n_nodes + pattern.indices


def dense_patch_blocks(A, node_groups):
    """Dense R_i A R_i^T for every patch of a homogeneous group
    (linsolve.py:120-129), gathered from the split operator by key lookup."""
    p, nc, n = A.pattern, A.nc, A.n_nodes
    bkeys = _block_keys(p)
    pkeys = (np.repeat(np.arange(n, dtype=np.int64), np.diff(p.pp_indptr)) * n
             + p.pp_indices)
    npn = node_groups.shape[1]
    out = np.zeros((len(node_groups), npn * nc, npn * nc))
    for s in range(0, len(node_groups), CHUNK):
        g = node_groups[s:s + CHUNK]
        keys = (g[:, :, None] * n + g[:, None, :]).reshape(-1)
        blk = np.zeros((len(keys), nc, nc))
        pos = np.searchsorted(bkeys, keys)
        hit = (pos < len(bkeys)) & (bkeys[np.minimum(pos, len(bkeys) - 1)] == keys)
        blk[hit] = A.data[pos[hit]]
        if len(pkeys):
            pos = np.searchsorted(pkeys, keys)
            hp = (pos < len(pkeys)) & (pkeys[np.minimum(pos, len(pkeys) - 1)] == keys)
            blk[hp, 0, 0] += A.pp_data[pos[hp]]
        blk = blk.reshape(len(g), npn, npn, nc, nc).transpose(0, 1, 3, 2, 4)
        out[s:s + len(g)] = blk.reshape(len(g), npn * nc, npn * nc)
    return out


class VankaOracle:
    """Damped additive Vanka with multiplicity weights (linsolve.py:137-178)."""

    def __init__(self, patchset, omega=0.8, threads=1):
        self.omega = omega
        self.nc = patchset.n_comp
        self.node_groups = [g for g, _ in patchset.groups]
        self.dofs = [(g[:, :, None] * self.nc + np.arange(self.nc)).reshape(len(g), -1)
                     for g in self.node_groups]
        n = 1 + max(int(d.max()) for d in self.dofs)
        mult = np.zeros(n)
        for d in self.dofs:
            np.add.at(mult, d.reshape(-1), 1.0)
        mult[mult == 0] = 1.0
        self.weights = [1.0 / mult[d] for d in self.dofs]
        self.inverses = None
        self.pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

    def factorize(self, A):
        self.inverses = []
        for g in self.node_groups:
            dense = dense_patch_blocks(A, g)
            try:
                self.inverses.append(np.linalg.inv(dense))
            except np.linalg.LinAlgError as exc:
                raise OracleSolverError(f"singular Vanka patch block: {exc}") from exc

    def _map(self, fn, chunks):
        if self.pool is None or len(chunks) <= 1:
            return [fn(c) for c in chunks]
        return list(self.pool.map(fn, chunks))

    def sweep(self, A, x, b):
        d = b - A @ x
        upd = np.zeros_like(x)
        for dofs, inv, wts in zip(self.dofs, self.inverses, self.weights):
            chunks = [slice(i, min(i + CHUNK, len(dofs))) for i in range(0, len(dofs), CHUNK)]

            def solve(sl, dofs=dofs, inv=inv, wts=wts):
                return wts[sl] * np.einsum("pij,pj->pi", inv[sl], d[dofs[sl]])
            for sl, y in zip(chunks, self._map(solve, chunks)):
                np.add.at(upd, dofs[sl].reshape(-1), y.reshape(-1))
        return x + self.omega * upd


class OracleOperator:
    """y = A x for the assembled operator: scipy block-CSR matvec over the
    cell-stencil blocks plus the scalar pressure extension (the reference's
    bsr.tocsr() matvec, without materialising the scalar CSR)."""

    def __init__(self, A, threads=1):
        p = A.pattern
        self.nc = A.nc
        self.shape = A.shape
        self.B = sp.bsr_matrix((A.data, p.indices, p.indptr), shape=A.shape)
        self.L = sp.csr_matrix((A.pp_data, p.pp_indices, p.pp_indptr),
                               shape=(p.n_nodes, p.n_nodes))

    def dot(self, x):
        y = self.B @ x
        if self.L.nnz:
            y[::self.nc] += self.L @ x[::self.nc]
        return y

    __matmul__ = dot


class MgOracle:
    """V-cycle with Vanka smoothing and a sparse-LU coarse solve
    (linsolve.py:229-270)."""

    def __init__(self, case=None, nu_pre=2, nu_post=2, omega=0.8, threads=1, levels=None,
                 inverses=None):
        """``inverses`` (optional): per level >= 1 the list of patch-group
        inverses to use instead of factorising (timing samples)."""
        self.nu_pre, self.nu_post = nu_pre, nu_post
        levels = levels if levels is not None else case.mg_levels()
        mats = [lv["matrix"] for lv in levels]
        self.nc = mats[0].nc
        self.A = [OracleOperator(m) for m in mats]
        self.P = [lv["P"] for lv in levels]
        self.constrained = [np.asarray(lv["constrained"]).reshape(-1) for lv in levels]
        self.smoothers = [None]
        for l in range(1, len(self.A)):
            sm = VankaOracle(levels[l]["patches"], omega, threads)
            if inverses is not None:
                sm.inverses = inverses[l]
            else:
                sm.factorize(mats[l])
            self.smoothers.append(sm)
        self.coarse_lu = spla.splu(sp.csc_matrix(mats[0].to_csr()))

    def dot(self, b):
        return self.cycle(len(self.A) - 1, np.asarray(b, dtype=float))

    def cycle(self, l, b):
        if l == 0:
            return self.coarse_lu.solve(b)
        A, sm = self.A[l], self.smoothers[l]
        x = np.zeros_like(b)
        for _ in range(self.nu_pre):
            x = sm.sweep(A, x, b)
        r = b - A @ x
        rc = (self.P[l].T @ r.reshape(-1, self.nc)).reshape(-1)
        rc[self.constrained[l - 1]] = 0.0
        zc = self.cycle(l - 1, rc)
        zf = (self.P[l] @ zc.reshape(-1, self.nc)).reshape(-1)
        zf[self.constrained[l]] = 0.0
        x += zf
        for _ in range(self.nu_post):
            x = sm.sweep(A, x, b)
        return x


class OracleLinearStack:
    """CPU counterpart of newton.LinearStack (reference newton.py:91-165) for
    the Newton-loop parity runs: same assembly, oracle MG-GMRES solves."""

    def __init__(self, problem, lin_cfg, threads=1):
        from paper_1904_02401_b200 import mesh as mm, transfer
        self.problem, self.cfg, self.threads = problem, lin_cfg, threads
        levels = problem.levels
        d = problem.dim
        self.transfers = [None] + [transfer.prolongation(levels[l - 1].mesh, levels[l].mesh)
                                   for l in range(1, len(levels))]
        fs, ss = lin_cfg.patch_strategies(d)
        self.mom_patches = [None] + [
            mm.build_patches(levels[l].mesh, fs, n_comp=d + 1,
                             per_subdomain={mm.FLUID: fs, mm.SOLID: ss})
            for l in range(1, len(levels))]
        self.ext_patches = [None] + [mm.build_patches(levels[l].mesh, mm.ONE_ELEMENT, n_comp=d)
                                     for l in range(1, len(levels))]
        self.mom_mg = None
        self.ext_mg = None
        self.last_rate = float("inf")

    def build_momentum(self, U, U_prev, k, theta):
        from paper_1904_02401_b200 import model
        p = self.problem
        levels = [{"matrix": model.momentum_jacobian(lvl, p.mats, p.flags, k, theta,
                                                     p.restrict_state(U, l),
                                                     p.restrict_state(U_prev, l)),
                   "patches": self.mom_patches[l], "P": self.transfers[l],
                   "constrained": lvl.momentum_dirichlet} for l, lvl in enumerate(p.levels)]
        self.mom_mg = MgOracle(None, self.cfg.nu_pre, self.cfg.nu_post, self.cfg.omega,
                               self.threads, levels=levels)

    def solve_momentum(self, b):
        return _solve(self.mom_mg, b, self.cfg.momentum_rel_tol, self.cfg.max_iter)

    def solve_extension(self, b):
        if self.ext_mg is None:
            p = self.problem
            levels = [{"matrix": p.extension_blocks(l)["bc"], "patches": self.ext_patches[l],
                       "P": self.transfers[l], "constrained": lvl.ext_dirichlet}
                      for l, lvl in enumerate(p.levels)]
            self.ext_mg = MgOracle(None, self.cfg.nu_pre, self.cfg.nu_post, self.cfg.omega,
                                   self.threads, levels=levels)
        return _solve(self.ext_mg, b, self.cfg.extension_rel_tol, self.cfg.max_iter)


def _solve(mg, b, rel_tol, max_iter):
    from paper_1904_02401_b200.device import SolverError
    try:
        return gmres(mg.A[-1], b, mg, rel_tol=rel_tol, max_iter=max_iter)
    except OracleSolverError as exc:
        raise SolverError(str(exc), exc.stats) from exc


def solve_case(case, wl, threads=1, mg=None):
    """GMRES(A_fine, b, V-cycle) exactly as LinearStack.solve_momentum does
    (reference newton.py:153-157)."""
    mg = mg or MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega, threads)
    return gmres(mg.A[-1], case.b, mg, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
