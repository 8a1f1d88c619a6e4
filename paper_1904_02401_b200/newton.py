"""Linear-stack entry points of the approximated Newton solver.

Mirror of the reference's newton module solver entry points (reference
pkg/src/alefsi/newton.py): ``LinearConfig`` (newton.py:42-56) and
``LinearStack`` (newton.py:91-165), whose ``build_momentum`` assembles the
condensed Jacobian on every level and factorises the Vanka smoothers, and
whose ``solve_momentum`` runs GMRES + V-cycle — here on the device.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import linsolve, model
from .mesh import MULTI_ELEMENT, ONE_ELEMENT
from .transfer import prolongation


@dataclass
class LinearConfig:
    momentum_rel_tol: float = 1e-4
    extension_rel_tol: float = 1e-8
    max_iter: int = 250
    nu_pre: int = 2
    nu_post: int = 2
    omega: float = 0.8
    fluid_patches: str = ""
    solid_patches: str = ""
    use_graph: bool = False
    device_assembly: bool = True      # assemble the Jacobian in HBM (else host numpy)

    def patch_strategies(self, dim):
        fluid = self.fluid_patches or (MULTI_ELEMENT if dim == 2 else ONE_ELEMENT)
        solid = self.solid_patches or MULTI_ELEMENT
        return fluid, solid


class LinearStack:
    """Per-level operators, smoothers and transfers, resident on the device."""

    def __init__(self, problem, lin_cfg: LinearConfig):
        self.problem = problem
        self.cfg = lin_cfg
        levels = problem.levels
        d = problem.dim
        self.transfers = [None] + [prolongation(levels[l - 1].mesh, levels[l].mesh)
                                   for l in range(1, len(levels))]
        fs, ss = lin_cfg.patch_strategies(d)
        self.mom_smoothers = [None]
        for l in range(1, len(levels)):
            ps, col = linsolve.build_momentum_patches(levels[l].mesh, d, fs, ss)
            self.mom_smoothers.append(linsolve.VankaSmoother(ps, col, lin_cfg.omega))
        self.mom_mg = None
        self.assembled = False
        self.last_rate = float("inf")

    def residual_device(self):
        """(device hierarchy, finest level) for device residual evaluation,
        or None with host assembly."""
        if not self.cfg.device_assembly:
            return None
        if self.mom_mg is None:
            self.mom_mg = self._device_hierarchy()
        return self.mom_mg, len(self.problem.levels) - 1

    def _device_hierarchy(self):
        """Device-resident momentum hierarchy with in-HBM assembly: patterns,
        patches, transfers and cell topology are uploaded once."""
        from .device import DeviceMgSolver
        p = self.problem
        spec = [{"pattern": lvl.pattern, "patches": self.mom_smoothers[l].patchset if l else None,
                 "P": self.transfers[l], "constrained": lvl.momentum_dirichlet.reshape(-1)}
                for l, lvl in enumerate(p.levels)]
        mg = DeviceMgSolver(spec, nu_pre=self.cfg.nu_pre, nu_post=self.cfg.nu_post,
                            omega=self.cfg.omega, use_graph=self.cfg.use_graph, factorize=False,
                            nc=p.dim + 1)
        for l, lvl in enumerate(p.levels):
            mg.asm_setup(l, lvl)
        return mg

    def build_momentum(self, U, U_prev, k, theta):
        """Assemble the reduced momentum Jacobian on every level and factorise
        the smoothers on the device (reference newton.py:134-151)."""
        p = self.problem
        self.assembled = True
        if self.cfg.device_assembly:
            if self.mom_mg is None:
                self.mom_mg = self._device_hierarchy()
            for l, lvl in enumerate(p.levels):
                self.mom_mg.asm_momentum(l, lvl, p.mats, k, theta, p.restrict_state(U, l),
                                         p.restrict_state(U_prev, l))
            self.mom_mg.factorize()
            return
        mg_levels = []
        for l, lvl in enumerate(p.levels):
            A = model.momentum_jacobian(lvl, p.mats, p.flags, k, theta,
                                        p.restrict_state(U, l), p.restrict_state(U_prev, l))
            mg_levels.append(linsolve.MgLevel(matrix=A, smoother=self.mom_smoothers[l],
                                              P=self.transfers[l],
                                              constrained=lvl.momentum_dirichlet.reshape(-1)))
        if self.mom_mg is not None:
            self.mom_mg.close()
        self.mom_mg = linsolve.MgSolver(mg_levels, self.cfg.nu_pre, self.cfg.nu_post,
                                        use_graph=self.cfg.use_graph)

    def solve_momentum(self, b):
        """GMRES + V-cycle on the finest momentum system (newton.py:153-157)."""
        if self.cfg.device_assembly:
            return self.mom_mg.gmres(b, rel_tol=self.cfg.momentum_rel_tol,
                                     max_iter=self.cfg.max_iter)
        return linsolve.gmres(self.mom_mg.levels[-1].matrix, b, self.mom_mg,
                              rel_tol=self.cfg.momentum_rel_tol, max_iter=self.cfg.max_iter)

    # extension stack: state independent, assembled and factorised once
    def _build_extension(self):
        p = self.problem
        d = p.dim
        levels = []
        for l, lvl in enumerate(p.levels):
            sm = None
            if l > 0:
                ps, col = linsolve.build_extension_patches(lvl.mesh, d, ONE_ELEMENT)
                sm = linsolve.VankaSmoother(ps, col, self.cfg.omega)
            levels.append(linsolve.MgLevel(matrix=p.extension_blocks(l)["bc"], smoother=sm,
                                           P=self.transfers[l],
                                           constrained=lvl.ext_dirichlet.reshape(-1)))
        # the extension operator never changes: its V-cycle is captured once
        # and replayed as a CUDA graph
        self.ext_mg = linsolve.MgSolver(levels, self.cfg.nu_pre, self.cfg.nu_post,
                                        use_graph=True)

    def solve_extension(self, b):
        """GMRES + V-cycle on the mesh-extension system (newton.py:159-165)."""
        if getattr(self, "ext_mg", None) is None:
            self._build_extension()
        return linsolve.gmres(self.ext_mg.levels[-1].matrix, b, self.ext_mg,
                              rel_tol=self.cfg.extension_rel_tol, max_iter=self.cfg.max_iter)


# ---------------------------------------------------------------------------------
# Approximated Newton iteration and time loop (reference newton.py:27-365)
# ---------------------------------------------------------------------------------

class StepFailure(Exception):
    def __init__(self, message, stats=None):
        super().__init__(message)
        self.stats = stats


@dataclass
class NewtonConfig:
    rel_tol: float = 1e-8
    abs_tol: float = 1e-8
    max_steps: int = 30
    gamma: float = 0.05
    max_halvings: int = 4


@dataclass
class TimeLoopConfig:
    k: float = 0.004
    theta_rule: str = "shifted_cn"
    t_start: float = 0.0
    t_end: float = 1.0


def theta_for(rule, k):
    if rule == "shifted_cn":
        return 0.5 + 2.0 * k
    if rule == "backward_euler":
        return 1.0
    return float(rule)


@dataclass
class NewtonStats:
    steps: int = 0
    assemblies: int = 0
    rates: list = field(default_factory=list)
    momentum_iters: list = field(default_factory=list)
    extension_iters: list = field(default_factory=list)
    residuals: list = field(default_factory=list)
    assemble_time: float = 0.0
    solve_time: float = 0.0
    residual_time: float = 0.0
    converged: bool = False


def solve_reduced_linear(problem, stack, R, U, U_prev, k, theta):
    """Three-stage exact solve of the reduced system (reference
    newton.py:168-201): momentum (device MG-GMRES), deformation update (vector
    addition), mesh extension (device MG-GMRES)."""
    lvl = problem.fine
    d = lvl.dim
    n = lvl.n_nodes
    x, mom_stats = stack.solve_momentum(-R[:, :d + 1].reshape(-1))
    dpv = np.asarray(x).reshape(n, d + 1)
    rel = lvl.relation_nodes
    Ur, Upr = U[rel], U_prev[rel]      # the deficit is needed on the relation nodes only
    deficit = (Ur[:, 1 + d:] - Upr[:, 1 + d:] - k * theta * Ur[:, 1:1 + d]
               - k * (1.0 - theta) * Upr[:, 1:1 + d])
    du = np.zeros((n, d))
    du[rel] = k * theta * dpv[rel, 1:] - deficit
    blocks = problem.extension_blocks(len(problem.levels) - 1)
    g = np.zeros((n, d))
    g[lvl.interface_nodes] = du[lvl.interface_nodes]
    if "interface_csr" not in blocks:
        blocks["interface_csr"] = interface_columns(blocks["raw"], lvl.interface_nodes, d)
    cols, sub = blocks["interface_csr"]
    rhs = -R[:, 1 + d:] / k - (sub @ g.reshape(-1)[cols]).reshape(n, d)
    rhs[lvl.ext_dirichlet] = 0.0
    z, ext_stats = stack.solve_extension(rhs.reshape(-1))
    W = np.zeros_like(U)
    W[:, :d + 1] = dpv
    W[:, 1 + d:] = np.asarray(z).reshape(n, d)
    W[lvl.interface_nodes, 1 + d:] = du[lvl.interface_nodes]
    W[rel, 1 + d:] = du[rel]
    W[lvl.u_dirichlet_nodes, 1 + d:] = 0.0
    return W, mom_stats, ext_stats


def interface_columns(raw, interface_nodes, d):
    """(cols, sub): the columns ``cols`` (interface node dofs, ascending) of
    the raw extension operator as a scalar CSR, built from the blocks whose
    column node is on the interface.  The lifting term ``g`` vanishes off the
    interface, so ``sub @ g[cols]`` equals the reference's full product row by
    row: same nonzeros, ascending columns, no explicit zeros."""
    import scipy.sparse as sp
    p = raw.pattern
    nodes = np.sort(np.asarray(interface_nodes))
    cols = (nodes[:, None] * d + np.arange(d)).reshape(-1)
    rank = np.full(p.n_nodes, -1, dtype=np.int64)
    rank[nodes] = np.arange(len(nodes))
    blk_col = rank[p.indices]
    sel = np.flatnonzero(blk_col >= 0)
    blk_row = np.repeat(np.arange(p.n_nodes), np.diff(p.indptr))[sel]
    a = np.arange(d)
    rows = (blk_row[:, None, None] * d + a[None, :, None]) + 0 * a[None, None, :]
    cc = (blk_col[sel][:, None, None] * d + a[None, None, :]) + 0 * a[None, :, None]
    sub = sp.csr_matrix((raw.data[sel].reshape(-1), (rows.reshape(-1), cc.reshape(-1))),
                        shape=(p.n_nodes * d, len(cols)))
    sub.sum_duplicates()
    sub.eliminate_zeros()
    sub.sort_indices()
    return cols, sub


def line_search(residual_of, U, W, res_norm, max_halvings=4):
    """Backtracking by halving on the residual sup-norm (newton.py:204-216)."""
    omega = 1.0
    for _ in range(max_halvings + 1):
        payload, res_try = residual_of(U + omega * W)
        if res_try <= res_norm:
            return omega, payload, res_try
        omega *= 0.5
    raise StepFailure("line search exhausted: residual would increase")


def newton_solve(problem, stack, U_guess, U_prev, k, theta, cfg: NewtonConfig):
    """Approximated Newton iteration for one time step (newton.py:219-273):
    reassemble the momentum Jacobian only when the last rate exceeds gamma."""
    lvl = problem.fine
    stats = NewtonStats()
    cache = [None]

    dev = stack.residual_device() if hasattr(stack, "residual_device") else None

    def residual_of(Ut):
        Ut = Ut.copy()
        model.deformation_update(Ut, U_prev, k, theta, lvl.relation_nodes)
        t0 = time.perf_counter()
        R, cache[0] = model.theta_residual(lvl, problem.mats, problem.flags, k, theta, Ut,
                                           U_prev, cache[0], device=dev)
        stats.residual_time += time.perf_counter() - t0
        return (Ut, R), float(np.abs(R).max())

    (U, R), res = residual_of(U_guess)
    stats.residuals.append(res)
    tol = max(cfg.abs_tol, cfg.rel_tol * res)
    while res > tol:
        if stats.steps >= cfg.max_steps:
            raise StepFailure(f"Newton did not converge in {cfg.max_steps} steps "
                              f"(residual {res:.3e})", stats)
        if not getattr(stack, "assembled", stack.mom_mg is not None) or \
                stack.last_rate > cfg.gamma:
            t0 = time.perf_counter()
            stack.build_momentum(U, U_prev, k, theta)
            stats.assemble_time += time.perf_counter() - t0
            stats.assemblies += 1
        t0 = time.perf_counter()
        try:
            W, ms, es = solve_reduced_linear(problem, stack, R, U, U_prev, k, theta)
        except linsolve.SolverError as exc:
            raise StepFailure(f"linear solve failed: {exc}", stats) from exc
        stats.solve_time += time.perf_counter() - t0
        stats.momentum_iters.append(ms.iterations)
        stats.extension_iters.append(es.iterations)
        try:
            _, (U, R), res_new = line_search(residual_of, U, W, res, cfg.max_halvings)
        except StepFailure as exc:
            exc.stats = stats
            raise
        rate = res_new / res if res > 0 else 0.0
        stack.last_rate = rate
        stats.rates.append(rate)
        stats.residuals.append(res_new)
        stats.steps += 1
        res = res_new
    stats.converged = True
    return U, stats


def run_time_loop(problem, tl: TimeLoopConfig, newton_cfg: NewtonConfig, stack,
                  U0=None, on_step=None):
    """Advance from t_start to t_end; a failing step is retried once as two
    half steps (reference newton.py:303-364).  Returns (U, per-step stats)."""
    if U0 is None:
        U0 = problem.zero_state()
        problem.impose_boundary_values(U0, tl.t_start)
    t = tl.t_start
    U_prev = U0
    all_stats = []
    while t < tl.t_end - 1e-12:
        k = min(tl.k, tl.t_end - t)
        t0 = time.perf_counter()
        U_n, sl = _advance(problem, stack, U_prev, t, k, tl, newton_cfg, True)
        wall = time.perf_counter() - t0
        t = t + k
        if on_step is not None:
            on_step(t, U_n, U_prev, k, theta_for(tl.theta_rule, k), sl, wall)
        all_stats.append((t, wall, sl))
        U_prev = U_n
    return U_prev, all_stats


def _advance(problem, stack, U_prev, t, k, tl, cfg, allow_halving):
    theta = theta_for(tl.theta_rule, k)
    guess = U_prev.copy()
    problem.impose_boundary_values(guess, t + k)
    try:
        U_n, stats = newton_solve(problem, stack, guess, U_prev, k, theta, cfg)
        return U_n, [stats]
    except StepFailure:
        stack.last_rate = float("inf")
        if not allow_halving:
            raise
        half = k / 2.0
        U_mid, s1 = _advance(problem, stack, U_prev, t, half, tl, cfg, False)
        U_n, s2 = _advance(problem, stack, U_mid, t + half, half, tl, cfg, False)
        return U_n, s1 + s2
