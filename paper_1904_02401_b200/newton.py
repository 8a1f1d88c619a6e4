"""Linear-stack entry points of the approximated Newton solver.

Mirror of the reference's newton module solver entry points (reference
pkg/src/alefsi/newton.py): ``LinearConfig`` (newton.py:42-56) and
``LinearStack`` (newton.py:91-165), whose ``build_momentum`` assembles the
condensed Jacobian on every level and factorises the Vanka smoothers, and
whose ``solve_momentum`` runs GMRES + V-cycle — here on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

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
        self.last_rate = float("inf")

    def build_momentum(self, U, U_prev, k, theta):
        """Assemble the reduced momentum Jacobian on every level and factorise
        the smoothers on the device (reference newton.py:134-151)."""
        p = self.problem
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
        return linsolve.gmres(self.mom_mg.levels[-1].matrix, b, self.mom_mg,
                              rel_tol=self.cfg.momentum_rel_tol, max_iter=self.cfg.max_iter)
