"""Reference-named solver API (drop-in for reference pkg/src/alefsi/linsolve.py).

The objects keep the reference's names, argument meaning and error
behaviour, but every operation runs on the device through the C ABI:

=========================  ===========================  =====================
reference (linsolve.py)    here                         device entry point
=========================  ===========================  =====================
gmres            :41-115   gmres                        alefsi_gmres
KrylovStats      :31-38    KrylovStats                  -
SolverError      :25-28    SolverError                  ALEFSI_ERR_*
patch_factorize  :120-134  VankaSmoother.factorize      alefsi_mg_factorize
VankaSmoother    :137-178  VankaSmoother                alefsi_mg_vanka_sweep
prolongation     :183-216  prolongation                 alefsi_mg_set_prolongation
MgLevel          :221-226  MgLevel                      -
MgSolver         :229-270  MgSolver                     alefsi_mg_apply
build_*_patches  :273-281  build_*_patches              alefsi_color_patches
=========================  ===========================  =====================

Differences a caller can observe: ``MgLevel.matrix`` is a
``fem.SplitBlockMatrix`` (the reference passes a scipy CSR; use
``fem.SplitBlockMatrix`` built from the reference BlockPattern/data pair,
see INTEGRATION.md), and the smoother factorisation happens on the device
when the ``MgSolver`` is built.  There is no CPU execution path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import mesh as meshmod
from .device import DeviceMgSolver, KrylovStats, SolverError  # noqa: F401
from .transfer import prolongation  # noqa: F401


class VankaSmoother:
    """Damped additive Vanka smoother with exact patch inverses
    (reference linsolve.py:137-178); the inverses live in HBM."""

    def __init__(self, patchset, coloring=None, omega=0.8):
        self.patchset = patchset
        self.coloring = coloring
        self.omega = omega
        self.inverses = None          # device resident; see MgSolver.inverses
        self._owner = None
        self._level = None

    def factorize(self, pattern=None, data=None):
        """Patch inverses are computed on the device by MgSolver (this call
        only re-factorises an already attached hierarchy)."""
        if self._owner is not None:
            self._owner.factorize()

    def sweep(self, A, x, b):
        """x + omega * sum_i w_i R_i^T A_i^{-1} R_i (b - A x) on device tensors."""
        if self._owner is None:
            raise SolverError("VankaSmoother is not attached to an MgSolver")
        y = x.clone()
        self._owner.sweep(self._level, y, b)
        return y


@dataclass
class MgLevel:
    matrix: object = None            # fem.SplitBlockMatrix
    smoother: VankaSmoother = None
    P: object = None                 # scipy CSR prolongation from the coarser level
    constrained: np.ndarray = None   # flat dof mask where corrections vanish


class MgSolver(DeviceMgSolver):
    """V-cycle over device-resident per-level operators; level 0 is solved
    with a factorised coarse operator (reference linsolve.py:229-270)."""

    def __init__(self, levels, nu_pre=2, nu_post=2, use_graph=False):
        omega = next((lv.smoother.omega for lv in levels[1:] if lv.smoother), 0.8)
        spec = [{"matrix": lv.matrix, "patches": lv.smoother.patchset if lv.smoother else None,
                 "P": lv.P, "constrained": lv.constrained} for lv in levels]
        super().__init__(spec, nu_pre=nu_pre, nu_post=nu_post, omega=omega,
                         use_graph=use_graph)
        self.levels = levels
        for l, lv in enumerate(levels):
            if lv.smoother is not None:
                lv.smoother._owner, lv.smoother._level = self, l


def gmres(operator, b, preconditioner=None, rel_tol=1e-4, abs_tol=0.0, max_iter=200,
          reorth_threshold=1e-8):
    """Right-preconditioned GMRES without restart (reference linsolve.py:41-115).

    ``preconditioner`` must be the device ``MgSolver`` whose finest level is
    ``operator``; raises ``SolverError`` (with stats) when max_iter is
    exceeded, exactly like the reference."""
    if not isinstance(preconditioner, DeviceMgSolver):
        raise TypeError("the device GMRES needs the device MgSolver as preconditioner "
                        "(there is no CPU path)")
    fine = getattr(preconditioner, "levels", None)
    if fine is not None and operator is not fine[-1].matrix:
        raise ValueError("operator must be the finest-level matrix of the preconditioner")
    return preconditioner.gmres(b, rel_tol=rel_tol, abs_tol=abs_tol, max_iter=max_iter)


def build_momentum_patches(mesh, dim, strategy_fluid, strategy_solid):
    """(PatchSet, Coloring) of the (p, v) system (reference linsolve.py:273-276)."""
    ps = meshmod.build_patches(mesh, strategy_fluid, n_comp=dim + 1,
                               per_subdomain={meshmod.FLUID: strategy_fluid,
                                              meshmod.SOLID: strategy_solid})
    return ps, meshmod.color_patches(ps)


def build_extension_patches(mesh, dim, strategy):
    """(PatchSet, Coloring) of the mesh-extension system (linsolve.py:279-281)."""
    ps = meshmod.build_patches(mesh, strategy, n_comp=dim)
    return ps, meshmod.color_patches(ps)
