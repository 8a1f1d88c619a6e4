"""Run the unmodified reference on a workload definition: the read-only
source tree ``/root/reference/pkg/src/alefsi`` in the build container, else
the copy installed into ``baseline/_ref`` (which travels to the GPU box).
Also used by ``tests/golden/make_golden.py`` to generate the committed
fixtures."""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
if not os.path.isdir(os.path.join(REF_SRC, "alefsi")):
    # GPU box: the unmodified reference installed into baseline/_ref travels
    REF_SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "baseline", "_ref")
AVAILABLE = os.path.isdir(os.path.join(REF_SRC, "alefsi"))


def ref():
    if not AVAILABLE:
        raise RuntimeError("reference not mounted")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import alefsi.mesh, alefsi.problem, alefsi.model, alefsi.newton, alefsi.linsolve  # noqa
    import alefsi
    return alefsi


def ref_problem(wl):
    """Reference FsiProblem for a workload (coarse arrays from box_mesh)."""
    a = ref()
    from paper_1904_02401_b200 import mesh as mm
    c = mm.box_mesh(wl.lengths, wl.coarse_cells)
    coarse = a.mesh.MeshLevel(c.dim, c.vertices, c.cells, c.cell_subdomain, c.facets)
    h = a.mesh.build_hierarchy(coarse, wl.n_levels - 1)
    lo, hi = wl.solid_box()
    for m in h.levels:
        cen = m.vertices[m.cells].mean(axis=1)
        inside = np.all((cen > np.asarray(lo)) & (cen < np.asarray(hi)), axis=1)
        m.cell_subdomain = np.where(inside, a.mesh.SOLID, a.mesh.FLUID).astype(np.int8)
    m0 = wl.materials()
    mats = a.model.MaterialParams(rho_f=m0.rho_f, nu_f=m0.nu_f, rho_s=m0.rho_s, mu_s=m0.mu_s,
                                  lam_s=m0.lam_s, body_force=m0.body_force)
    flags = a.problem.FsiFlags(lps_dt=wl.dt)
    return a.problem.FsiProblem(h, mats, flags)


def ref_timestepping(ts, n_steps=None, on_record=None):
    """The reference's own run_time_loop (newton.py:303-343) on a
    TimeStepping workload; returns (U, per-step records)."""
    a = ref()
    wl = ts.base
    prob = ref_problem(wl)
    prob.flags.extension_model = "harmonic"
    prob.inflow_fn = ts.inflow
    lin, nt, tl = ts.configs()
    if n_steps is not None:
        tl.t_end = n_steps * wl.dt
    rlin = a.newton.LinearConfig(momentum_rel_tol=lin.momentum_rel_tol,
                                 extension_rel_tol=lin.extension_rel_tol, max_iter=lin.max_iter,
                                 nu_pre=lin.nu_pre, nu_post=lin.nu_post, omega=lin.omega,
                                 fluid_patches=lin.fluid_patches, solid_patches=lin.solid_patches)
    rnt = a.newton.NewtonConfig(rel_tol=nt.rel_tol, abs_tol=nt.abs_tol, gamma=nt.gamma,
                                max_steps=nt.max_steps, max_halvings=nt.max_halvings)
    rtl = a.newton.TimeLoopConfig(k=tl.k, theta_rule=tl.theta_rule, t_start=tl.t_start,
                                  t_end=tl.t_end)
    records = []

    def cb(t, U, U_prev, k, theta, stats_list):
        records.append({"t": t,
                        "newton_steps": [s.steps for s in stats_list],
                        "assemblies": [s.assemblies for s in stats_list],
                        "momentum_iters": [list(s.momentum_iters) for s in stats_list],
                        "extension_iters": [list(s.extension_iters) for s in stats_list],
                        "residuals": [[float(r) for r in s.residuals] for s in stats_list]})
        if on_record is not None:
            on_record(records)
    state, _ = a.newton.run_time_loop(prob, rtl, rnt, rlin, on_step=cb)
    return state.U, records


def ref_stack(wl, prob, U, Up):
    a = ref()
    fp, spt = wl.patch_strategies()
    cfg = a.newton.LinearConfig(fluid_patches=fp, solid_patches=spt, nu_pre=wl.nu_pre,
                                nu_post=wl.nu_post, omega=wl.omega, max_iter=wl.max_iter)
    stack = a.newton.LinearStack(prob, cfg)
    stack.build_momentum(U, Up, wl.dt, wl.theta)
    return stack


def ref_solve(wl, stack, b):
    a = ref()
    mg = stack.mom_mg
    return a.linsolve.gmres(mg.levels[-1].matrix, b, mg, rel_tol=wl.rel_tol,
                            max_iter=wl.max_iter)
