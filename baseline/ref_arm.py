"""Reference arm of ``bench.py``: the UNMODIFIED reference package
(``alefsi``, pure Python/numpy/scipy, installed into ``baseline/_ref`` by
``python -m pip install --no-index --no-build-isolation --find-links
/opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>``)
driven through its own public API on the same seeded workload as the
device arm:

    problem   alefsi.mesh.MeshLevel / build_hierarchy, alefsi.problem.FsiProblem
    setup     alefsi.newton.LinearStack(problem, LinearConfig(...)).build_momentum
              (reference newton.py:134-151: per-level Jacobian assembly,
              Vanka patch inverses, coarse splu)
    solve     alefsi.linsolve.gmres(A, b, MgSolver, rel_tol=1e-8)
              (reference linsolve.py:41-115 with MgSolver :229-270)

Nothing here imports ``paper_1904_02401_b200`` or loads its ``.so``.  The
workload definition (box mesh arrays, solid box, seeded sine-mode state and
right-hand side) is restated below; ``tests/test_ref_arm.py`` checks it is
bitwise the one ``paper_1904_02401_b200.workloads`` builds.

Threads: the timed solves use the reference's own knobs — its patch-solve
pool (``alefsi._parallel.set_threads``, reference _parallel.py:17) and the
BLAS thread pool.  The one-off setup (not timed) may additionally run
``numpy.einsum`` batch-split over threads (``threaded_einsum``): the
reference's assembly is einsum-bound and single-threaded, and without this
the config-3 setup alone would not fit a benchmark run; the split is along
the cell axis only, so every output element is computed by the same
sequence of operations (checked bitwise in tests/test_ref_arm.py).
"""

from __future__ import annotations

import contextlib
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def available():
    return os.path.isdir(os.path.join(REF_DIR, "alefsi"))


def ref():
    """Import the installed reference package (baseline/_ref)."""
    if not available():
        raise ImportError(f"reference not installed in {REF_DIR}")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import alefsi.linsolve  # noqa: F401
    import alefsi.mesh  # noqa: F401
    import alefsi.model  # noqa: F401
    import alefsi.newton  # noqa: F401
    import alefsi.problem  # noqa: F401
    import alefsi._parallel  # noqa: F401
    import alefsi
    # the unmodified reference: this install, or (tests in the build
    # container) the read-only source tree imported first by another test
    src = os.path.abspath(alefsi.__file__)
    if not (src.startswith(REF_DIR) or src.startswith("/root/reference/")):
        raise ImportError(f"alefsi resolved to {src}, not the reference")
    return alefsi


# -- workload definition (BASELINE configs 0-3; see paper_1904_02401_b200/workloads.py)

SPECS = {
    "2d_small": dict(dim=2, lengths=(4.0, 1.0), coarse=(32, 8), levels=4, taper=0.0),
    "2d_large": dict(dim=2, lengths=(4.0, 1.0), coarse=(32, 8), levels=6, taper=0.0625),
    "3d_small": dict(dim=3, lengths=(4.0, 1.0, 1.0), coarse=(8, 2, 2), levels=4, taper=0.0),
    "3d_large": dict(dim=3, lengths=(4.0, 1.0, 1.0), coarse=(8, 2, 2), levels=5, taper=0.0),
    "2d_mini": dict(dim=2, lengths=(4.0, 1.0), coarse=(8, 2), levels=3, taper=0.0),
    "3d_mini": dict(dim=3, lengths=(4.0, 1.0, 1.0), coarse=(8, 2, 2), levels=3, taper=0.0),
    # the reference's 3D default blocking (one-element fluid, 2x2x2-cell solid
    # macros) on a corner solid block nested in the coarse grid
    "3d_large_refblock": dict(dim=3, lengths=(4.0, 1.0, 1.0), coarse=(8, 2, 2), levels=5,
                              taper=0.0, solid=((1.0, 0.0, 0.0), (2.0, 0.5, 0.5)),
                              patches=("one", "multi")),
    "3d_mini_refblock": dict(dim=3, lengths=(4.0, 1.0, 1.0), coarse=(8, 2, 2), levels=3,
                             taper=0.0, solid=((1.0, 0.0, 0.0), (2.0, 0.5, 0.5)),
                             patches=("one", "multi")),
}
DT = 0.01
THETA = 0.5 + 2.0 * DT          # shifted Crank-Nicolson (reference newton.py:69-74)
REL_TOL = 1e-8
MAX_ITER = 250
SOLID_SNAP = 0.125


def solid_box(dim, box=None):
    lo = np.array(box[0] if box else [1.0, 0.4, 0.4][:dim])
    hi = np.array(box[1] if box else [2.0, 0.6, 0.6][:dim])
    s = SOLID_SNAP
    return np.floor(lo / s + 1e-9) * s, np.ceil(hi / s - 1e-9) * s


def box_arrays(lengths, cells_per_dim):
    """Coarse structured channel: vertices (x fastest), bilinear/trilinear
    cell connectivity, facets labelled inflow (x=0) / outflow (x=Lx) /
    wall — the arrays the reference's MeshLevel constructor takes."""
    L = [float(v) for v in lengths]
    n = [int(v) for v in cells_per_dim]
    dim = len(n)
    axes = [np.linspace(0.0, L[i], n[i] + 1) for i in range(dim)]
    grids = np.meshgrid(*axes[::-1], indexing="ij")
    verts = np.stack([g.reshape(-1) for g in grids[::-1]], axis=1)
    stride = np.cumprod([1] + [n[i] + 1 for i in range(dim - 1)])

    def vid(*ijk):
        return sum(stride[i] * ijk[i] for i in range(dim))

    if dim == 2:
        j, i = (a.reshape(-1) for a in np.meshgrid(np.arange(n[1]), np.arange(n[0]),
                                                    indexing="ij"))
        cells = np.stack([vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)], axis=1)
        jj, ii = np.arange(n[1]), np.arange(n[0])
        inflow = np.stack([vid(0, jj + 1), vid(0, jj)], axis=1)
        outflow = np.stack([vid(n[0], jj), vid(n[0], jj + 1)], axis=1)
        wall = np.stack([np.stack([vid(ii, 0), vid(ii + 1, 0)], axis=1),
                         np.stack([vid(ii + 1, n[1]), vid(ii, n[1])], axis=1)],
                        axis=1).reshape(-1, 2)
    else:
        k, j, i = (a.reshape(-1) for a in np.meshgrid(np.arange(n[2]), np.arange(n[1]),
                                                       np.arange(n[0]), indexing="ij"))
        cells = np.stack([vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k), vid(i, j + 1, k),
                          vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i + 1, j + 1, k + 1),
                          vid(i, j + 1, k + 1)], axis=1)
        kk, jj = (a.reshape(-1) for a in np.meshgrid(np.arange(n[2]), np.arange(n[1]),
                                                      indexing="ij"))

        def xface(x):
            return np.stack([vid(x, jj, kk), vid(x, jj + 1, kk), vid(x, jj + 1, kk + 1),
                             vid(x, jj, kk + 1)], axis=1)
        inflow, outflow = xface(0), xface(n[0])
        kk2, ii = (a.reshape(-1) for a in np.meshgrid(np.arange(n[2]), np.arange(n[0]),
                                                       indexing="ij"))

        def yface(y):
            return np.stack([vid(ii, y, kk2), vid(ii + 1, y, kk2), vid(ii + 1, y, kk2 + 1),
                             vid(ii, y, kk2 + 1)], axis=1)
        jj3, ii3 = (a.reshape(-1) for a in np.meshgrid(np.arange(n[1]), np.arange(n[0]),
                                                        indexing="ij"))

        def zface(z):
            return np.stack([vid(ii3, jj3, z), vid(ii3 + 1, jj3, z), vid(ii3 + 1, jj3 + 1, z),
                             vid(ii3, jj3 + 1, z)], axis=1)
        wall = np.concatenate([np.stack([yface(0), yface(n[1])], axis=1).reshape(-1, 4),
                               np.stack([zface(0), zface(n[2])], axis=1).reshape(-1, 4)])
    facets = {"inflow": inflow, "outflow": outflow, "wall": wall}
    return verts, cells.astype(np.int64), np.zeros(len(cells), dtype=np.int8), facets


def sine_field(rng, X, lengths, ncomp, n_modes=8):
    out = np.zeros((len(X), ncomp))
    dim = X.shape[1]
    for _ in range(n_modes):
        kv = rng.integers(1, 5, size=dim)
        amp = rng.normal(0.0, 0.1, size=ncomp)
        s = np.ones(len(X))
        for i in range(dim):
            s = s * np.sin(kv[i] * np.pi * X[:, i] / lengths[i])
        out += s[:, None] * amp[None, :]
    return out


def linearisation_state(spec, X, node_class, node_fluid=0):
    d = spec["dim"]
    rng = np.random.default_rng(0)
    U = np.zeros((len(X), 1 + 2 * d))
    U[:, 1:1 + d] = sine_field(rng, X, spec["lengths"], d)
    u = 0.01 * sine_field(rng, X, spec["lengths"], d)
    if spec["taper"] > 0:
        lo, hi = solid_box(d, spec.get("solid"))
        gap = np.maximum(np.maximum(lo - X, X - hi), 0.0)
        phi = np.maximum(0.0, 1.0 - np.linalg.norm(gap, axis=1) / spec["taper"])
        phi[node_class != node_fluid] = 1.0
        u *= phi[:, None]
    else:
        u[node_class == node_fluid] = 0.0
    U[:, 1 + d:] = u
    U[:, 0] = sine_field(rng, X, spec["lengths"], 1)[:, 0]
    return U, np.zeros_like(U)


def right_hand_side(spec, X, momentum_dirichlet):
    rng = np.random.default_rng(1)
    b = sine_field(rng, X, spec["lengths"], spec["dim"] + 1)
    b[momentum_dirichlet] = 0.0
    return b.reshape(-1)


# -- setup-only einsum threading ------------------------------------------------

@contextlib.contextmanager
def threaded_einsum(threads, min_batch=4096):
    """Within the block, ``numpy.einsum`` calls whose output's leading index
    also leads every operand that carries it are split along that (cell)
    axis over ``threads`` threads; everything else runs unchanged."""
    if threads <= 1:
        yield
        return
    orig = np.einsum
    pool = ThreadPoolExecutor(max_workers=threads)
    lock = threading.Lock()

    def einsum(*operands, **kw):
        if kw or not operands or not isinstance(operands[0], str) or "." in operands[0] \
                or "->" not in operands[0]:
            return orig(*operands, **kw)
        subs, arrs = operands[0], operands[1:]
        ins, out = subs.replace(" ", "").split("->")
        ins = ins.split(",")
        if not out or len(ins) != len(arrs):
            return orig(*operands, **kw)
        lead = out[0]
        arrs = [np.asarray(a) for a in arrs]
        carry = [s.find(lead) for s in ins]
        if any(c > 0 for c in carry) or all(c < 0 for c in carry):
            return orig(*operands, **kw)
        n = next(a.shape[0] for a, c in zip(arrs, carry) if c == 0)
        if n < min_batch:
            return orig(*operands, **kw)
        step = -(-n // threads)
        bounds = [(s, min(s + step, n)) for s in range(0, n, step)]

        def part(se):
            s, e = se
            return orig(subs, *[a[s:e] if c == 0 else a for a, c in zip(arrs, carry)])
        with lock:
            parts = list(pool.map(part, bounds))
        return np.concatenate(parts, axis=0)

    np.einsum = einsum
    try:
        yield
    finally:
        np.einsum = orig
        pool.shutdown(wait=True)


# -- build + solve through the reference API -------------------------------------

def build(name, setup_threads=1, log=None, min_batch=4096):
    """Reference problem + LinearStack with the momentum Jacobian assembled
    and factorised (the state the timed solves start from)."""
    a = ref()
    spec = SPECS[name]
    d = spec["dim"]
    t0 = time.perf_counter()
    v, c, s, f = box_arrays(spec["lengths"], spec["coarse"])
    coarse = a.mesh.MeshLevel(d, v, c, s, f)
    h = a.mesh.build_hierarchy(coarse, spec["levels"] - 1)
    lo, hi = solid_box(d, spec.get("solid"))
    for m in h.levels:
        cen = m.vertices[m.cells].mean(axis=1)
        inside = np.all((cen > lo) & (cen < hi), axis=1)
        m.cell_subdomain = np.where(inside, a.mesh.SOLID, a.mesh.FLUID).astype(np.int8)
    mats, _ = a.model.MaterialParams(rho_f=1000.0, nu_f=1e-3, rho_s=1000.0, mu_s=5e5,
                                     lam_s=2e6, body_force=(0.0,) * d).density_scaled()
    flags = a.problem.FsiFlags(lps_dt=DT)
    one, multi = a.mesh.ONE_ELEMENT, a.mesh.MULTI_ELEMENT
    strat = multi if d == 2 else one
    fp, sp_ = spec.get("patches", (strat, strat))
    cfg = a.newton.LinearConfig(momentum_rel_tol=REL_TOL, max_iter=MAX_ITER, nu_pre=2,
                                nu_post=2, omega=0.8, fluid_patches=fp, solid_patches=sp_)
    with threaded_einsum(setup_threads, min_batch):
        prob = a.problem.FsiProblem(h, mats, flags)
        t1 = time.perf_counter()
        if log:
            log(f"[reference] problem {t1 - t0:.1f}s")
        fine = prob.fine
        U, Up = linearisation_state(spec, fine.mesh.nodes, fine.cls.node_class,
                                    a.mesh.NODE_FLUID)
        b = right_hand_side(spec, fine.mesh.nodes, fine.momentum_dirichlet)
        stack = a.newton.LinearStack(prob, cfg)
        t2 = time.perf_counter()
        if log:
            log(f"[reference] patches/transfers {t2 - t1:.1f}s")
        stack.build_momentum(U, Up, DT, THETA)
    t3 = time.perf_counter()
    if log:
        log(f"[reference] build_momentum {t3 - t2:.1f}s")
    return stack, b, {"problem": t1 - t0, "stack": t2 - t1, "build_momentum": t3 - t2}


def solve(stack, b):
    """One complete solve through the reference's stock GMRES + MgSolver."""
    a = ref()
    mg = stack.mom_mg
    return a.linsolve.gmres(mg.levels[-1].matrix, b, mg, rel_tol=REL_TOL, max_iter=MAX_ITER)


def set_solve_threads(threads):
    """The reference's own patch-solve thread pool (reference _parallel.py)."""
    ref()._parallel.set_threads(threads)
