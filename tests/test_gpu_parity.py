"""Device path (C ABI, sm_100a kernels) vs the reference's golden outputs and
the CPU oracle.  Tolerances: GMRES residual histories 1e-10 relative with
identical iteration counts, solutions 1e-9 relative (north_star); operator
products and transfers 1e-13, one sweep / one V-cycle 1e-11 (FP64
summation-order differences only, amplified by the patch inverses)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, get_case, gpu_available, load_golden
from golden_util import vector_checksums

from oracle import linsolve_oracle as orc
from paper_1904_02401_b200 import device, workloads as W

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="no CUDA device")]

SMALL = ["2d_mini", "2d_one", "3d_tiny", "3d_slab_multi"]
_SOLVERS = {}


def solver_for(name, **kw):
    key = (name, tuple(sorted(kw.items())))
    if key not in _SOLVERS:
        case = get_case(name)
        _SOLVERS[key] = device.DeviceMgSolver.from_case(case, W.CONFIGS[name], **kw)
    return _SOLVERS[key]


def assert_history(st, residuals, iterations):
    assert st.iterations == iterations
    r, rr = np.array(st.residuals), np.array(residuals)
    assert np.max(np.abs(r - rr) / rr) < 1e-10


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("graph", [False, True])
def test_device_gmres_matches_reference_golden(name, graph):
    g, arr = load_golden(name)
    wl = W.CONFIGS[name]
    s = solver_for(name, use_graph=graph)
    x, st = s.gmres(arr["b"], rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    assert_history(st, g["residuals"], g["iterations"])
    assert np.linalg.norm(x - arr["x"]) <= 1e-9 * np.linalg.norm(arr["x"])


@pytest.mark.parametrize("name", SMALL)
def test_device_vcycle_matches_reference_and_oracle(name):
    """One V-cycle against the reference's output and the oracle's, both at
    1e-11 relative: the small-level kernels sum restriction rows and patch
    columns in split order, and the 108x108 patch inverses amplify that
    round-off to ~1e-12 of the output (3d_tiny)."""
    _, arr = load_golden(name)
    case = get_case(name)
    wl = W.CONFIGS[name]
    z = solver_for(name).dot(case.b)
    assert np.linalg.norm(z - arr["vcycle"]) <= 1e-11 * np.linalg.norm(arr["vcycle"])
    zo = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega).dot(case.b)
    assert np.linalg.norm(z - zo) <= 1e-11 * np.linalg.norm(zo)


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("name", SMALL)
def test_device_kernels_vs_oracle(name):
    import torch
    case = get_case(name)
    wl = W.CONFIGS[name]
    s = solver_for(name)
    mg = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega)
    rng = np.random.default_rng(7)
    for l in range(len(case.matrices)):
        A = mg.A[l]
        x = rng.standard_normal(A.shape[0])
        b = rng.standard_normal(A.shape[0])
        y = s.spmv(l, _t(x)).cpu().numpy()
        assert np.linalg.norm(y - A @ x) <= 1e-13 * np.linalg.norm(A @ x)
        d = s.spmv(l, _t(x), _t(b)).cpu().numpy()
        assert np.linalg.norm(d - (b - A @ x)) <= 1e-13 * np.linalg.norm(b - A @ x)
        if l == 0:
            xc = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
            s.coarse_solve(_t(b), xc)
            ref = mg.coarse_lu.solve(b)
            assert np.linalg.norm(xc.cpu().numpy() - ref) <= 1e-9 * np.linalg.norm(ref)
            continue
        # one Vanka sweep from a nonzero iterate (1e-11: column-split patch
        # products on small levels, amplified by the patch inverses)
        xs = _t(x)
        s.sweep(l, xs, _t(b))
        ref = mg.smoothers[l].sweep(A, x, b)
        assert np.linalg.norm(xs.cpu().numpy() - ref) <= 1e-11 * np.linalg.norm(ref)
        # stored inverses
        for gi, inv_ref in enumerate(mg.smoothers[l].inverses):
            inv = s.inverses(l, gi)
            assert np.max(np.abs(inv - inv_ref)) <= 1e-10 * np.max(np.abs(inv_ref))
        # transfers
        nc = case.matrices[l].nc
        P = case.prolongations[l]
        con_c = case.problem.levels[l - 1].momentum_dirichlet.reshape(-1)
        con_f = case.problem.levels[l].momentum_dirichlet.reshape(-1)
        rc = torch.empty(P.shape[1] * nc, dtype=torch.float64, device="cuda")
        s.restrict(l, _t(x), rc)
        ref = (P.T @ x.reshape(-1, nc)).reshape(-1)
        ref[con_c] = 0.0
        np.testing.assert_allclose(rc.cpu().numpy(), ref, rtol=1e-13, atol=1e-13)
        zc = rng.standard_normal(P.shape[1] * nc)
        xf = _t(x)
        s.prolong_add(l, _t(zc), xf)
        add = (P @ zc.reshape(-1, nc)).reshape(-1)
        add[con_f] = 0.0
        np.testing.assert_allclose(xf.cpu().numpy(), x + add, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("nu_pre,nu_post,omega", [(0, 1, 0.5), (1, 0, 1.0), (3, 2, 0.7)])
def test_device_vcycle_variants_vs_oracle(nu_pre, nu_post, omega):
    """Smoothing counts and damping are parameters of the reference MgSolver /
    VankaSmoother (linsolve.py:147, 232); every combination matches."""
    case = get_case("3d_tiny")
    s = device.DeviceMgSolver(case.mg_levels(), nu_pre=nu_pre, nu_post=nu_post, omega=omega)
    mg = orc.MgOracle(case, nu_pre, nu_post, omega)
    z, zo = s.dot(case.b), mg.dot(case.b)
    assert np.linalg.norm(z - zo) <= 1e-11 * np.linalg.norm(zo)
    x, st = s.gmres(case.b, rel_tol=1e-8, max_iter=250)
    xo, so = orc.gmres(mg.A[-1], case.b, mg, rel_tol=1e-8, max_iter=250)
    assert_history(st, so.residuals, so.iterations)
    s.close()


def test_single_level_hierarchy_is_a_direct_solve():
    """A one-level hierarchy is the coarse solve alone: GMRES converges in one
    iteration (SPEC: 'one-level hierarchy -> exact coarse solve')."""
    case = get_case("2d_mini")
    lv = case.mg_levels()[:1]
    s = device.DeviceMgSolver(lv)
    A = case.matrices[0].to_csr()
    b = np.random.default_rng(3).standard_normal(A.shape[0])
    x, st = s.gmres(b, rel_tol=1e-10, max_iter=5)
    assert st.iterations == 1
    assert np.linalg.norm(b - A @ x) <= 1e-9 * np.linalg.norm(b)
    s.close()


def test_reference_named_linear_stack_api():
    """newton.LinearStack / linsolve.gmres mirror the reference entry points
    (build_momentum + solve_momentum) and reproduce the golden history."""
    from paper_1904_02401_b200 import newton
    g, arr = load_golden("2d_mini")
    wl = W.CONFIGS["2d_mini"]
    case = get_case("2d_mini")
    fs, ss = wl.patch_strategies()
    cfg = newton.LinearConfig(momentum_rel_tol=wl.rel_tol, fluid_patches=fs, solid_patches=ss)
    stack = newton.LinearStack(case.problem, cfg)
    stack.build_momentum(case.U, case.U_prev, wl.dt, wl.theta)
    x, st = stack.solve_momentum(arr["b"])
    assert_history(st, g["residuals"], g["iterations"])
    assert np.linalg.norm(x - arr["x"]) <= 1e-9 * np.linalg.norm(arr["x"])


def test_device_gmres_is_deterministic_and_device_resident():
    import torch
    name = "3d_tiny"
    wl = W.CONFIGS[name]
    case = get_case(name)
    s = solver_for(name)
    b = _t(case.b)
    x1, st1 = s.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    x2, st2 = s.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    assert torch.equal(x1, x2)
    assert st1.residuals == st2.residuals
    xh, _ = s.gmres(case.b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    np.testing.assert_array_equal(xh, x1.cpu().numpy())


def test_device_gmres_not_converged_raises():
    name = "2d_mini"
    s = solver_for(name)
    case = get_case(name)
    with pytest.raises(device.SolverError) as exc:
        s.gmres(case.b, rel_tol=1e-14, max_iter=3)
    assert exc.value.stats.iterations == 3 and not exc.value.stats.converged


def test_zero_rhs_returns_zero():
    s = solver_for("2d_mini")
    case = get_case("2d_mini")
    x, st = s.gmres(np.zeros_like(case.b), rel_tol=1e-8)
    assert st.iterations == 0 and not x.any()


def test_device_gmres_tolerance_edges_vs_oracle():
    """Stopping rules of reference linsolve.py:55-60,107-115 on the device:
    tol = max(rel_tol * beta, abs_tol); beta <= tol returns zero after no
    iteration; an absolute tolerance alone stops at the oracle's iteration;
    a failed solve raises with the same partial history."""
    name = "3d_tiny"
    wl = W.CONFIGS[name]
    case = get_case(name)
    s = solver_for(name)
    mg = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega)
    beta = np.linalg.norm(case.b)
    # early return: abs_tol at beta (reference: beta <= tol); the device norm
    # is a fixed-order tree sum, equal to numpy's to the last bits only
    x, st = s.gmres(case.b, rel_tol=0.0, abs_tol=beta * (1 + 1e-12))
    assert st.iterations == 0 and not x.any() and len(st.residuals) == 1
    assert abs(st.residuals[0] - beta) <= 1e-14 * beta
    # absolute tolerance only
    xo, so = orc.gmres(mg.A[-1], case.b, mg, rel_tol=0.0, abs_tol=1e-6 * beta, max_iter=250)
    x, st = s.gmres(case.b, rel_tol=0.0, abs_tol=1e-6 * beta, max_iter=250)
    assert_history(st, so.residuals, so.iterations)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
    # the larger of the two tolerances wins
    _, st2 = s.gmres(case.b, rel_tol=1e-6, abs_tol=1e-12 * beta, max_iter=250)
    assert st2.iterations == so.iterations
    # iteration limit: same partial history as the oracle's failed solve
    with pytest.raises(orc.OracleSolverError) as eo:
        orc.gmres(mg.A[-1], case.b, mg, rel_tol=1e-14, max_iter=4)
    with pytest.raises(device.SolverError) as ed:
        s.gmres(case.b, rel_tol=1e-14, max_iter=4)
    assert_history(ed.value.stats, eo.value.stats.residuals, 4)
    # one iteration allowed and enough
    r1 = so.residuals[1]
    x1, st1 = s.gmres(case.b, rel_tol=0.0, abs_tol=r1 * (1 + 1e-6), max_iter=1)
    assert st1.iterations == 1 and st1.converged


@pytest.mark.parametrize("name", ["2d_small", "3d_small"])
def test_device_full_size_vs_reference_history(name):
    """BASELINE configs 0 and 2 at full size against the reference's own run."""
    if not os.path.exists(os.path.join(GOLDEN, f"{name}.json")):
        pytest.skip("golden file not generated")
    g, _ = load_golden(name)
    wl = W.CONFIGS[name]
    s = solver_for(name)
    x, st = s.gmres(get_case(name).b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    assert_history(st, g["residuals"], g["iterations"])
    np.testing.assert_allclose(vector_checksums(x), g["x_checksums"], rtol=1e-9)


@pytest.mark.parametrize("name", ["3d_large", "2d_large"])
def test_device_full_size_vs_oracle_history(name):
    """The headline 4.3M-dof solve (and the 3.2M-dof 2D config 1) against the CPU oracle's full-size run
    (tests/golden/make_oracle_golden.py; the oracle is pinned to the
    reference on every size the reference can run here)."""
    if not os.path.exists(os.path.join(GOLDEN, f"{name}_oracle.json")):
        pytest.skip("oracle golden file not generated")
    g, _ = load_golden(f"{name}_oracle")
    wl = W.CONFIGS[name]
    s = solver_for(name)
    x, st = s.gmres(get_case(name).b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    assert_history(st, g["residuals"], g["iterations"])
    np.testing.assert_allclose(vector_checksums(x), g["x_checksums"], rtol=1e-9)


def test_device_headline_size_properties():
    """3D 4.3M-dof workload (BASELINE config 3): size-independent checks —
    convergence with a monotone history, true residual, V-cycle linearity,
    bitwise determinism."""
    import torch
    name = "3d_large"
    wl = W.CONFIGS[name]
    s = solver_for(name)
    case = get_case(name)
    b = _t(case.b)
    x, st = s.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    res = np.array(st.residuals)
    assert st.converged and res[-1] <= wl.rel_tol * res[0]
    assert np.all(np.diff(res) <= 1e-12 * res[0])
    r = s.spmv(len(case.matrices) - 1, x, b)
    true_rel = float(torch.linalg.norm(r) / torch.linalg.norm(b))
    assert true_rel <= 10 * wl.rel_tol
    b2 = torch.roll(b, 17)
    lin = s.dot(2.0 * b - 0.5 * b2) - (2.0 * s.dot(b) - 0.5 * s.dot(b2))
    assert float(torch.linalg.norm(lin)) <= 1e-11 * float(torch.linalg.norm(s.dot(b)))
    x2, st2 = s.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    assert torch.equal(x, x2) and st.residuals == st2.residuals


@pytest.mark.parametrize("name", ["2d_mini", "3d_tiny"])
def test_singular_patch_and_coarse_block_are_reported(name):
    """A node row of zeros makes every patch containing it singular: the
    factorisation fails with ALEFSI_ERR_SINGULAR (reference linsolve.py:
    132-133 raises for a singular patch block) instead of producing NaNs;
    the same row on the coarse level trips the dense inverse's zero pivot."""
    import copy
    from paper_1904_02401_b200 import _lib
    case = get_case(name)
    wl = W.CONFIGS[name]
    for level in (len(case.matrices) - 1, 0):
        levels = case.mg_levels()
        A = copy.deepcopy(levels[level]["matrix"])
        p = A.pattern
        r = p.n_nodes // 2
        A.data[p.indptr[r]:p.indptr[r + 1]] = 0.0
        A.pp_data[p.pp_indptr[r]:p.pp_indptr[r + 1]] = 0.0
        levels[level] = dict(levels[level], matrix=A)
        with pytest.raises(_lib.NativeError) as exc:
            device.DeviceMgSolver(levels, nu_pre=wl.nu_pre, nu_post=wl.nu_post, omega=wl.omega)
        assert exc.value.code == 3, str(exc.value)


@pytest.mark.parametrize("name", ["2d_mini", "2d_one"])
def test_sliced_ell_layouts_vs_oracle(name):
    """Every 2D SpMV layout (CSR half-warp; sliced ELL with 1, 2, 4 lanes per
    row, alefsi_mg_set_sell) on every level: y = A x and y = b - A x within
    1e-13 of the oracle's operator product (only the order in which a row's
    blocks are summed differs)."""
    case = get_case(name)
    wl = W.CONFIGS[name]
    s = device.DeviceMgSolver.from_case(case, wl)
    mg = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega)
    rng = np.random.default_rng(11)
    try:
        for l in range(len(case.matrices)):
            A = mg.A[l]
            x = rng.standard_normal(A.shape[0])
            b = rng.standard_normal(A.shape[0])
            ref, refd = A @ x, b - A @ x
            for lanes in (0, 1, 2, 4):
                s.set_sell(l, lanes)
                y = s.spmv(l, _t(x)).cpu().numpy()
                assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref), (l, lanes)
                d = s.spmv(l, _t(x), _t(b)).cpu().numpy()
                assert np.linalg.norm(d - refd) <= 1e-13 * np.linalg.norm(refd), (l, lanes)
        # a re-laid-out hierarchy still solves to the golden history
        g, arr = load_golden(name)
        xs, st = s.gmres(arr["b"], rel_tol=wl.rel_tol, max_iter=wl.max_iter)
        assert_history(st, g["residuals"], g["iterations"])
    finally:
        s.close()


@pytest.mark.parametrize("name", ["2d_mini", "3d_tiny"])
def test_graph_solve_edge_cases_match_host_stepped(name):
    """The one-graph-per-solve GMRES (conditional while node) and the
    host-stepped loop run the same kernels: identical results for a
    converged solve, a solve stopped by max_iter (SolverError with the same
    partial history) and a zero right-hand side (x = 0, no iteration)."""
    case = get_case(name)
    wl = W.CONFIGS[name]
    sg = solver_for(name, use_graph=True)
    sh = solver_for(name)
    xg, stg = sg.gmres(case.b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    xh, sth = sh.gmres(case.b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    np.testing.assert_array_equal(xg, xh)
    assert stg.residuals == sth.residuals
    for s in (sg, sh):
        with pytest.raises(device.SolverError) as exc:
            s.gmres(case.b, rel_tol=1e-14, max_iter=3)
        assert exc.value.stats.iterations == 3 and not exc.value.stats.converged
        assert exc.value.stats.residuals == sth.residuals[:4]
        x0, st0 = s.gmres(np.zeros_like(case.b), rel_tol=1e-8)
        assert st0.iterations == 0 and not x0.any()
    # back to a full solve after the early stops: same result again
    xg2, stg2 = sg.gmres(case.b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    np.testing.assert_array_equal(xg2, xg)
