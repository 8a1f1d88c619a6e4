"""The CPU oracle is pinned against the reference's golden outputs and the
algorithmic properties the reference's SPEC lists for linsolve."""

import numpy as np
import pytest
import scipy.sparse as sp

import refbridge as rb
from conftest import get_case, load_golden
from golden_util import vector_checksums

from oracle import linsolve_oracle as orc
from paper_1904_02401_b200 import workloads as W

SMALL = ["2d_mini", "2d_one", "3d_tiny", "3d_slab_multi"]


@pytest.mark.parametrize("name", SMALL)
def test_oracle_reproduces_reference_gmres(name):
    g, arr = load_golden(name)
    case = get_case(name)
    wl = W.CONFIGS[name]
    np.testing.assert_array_equal(case.b, arr["b"])
    x, st = orc.solve_case(case, wl)
    assert st.iterations == g["iterations"]
    r, rr = np.array(st.residuals), np.array(g["residuals"])
    assert np.max(np.abs(r - rr) / rr) < 1e-10
    assert np.linalg.norm(x - arr["x"]) <= 1e-9 * np.linalg.norm(arr["x"])


@pytest.mark.parametrize("name", SMALL)
def test_oracle_vcycle_and_sweep_match_reference(name):
    _, arr = load_golden(name)
    case = get_case(name)
    wl = W.CONFIGS[name]
    mg = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega)
    z = mg.dot(case.b)
    assert np.linalg.norm(z - arr["vcycle"]) <= 1e-11 * np.linalg.norm(arr["vcycle"])
    A, sm = mg.A[-1], mg.smoothers[-1]
    s2 = sm.sweep(A, sm.sweep(A, np.zeros_like(case.b), case.b), case.b)
    assert np.linalg.norm(s2 - arr["sweep2"]) <= 1e-12 * np.linalg.norm(arr["sweep2"])


def test_gmres_identity_converges_in_one_iteration():
    b = np.random.default_rng(0).standard_normal(20)
    x, st = orc.gmres(sp.identity(20, format="csr"), b, rel_tol=1e-12)
    assert st.iterations == 1
    np.testing.assert_allclose(x, b, rtol=1e-14)


def test_gmres_random_spd_matches_dense_solve_and_is_monotone():
    rng = np.random.default_rng(1)
    Q = rng.standard_normal((10, 10))
    A = Q @ Q.T + 10 * np.eye(10)
    b = rng.standard_normal(10)
    x, st = orc.gmres(A, b, rel_tol=1e-14, max_iter=10)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-10)
    res = np.array(st.residuals)
    assert np.all(np.diff(res) <= 1e-14 * res[0])


def test_gmres_raises_when_stalled():
    A = np.diag(np.arange(1.0, 101.0))
    b = np.ones(100)
    with pytest.raises(orc.OracleSolverError):
        orc.gmres(A, b, rel_tol=1e-14, max_iter=3)


def test_vcycle_is_linear():
    case = get_case("2d_mini")
    wl = W.CONFIGS["2d_mini"]
    mg = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega)
    rng = np.random.default_rng(3)
    b1, b2 = rng.standard_normal(len(case.b)), rng.standard_normal(len(case.b))
    lhs = mg.dot(2.0 * b1 - 0.5 * b2)
    rhs = 2.0 * mg.dot(b1) - 0.5 * mg.dot(b2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_single_global_patch_solves_in_one_sweep():
    """One patch covering all dofs with omega=1 is an exact solve (SPEC)."""
    from paper_1904_02401_b200 import mesh as mm
    case = get_case("2d_mini")
    A = case.matrices[0]
    n = A.n_nodes
    ps = mm.PatchSet(n_comp=A.nc)
    ps.add(np.arange(n)[None, :], 0)
    sm = orc.VankaOracle(ps, omega=1.0)
    sm.factorize(A)
    Acsr = A.to_csr()
    b = np.random.default_rng(4).standard_normal(Acsr.shape[0])
    x = sm.sweep(Acsr, np.zeros_like(b), b)
    assert np.linalg.norm(b - Acsr @ x) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("name", ["2d_small"])
def test_oracle_full_size_history(name):
    """Config 0 at full size (~200k dofs): iteration count and residual
    history of the reference's own run."""
    import os
    from conftest import GOLDEN
    if not os.path.exists(os.path.join(GOLDEN, f"{name}.json")):
        pytest.skip("golden file not generated")
    g, _ = load_golden(name)
    case = get_case(name)
    x, st = orc.solve_case(case, W.CONFIGS[name])
    assert st.iterations == g["iterations"]
    r, rr = np.array(st.residuals), np.array(g["residuals"])
    assert np.max(np.abs(r - rr) / rr) < 1e-10
    np.testing.assert_allclose(vector_checksums(x), g["x_checksums"], rtol=1e-9)


@pytest.mark.skipif(not rb.AVAILABLE, reason="reference not mounted")
def test_oracle_vs_live_reference_sweep_weights():
    """Multiplicity weights equal the reference smoother's weights."""
    wl = W.CONFIGS["2d_mini"]
    case = get_case("2d_mini")
    rp = rb.ref_problem(wl)
    stack = rb.ref_stack(wl, rp, case.U, case.U_prev)
    sm_ref = stack.mom_smoothers[-1]
    sm = orc.VankaOracle(case.patches[-1], wl.omega)
    for a, b in zip(sm.weights, sm_ref.weights):
        np.testing.assert_array_equal(a, b)


def test_oracle_accepts_precomputed_patch_inverses():
    """bench.py's cpu_baseline feeds the device's patch inverses to the oracle
    V-cycle instead of refactorising on the CPU: same V-cycle."""
    from conftest import get_case
    case = get_case("2d_mini")
    mg1 = orc.MgOracle(case)
    inv = [None] + [sm.inverses for sm in mg1.smoothers[1:]]
    mg2 = orc.MgOracle(case, inverses=inv)
    np.testing.assert_array_equal(mg1.dot(case.b), mg2.dot(case.b))
