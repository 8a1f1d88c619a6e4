"""Device assembly of the condensed Jacobian (reference model.py:297-381) vs
the host mirror (itself pinned to the reference to 1e-14): every level's
block data and pressure extension, and the solve it feeds."""

import numpy as np
import pytest

from conftest import get_case, gpu_available, load_golden

from paper_1904_02401_b200 import workloads as W

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="no CUDA device")]


@pytest.mark.parametrize("name", ["2d_mini", "2d_one", "3d_tiny", "3d_mini"])
def test_device_assembly_matches_host(name):
    wl = W.CONFIGS[name]
    case = get_case(name)
    prob, mg, b, _ = W.build_device_solver(wl)
    for l, lvl in enumerate(prob.levels):
        data, pp = mg.matrix_data(l, lvl.pattern)
        ref = case.matrices[l]
        scale = np.abs(ref.data).max()
        assert np.abs(data - ref.data).max() <= 1e-13 * scale, l
        if ref.pp_data.size:
            assert np.abs(pp - ref.pp_data).max() <= 1e-13 * np.abs(ref.pp_data).max(), l


@pytest.mark.parametrize("name", ["2d_mini", "3d_tiny"])
@pytest.mark.parametrize("ext", ["harmonic", "linear_elasticity"])
def test_device_residual_matches_host(name, ext):
    """Cell integrals of the theta residual and explicit forces on the device
    vs the host mirror (bitwise-pinned to the reference)."""
    from paper_1904_02401_b200 import model
    wl = W.CONFIGS[name]
    prob, mg, b, _ = W.build_device_solver(wl)
    prob.flags.extension_model = ext
    U, _ = W.linearisation_state(wl, prob)
    Up = 0.5 * U + 1e-3 * np.random.default_rng(5).standard_normal(U.shape)
    for l, lvl in enumerate(prob.levels):
        n = lvl.n_nodes
        R, ex = model.theta_residual(lvl, prob.mats, prob.flags, wl.dt, wl.theta, U[:n], Up[:n])
        Rd, exd = model.theta_residual(lvl, prob.mats, prob.flags, wl.dt, wl.theta, U[:n],
                                       Up[:n], device=(mg, l))
        assert np.abs(ex - exd).max() <= 1e-13 * max(1.0, np.abs(ex).max())
        assert np.abs(R - Rd).max() <= 1e-13 * max(1.0, np.abs(R).max())


@pytest.mark.parametrize("name", ["2d_mini", "3d_tiny"])
def test_device_assembled_solve_matches_reference(name):
    g, arr = load_golden(name)
    wl = W.CONFIGS[name]
    _, mg, b, _ = W.build_device_solver(wl)
    x, st = mg.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    assert st.iterations == g["iterations"]
    r, rr = np.array(st.residuals), np.array(g["residuals"])
    assert np.max(np.abs(r - rr) / rr) < 1e-10
    assert np.linalg.norm(x - arr["x"]) <= 1e-9 * np.linalg.norm(arr["x"])


@pytest.mark.parametrize("name", ["2d_mini", "3d_tiny"])
def test_reassembly_restarts_the_early_coarse_inverse(name):
    """Assembling level 0 starts the coarse inverse on the side stream
    (alefsi_mg_asm_momentum); assembling a different state and then the
    original one again, without a factorisation in between, must discard the
    stale inverses: the solve after one factorisation equals the golden."""
    g, arr = load_golden(name)
    wl = W.CONFIGS[name]
    prob, mg, b, _ = W.build_device_solver(wl)
    U, Up = W.linearisation_state(wl, prob)
    rng = np.random.default_rng(11)
    U2 = U.copy()
    U2[:, 1:1 + wl.dim] += 1e-2 * rng.standard_normal(U2[:, 1:1 + wl.dim].shape)
    for state in (U2, U):
        for l, lvl in enumerate(prob.levels):
            mg.asm_momentum(l, lvl, prob.mats, wl.dt, wl.theta, prob.restrict_state(state, l),
                            prob.restrict_state(Up, l))
    mg.factorize()
    x, st = mg.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    assert st.iterations == g["iterations"]
    r, rr = np.array(st.residuals), np.array(g["residuals"])
    assert np.max(np.abs(r - rr) / rr) < 1e-10
    assert np.linalg.norm(x - arr["x"]) <= 1e-9 * np.linalg.norm(arr["x"])
    # a second factorisation without reassembly (nothing in flight) gives the same solve
    mg.factorize()
    x2, st2 = mg.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    assert st2.iterations == st.iterations and np.array_equal(x2, x)
