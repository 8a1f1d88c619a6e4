"""INTEGRATION.md's reference-side binding (integration/_b200.py) inside the
UNMODIFIED reference: the reference's own ``LinearStack`` with its two
methods replaced (reference newton.py:134-157) — once for a single solve
and once under the reference's own ``run_time_loop`` (newton.py:303-343).

CPU tests check the binding's pure-numpy operator hand-over and that the
library exports every symbol it binds; the GPU tests run it."""

import importlib
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, gpu_available, load_golden

import refbridge as rb

sys.path.insert(0, os.path.join(ROOT, "integration"))

pytestmark = pytest.mark.skipif(not rb.AVAILABLE, reason="reference not available")


@pytest.fixture
def binding():
    return importlib.import_module("_b200")


@pytest.fixture
def patched(binding):
    """The reference's newton module with LinearStack patched; restored after."""
    a = rb.ref()
    orig = binding.install(a.newton)
    yield a
    a.newton.LinearStack.build_momentum, a.newton.LinearStack.solve_momentum = orig


def test_binding_symbols_exported(binding):
    for name in ("alefsi_mg_create", "alefsi_mg_set_matrix", "alefsi_mg_set_patches",
                 "alefsi_mg_set_prolongation", "alefsi_mg_set_constrained",
                 "alefsi_mg_factorize", "alefsi_mg_use_graph", "alefsi_gmres",
                 "alefsi_mg_destroy", "alefsi_last_error"):
        assert hasattr(binding.lib, name)


def test_split_is_an_exact_reencoding(binding):
    """The binding's hand-over of the reference's (pattern, data): blocks +
    scalar pressure extension reproduce the reference operator exactly."""
    from paper_1904_02401_b200 import workloads as W
    wl = W.CONFIGS["2d_mini"]
    a = rb.ref()
    prob = rb.ref_problem(wl)
    U, Up = W.linearisation_state(wl, prob)
    lvl = prob.fine
    data = a.model.momentum_jacobian_data(lvl, prob.mats, prob.flags, wl.dt, wl.theta, U, Up)
    A = lvl.pattern.to_bsr(data, wl.dim + 1).tocsr()
    ip, ix, d, pp, px, pd = binding.split(lvl.pattern, data)
    nc = wl.dim + 1
    import scipy.sparse as sp
    B = sp.bsr_matrix((d, ix, ip), shape=A.shape).tocsr()
    L = sp.csr_matrix((pd, px, pp), shape=(lvl.n_nodes, lvl.n_nodes)).tocoo()
    E = sp.csr_matrix((L.data, (L.row * nc, L.col * nc)), shape=A.shape)
    assert abs(A - (B + E)).max() == 0.0


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="no CUDA device")
def test_reference_linear_stack_with_binding_matches_golden(patched):
    from paper_1904_02401_b200 import workloads as W
    name = "2d_mini"
    g, arr = load_golden(name)
    wl = W.CONFIGS[name]
    prob = rb.ref_problem(wl)
    U, Up = W.linearisation_state(wl, prob)
    stack = rb.ref_stack(wl, prob, U, Up)          # patched build_momentum: GPU
    assert hasattr(stack, "mom_b200")
    stack.cfg.momentum_rel_tol = wl.rel_tol
    x, st = stack.solve_momentum(arr["b"])
    assert st.iterations == g["iterations"]
    np.testing.assert_allclose(st.residuals, g["residuals"], rtol=1e-10)
    assert np.linalg.norm(x - arr["x"]) <= 1e-9 * np.linalg.norm(arr["x"])


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="no CUDA device")
def test_reference_time_loop_with_binding(patched):
    """The reference's own run_time_loop on the 2D config-4 family fixture,
    momentum solves through the binding: same Newton steps and assemblies
    per time step as the reference's stock run (tests/golden/
    2d_timestep_mini.json), momentum GMRES counts within the reference's
    own run-to-run envelope (see test_timestepping.py)."""
    from paper_1904_02401_b200 import workloads as W
    g, _ = load_golden("2d_timestep_mini")
    ts = W.TIMESTEPPING["2d_timestep_mini"]
    U, records = rb.ref_timestepping(ts)
    assert len(records) == len(g["records"])
    for r, rg in zip(records, g["records"]):
        assert r["newton_steps"] == rg["newton_steps"]
        assert r["assemblies"] == rg["assemblies"]
        for a, b in zip(r["momentum_iters"], rg["momentum_iters"]):
            assert np.max(np.abs(np.array(a) - np.array(b))) <= 2
    np.testing.assert_allclose(np.linalg.norm(U), g["U_checksums"][0], rtol=1e-6)
