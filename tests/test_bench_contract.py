"""bench.py's parity gate and the reference arm's inputs (CPU only)."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden

sys.path.insert(0, os.path.join(ROOT, "baseline"))

import bench  # noqa: E402
import ref_arm  # noqa: E402

from paper_1904_02401_b200 import mesh as mm, workloads as W  # noqa: E402


def test_bench_golden_gate_rejects_a_wrong_history():
    """bench.py refuses to print a line whose warm-up history differs from
    the committed golden."""
    g, _ = load_golden("3d_large")
    ok = bench.check_against_golden("3d_large", g["iterations"], g["residuals"],
                                    g["x_checksums"])
    assert ok["source"].endswith("3d_large.json")      # the reference's own run
    go, _ = load_golden("3d_large_oracle")             # the pinned oracle agrees
    bench.check_against_golden("3d_large", go["iterations"], go["residuals"], go["x_checksums"])
    bad = list(g["residuals"])
    bad[3] *= 1 + 1e-8
    with pytest.raises(bench.ParityError):
        bench.check_against_golden("3d_large", g["iterations"], bad, None)
    with pytest.raises(bench.ParityError):
        bench.check_against_golden("3d_large", g["iterations"] + 1, g["residuals"] + [1e-9], None)
    xc = list(g["x_checksums"])
    xc[0] *= 1 + 1e-7
    with pytest.raises(bench.ParityError):
        bench.check_against_golden("3d_large", g["iterations"], g["residuals"], xc)
    # the reference's own golden wins where it exists
    assert bench.golden_for("3d_small")[0].endswith("3d_small.json")


def test_bench_vector_checksums_match_golden_util():
    from golden_util import vector_checksums
    x = np.random.default_rng(5).standard_normal(1000)
    assert bench.vector_checksums(x) == vector_checksums(x)


@pytest.mark.parametrize("name", sorted(ref_arm.SPECS))
def test_ref_arm_workload_is_the_device_workload(name):
    """The reference arm restates the workload without importing the
    product package; its coarse mesh arrays and parameters are the same."""
    wl = W.CONFIGS[name]
    spec = ref_arm.SPECS[name]
    v, c, s, f = ref_arm.box_arrays(spec["lengths"], spec["coarse"])
    m = mm.box_mesh(wl.lengths, wl.coarse_cells)
    np.testing.assert_array_equal(v, m.vertices)
    np.testing.assert_array_equal(c, m.cells)
    for key, arr in f.items():
        np.testing.assert_array_equal(arr, m.facets[key])
    assert set(f) == {k for k, a in m.facets.items() if len(a)}
    assert spec["levels"] == wl.n_levels and spec["taper"] == wl.deform_taper
    lo, hi = ref_arm.solid_box(spec["dim"], spec.get("solid"))
    assert tuple(spec.get("patches", wl.patch_strategies())) == wl.patch_strategies()
    wlo, whi = wl.solid_box()
    np.testing.assert_array_equal(lo, wlo)
    np.testing.assert_array_equal(hi, whi)
    assert ref_arm.DT == wl.dt and ref_arm.THETA == wl.theta
    assert ref_arm.REL_TOL == wl.rel_tol and ref_arm.MAX_ITER == wl.max_iter


@pytest.mark.skipif(not ref_arm.available(), reason="reference not installed in baseline/_ref")
def test_ref_arm_state_rhs_and_threaded_setup_are_exact():
    """State/RHS equal the device arm's; the setup-only einsum split (forced
    on a small case) leaves the reference's operators and patch inverses
    bitwise unchanged; the installed reference solves to the golden."""
    name = "2d_mini"
    s1, b1, _ = ref_arm.build(name, setup_threads=1)
    s4, b4, _ = ref_arm.build(name, setup_threads=4, min_batch=8)
    np.testing.assert_array_equal(b1, b4)
    for l1, l4 in zip(s1.mom_mg.levels, s4.mom_mg.levels):
        assert (l1.matrix != l4.matrix).nnz == 0
        np.testing.assert_array_equal(l1.matrix.data, l4.matrix.data)
    for sm1, sm4 in zip(s1.mom_smoothers[1:], s4.mom_smoothers[1:]):
        for i1, i4 in zip(sm1.inverses, sm4.inverses):
            np.testing.assert_array_equal(i1, i4)
    g, arr = load_golden(name)
    np.testing.assert_array_equal(b1, arr["b"])
    x, st = ref_arm.solve(s4, b4)
    assert st.iterations == g["iterations"]
    np.testing.assert_allclose(st.residuals, g["residuals"], rtol=1e-10)
    assert "paper_1904_02401_b200" not in ref_arm.ref().__file__


def test_clock_sampler_summary_contract():
    """The `clocks` object of the JSON line: keys present with and without a
    device (no samples here), and the nvidia-smi line parser (median SM clock,
    max clock, throttle reasons that were active in any sample)."""
    with bench.ClockSampler(0) as clk:
        pass
    s = clk.summary()
    assert set(s) >= {"sm_mhz", "sm_max_mhz", "reasons", "samples", "sampler"}
    clk.lines = ["1500, 1965, Not Active, Not Active, Not Active, Active",
                 "1700, 1965, Not Active, Not Active, Not Active, Not Active",
                 "1600, 1965, Not Active, Not Active, Not Active, Active"]
    s = clk.summary()
    assert s["sm_mhz"] == 1600 and s["sm_max_mhz"] == 1965 and s["samples"] == 3
    assert s["reasons"] == ["sw_power_cap"]
