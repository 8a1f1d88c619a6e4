"""Parity of the exact path ``bench.py`` times: the hierarchy built by
``workloads.build_device_solver`` — host index structures, condensed
Jacobian ASSEMBLED ON THE DEVICE (reference model.py:297-381 through
LinearStack.build_momentum, newton.py:134-151), Vanka + coarse
factorisation on the device, graph-replayed V-cycle, device-resident RHS —
at the BASELINE sizes (configs 0-3).

Against the committed goldens:
* index structures (node numbering, union pattern, Dirichlet masks, patches,
  coloring, prolongation): SHA-256 equal to the reference's own
  (``{name}_setup.json``, tests/golden/make_golden.py --setup-only);
* the device-assembled operator on every level: seeded projections
  u^T A v within 1e-12 of the reference's (same file);
* GMRES: identical iteration count, residual history within 1e-10
  relative, solution checksums within 1e-9 (north_star), against the
  reference's own full-size run (configs 0 and 2 in the build container;
  configs 1 and 3 on the GPU box's host, tests/golden/make_golden_ref_arm.py,
  which also agree with the pinned CPU oracle's runs *_oracle.json).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, gpu_available, load_golden
from golden_util import operator_checksums, probe_vectors, sha, vector_checksums

from paper_1904_02401_b200 import fem, mesh as mm, workloads as W

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="no CUDA device")]

HISTORY = {"2d_small": "2d_small", "3d_small": "3d_small",
           "2d_large": "2d_large", "3d_large": "3d_large",
           # the reference's 3D default blocking (500x500 solid macro patches)
           "3d_mini_refblock": "3d_mini_refblock", "3d_large_refblock": "3d_large_refblock"}


def _build(name):
    import torch
    wl = W.CONFIGS[name]
    stream = torch.cuda.current_stream()
    prob, solver, b, _ = W.build_device_solver(wl, stream=stream.cuda_stream, use_graph=True)
    solver.reserve(wl.max_iter)
    return wl, prob, solver, b


def _device_projections(solver, level, n):
    """operator_checksums of the device-assembled operator: A v on the
    device (the product SpMV), u^T (A v) on the host."""
    import torch
    us = probe_vectors(n, 3, 1234)
    vs = probe_vectors(n, 3, 4321)
    out = []
    for u, v in zip(us, vs):
        y = solver.spmv(level, torch.from_numpy(v).cuda()).cpu().numpy()
        out.append(float(u @ y))
    return out


def _check_structures(name, prob, solver):
    src = f"{name}_setup"
    if not os.path.exists(os.path.join(GOLDEN, f"{src}.json")):
        src = name                       # full-detail golden of a small fixture
    g, _ = load_golden(src)
    if "levels" not in g:
        pytest.skip(f"no reference setup digests for {name}")
    assert len(g["levels"]) == len(prob.levels)
    for l, (lvl, rec) in enumerate(zip(prob.levels, g["levels"])):
        m = lvl.mesh
        assert lvl.n_nodes == rec["n_nodes"]
        assert sha(m.cell_nodes.astype(np.int64)) == rec["cell_nodes"], l
        assert sha(m.nodes.astype(np.float64)) == rec["node_coords"], l
        assert sha(lvl.cls.node_class.astype(np.int8)) == rec["node_class"], l
        ui, uj = fem.pattern_from_elements(
            lvl.n_nodes, [m.cell_nodes[lvl.fluid_cells], m.cell_nodes[lvl.solid_cells],
                          lvl.macro_nodes])
        assert sha(ui.astype(np.int64), uj.astype(np.int32)) == rec["union_pattern"], l
        assert sha(lvl.momentum_dirichlet.astype(np.uint8)) == rec["momentum_dirichlet"], l
        nc = lvl.dim + 1
        np.testing.assert_allclose(_device_projections(solver, l, lvl.n_nodes * nc),
                                   rec["operator"], rtol=1e-12, atol=1e-12)
        if l == 0:
            continue
        ps = solver.patches[l]
        assert [sha(gr.astype(np.int64)) for gr, _ in ps.groups] == rec["patches"], l
        assert [s for _, s in ps.groups] == rec["patch_subdomains"]
        col = mm.color_patches(ps)
        assert col.n_colors == rec["n_colors"]
        assert sha(col.color.astype(np.int64)) == rec["colors"], l
        P = solver.prolongations[l]
        assert sha(P.indptr.astype(np.int64), P.indices.astype(np.int32),
                   P.data.astype(np.float64)) == rec["prolongation"], l


def _check_solve(name, wl, solver, b):
    import torch
    g, _ = load_golden(HISTORY[name])
    b_dev = torch.from_numpy(b).cuda()
    x_dev = torch.empty_like(b_dev)
    for _ in range(2):          # second solve = a graph replay, as in the timed loop
        x, st = solver.gmres(b_dev, rel_tol=wl.rel_tol, max_iter=wl.max_iter, x_out=x_dev)
        assert st.iterations == g["iterations"]
        r, rr = np.array(st.residuals), np.array(g["residuals"])
        assert np.max(np.abs(r - rr) / rr) < 1e-10
        np.testing.assert_allclose(vector_checksums(x.cpu().numpy()), g["x_checksums"],
                                   rtol=1e-9)
    # end-to-end public call from host buffers: bitwise the device-resident result
    xh, sth = solver.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    np.testing.assert_array_equal(xh, x.cpu().numpy())
    assert sth.residuals == st.residuals


@pytest.mark.parametrize("name", list(HISTORY))
def test_benchmarked_path_matches_goldens(name):
    if not os.path.exists(os.path.join(GOLDEN, f"{HISTORY[name]}.json")):
        pytest.skip(f"golden {HISTORY[name]}.json not generated")
    wl, prob, solver, b = _build(name)
    try:
        _check_solve(name, wl, solver, b)
        _check_structures(name, prob, solver)
    finally:
        solver.close()
