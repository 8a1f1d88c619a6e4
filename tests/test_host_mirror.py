"""Host-side mirror vs the reference: node numbering, patterns, patches,
coloring, prolongation (bit-exact via SHA-256 of the reference's arrays) and
the assembled condensed Jacobian (storage-independent projections)."""

import numpy as np
import pytest

import refbridge as rb
from conftest import get_case, load_golden
from golden_util import sha, operator_checksums

from paper_1904_02401_b200 import fem, mesh as mm, workloads as W

SMALL = ["2d_mini", "2d_one", "3d_tiny", "3d_slab_multi"]


@pytest.mark.parametrize("name", SMALL)
def test_index_structures_match_reference_digests(name):
    g, _ = load_golden(name)
    case = get_case(name)
    for l, (lvl, rec) in enumerate(zip(case.problem.levels, g["levels"])):
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
        if l == 0:
            continue
        ps = case.patches[l]
        assert [sha(gr.astype(np.int64)) for gr, _ in ps.groups] == rec["patches"], l
        assert [s for _, s in ps.groups] == rec["patch_subdomains"]
        assert case.colorings[l].n_colors == rec["n_colors"]
        assert sha(case.colorings[l].color.astype(np.int64)) == rec["colors"], l
        P = case.prolongations[l]
        assert sha(P.indptr.astype(np.int64), P.indices.astype(np.int32),
                   P.data.astype(np.float64)) == rec["prolongation"], l


@pytest.mark.parametrize("name", SMALL)
def test_assembled_operator_matches_reference_projections(name):
    g, _ = load_golden(name)
    case = get_case(name)
    for l, rec in enumerate(g["levels"]):
        mine = operator_checksums(case.matrices[l].to_csr())
        np.testing.assert_allclose(mine, rec["operator"], rtol=1e-12, atol=1e-12)


def test_coloring_is_sound_and_greedy():
    """Same-color patches share no dof (exhaustive), colors hold one size."""
    for name in SMALL:
        case = get_case(name)
        for l in range(1, len(case.problem.levels)):
            ps, col = case.patches[l], case.colorings[l]
            rows = [r for r in ps.patch_nodes()]
            sizes = np.array([len(r) for r in rows])
            for c in range(col.n_colors):
                members = np.flatnonzero(col.color == c)
                nodes = np.concatenate([rows[i] for i in members])
                assert len(np.unique(nodes)) == len(nodes)
                assert len(set(sizes[members])) == 1


def test_patch_sizes_of_strategies():
    m = mm.build_hierarchy(mm.box_mesh((4.0, 1.0), (4, 2)), 1).finest
    assert mm.build_patches(m, mm.ONE_ELEMENT, 3).sizes() == [27]
    assert mm.build_patches(m, mm.MULTI_ELEMENT, 3).sizes() == [75]
    m3 = mm.build_hierarchy(mm.box_mesh((4.0, 1.0, 1.0), (2, 1, 1)), 1).finest
    assert mm.build_patches(m3, mm.ONE_ELEMENT, 4).sizes() == [108]
    assert mm.build_patches(m3, mm.MULTI_ELEMENT, 4).sizes() == [500]


def test_split_layout_reencodes_union_layout():
    case = get_case("2d_mini")
    lvl = case.problem.fine
    A = case.matrices[-1]
    m = lvl.mesh
    ui, uj = fem.pattern_from_elements(lvl.n_nodes, [m.cell_nodes[lvl.fluid_cells],
                                                     m.cell_nodes[lvl.solid_cells],
                                                     lvl.macro_nodes])
    data = fem.union_layout(A, ui, uj)
    import scipy.sparse as sp
    B = sp.bsr_matrix((data, uj, ui), shape=A.shape).tocsr()
    assert abs(B - A.to_csr()).max() == 0.0
    # blocks outside the cell pattern only carry the pressure-pressure entry
    cell = set(zip(np.repeat(np.arange(lvl.n_nodes), np.diff(A.pattern.indptr)).tolist(),
                   A.pattern.indices.tolist()))
    rows = np.repeat(np.arange(lvl.n_nodes), np.diff(ui))
    for k in range(len(uj)):
        if (rows[k], uj[k]) not in cell:
            blk = data[k].copy()
            blk[0, 0] = 0.0
            assert not blk.any()


@pytest.mark.parametrize("name", ["2d_mini", "3d_tiny"])
def test_value_split_of_reference_layout_is_exact(name):
    """INTEGRATION.md's hand-over: a reference-layout (union pattern) operator
    split by value gives the same operator."""
    case = get_case(name)
    for l, lvl in enumerate(case.problem.levels):
        m = lvl.mesh
        ui, uj = fem.pattern_from_elements(lvl.n_nodes, [m.cell_nodes[lvl.fluid_cells],
                                                         m.cell_nodes[lvl.solid_cells],
                                                         lvl.macro_nodes])
        data = fem.union_layout(case.matrices[l], ui, uj)
        S = fem.SplitBlockMatrix.from_union(lvl.n_nodes, ui, uj, data)
        assert abs(S.to_csr() - case.matrices[l].to_csr()).max() == 0.0


@pytest.mark.skipif(not rb.AVAILABLE, reason="reference not mounted")
def test_live_reference_jacobian_2d_mini():
    """Entry-wise comparison with the reference's momentum_jacobian_data."""
    wl = W.CONFIGS["2d_mini"]
    case = get_case("2d_mini")
    rp = rb.ref_problem(wl)
    a = rb.ref()
    for l, (lvl, rl) in enumerate(zip(case.problem.levels, rp.levels)):
        n = lvl.n_nodes
        ref = a.model.momentum_jacobian_data(rl, rp.mats, rp.flags, wl.dt, wl.theta,
                                             case.U[:n], case.U_prev[:n])
        mine = fem.union_layout(case.matrices[l], rl.pattern.indptr, rl.pattern.indices)
        assert np.max(np.abs(mine - ref)) <= 1e-14 * max(1.0, np.abs(ref).max())


@pytest.mark.skipif(not rb.AVAILABLE, reason="reference not mounted")
def test_live_reference_mesh_entities_3d():
    wl = W.CONFIGS["3d_tiny"]
    rp = rb.ref_problem(wl)
    mine = wl.hierarchy()
    for ma, mb in zip(mine.levels, rp.hierarchy.levels):
        assert np.array_equal(ma.edges, mb.edges)
        assert np.array_equal(ma.faces, mb.faces)
        assert np.array_equal(ma.cell_faces, mb.cell_faces)
        for lab in mb.facets:
            assert np.array_equal(ma.facets[lab], mb.facets[lab])
            assert np.array_equal(ma.facet_cells[lab], mb.facet_cells[lab])
            assert np.array_equal(ma.boundary_nodes[lab], mb.boundary_nodes[lab])


@pytest.mark.parametrize("name", ["2d_mini", "3d_tiny"])
def test_interface_columns_match_full_product(name):
    """The extension lifting uses only the interface columns of the raw
    extension operator: same CSR (values, order) as slicing the full scalar
    operator, bitwise-equal products."""
    from paper_1904_02401_b200 import newton
    prob = W.CONFIGS[name].problem()
    lvl = prob.fine
    d = lvl.dim
    raw = prob.extension_blocks(len(prob.levels) - 1)["raw"]
    cols = np.sort((np.asarray(lvl.interface_nodes)[:, None] * d + np.arange(d)).reshape(-1))
    ref = raw.to_csr()[:, cols].tocsr()
    ref.sort_indices()
    c2, sub = newton.interface_columns(raw, lvl.interface_nodes, d)
    assert np.array_equal(cols, c2)
    assert np.array_equal(ref.indptr, sub.indptr) and np.array_equal(ref.indices, sub.indices)
    assert np.array_equal(ref.data, sub.data)
    g = np.random.default_rng(1).standard_normal(len(cols))
    assert np.array_equal(ref @ g, sub @ g)


def test_solid_mass_rows_match_full_product():
    """Residual relation rows from the row-sliced solid mass matrix: bitwise
    equal to the rows of the full product."""
    prob = W.CONFIGS["3d_tiny"].problem()
    lvl = prob.fine
    x = np.random.default_rng(2).standard_normal((lvl.n_nodes, lvl.dim))
    full = lvl.solid_mass_csr() @ x
    assert np.array_equal(full[lvl.relation_nodes], lvl.solid_mass_rows() @ x)
