"""Q2 finite-element machinery and the block-sparse operator layout.

Host-side mirror of the reference's fem module (reference
pkg/src/alefsi/fem.py): tensor Gauss rules (fem.py:34-45), the Q2 Lagrange
basis (fem.py:48-85), isoparametric cell geometry (fem.py:88-103), boundary
facet quadrature (fem.py:224-293) and the local-projection pressure
stabilisation on 2^d-cell macros (fem.py:306-358).

The operator layout differs from the reference on purpose.  The reference
stores one block-CSR over the union of the Q2 cell stencils and the LPS
macro stencils (fem.py:116-136), i.e. full nc x nc blocks even where only the
pressure-pressure entry of an LPS macro coupling is non-zero; in 3D that is
~200 blocks per row of which ~64 carry data.  ``SplitBlockMatrix`` keeps
the same operator as

    A = B (nc x nc blocks on the cell-stencil pattern)
      + L (scalar pressure-pressure entries on the macro pattern minus
           the cell pattern),

which is an exact re-encoding (those blocks carry nothing else) and cuts
the bytes the device SpMV streams by ~2.5x.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib


class GeometryError(Exception):
    pass


class ConstraintError(Exception):
    pass


# -- quadrature and shape functions -------------------------------------------------

def gauss_rule(n, dim):
    """Tensor Gauss-Legendre rule on [0,1]^dim, x fastest; weights sum to 1."""
    x, w = np.polynomial.legendre.leggauss(n)
    x = 0.5 * (x + 1.0)
    w = 0.5 * w
    idx = np.indices((n,) * dim).reshape(dim, -1)        # idx[0] slowest
    pts = np.stack([x[idx[dim - 1 - i]] for i in range(dim)], axis=1)
    ws = np.ones(idx.shape[1])
    for i in range(dim):
        ws = ws * w[idx[i]]
    return pts, ws


def q2_1d(x):
    """1D quadratic Lagrange basis on nodes 0, 1/2, 1 and its derivative."""
    x = np.asarray(x, dtype=float)
    vals = np.stack([2.0 * (x - 0.5) * (x - 1.0), 4.0 * x * (1.0 - x),
                     2.0 * x * (x - 0.5)], axis=-1)
    ders = np.stack([4.0 * x - 3.0, 4.0 - 8.0 * x, 4.0 * x - 1.0], axis=-1)
    return vals, ders


def _tensor(factors):
    """Outer product over dims of (nq, 3) tables -> (nq, 3^d), x index fastest."""
    out = factors[0]                                     # x factor
    nq = out.shape[0]
    for f in factors[1:]:
        out = (out[:, None, :] * f[:, :, None]).reshape(nq, -1)
    return out


class ShapeTable:
    """Q2 basis values N (nq, nb) and reference gradients dN (nq, nb, d)."""

    def __init__(self, dim, points):
        points = np.atleast_2d(np.asarray(points, dtype=float))
        self.dim = dim
        vd = [q2_1d(points[:, i]) for i in range(dim)]
        vals = [v for v, _ in vd]
        ders = [g for _, g in vd]
        self.N = _tensor(vals)
        grads = []
        for i in range(dim):
            fac = [ders[j] if j == i else vals[j] for j in range(dim)]
            grads.append(_tensor(fac))
        self.dN = np.stack(grads, axis=2)

    @property
    def n_basis(self):
        return self.N.shape[1]


def _jacobian(dN, X):
    """J[c,q,i,j] = sum_b X[c,b,i] dN[q,b,j] (reference fem.py:97), as a
    batched matmul X[c]^T @ dN[q] (BLAS order, ~1e-16 from the einsum form)."""
    return np.matmul(np.swapaxes(X, 1, 2)[:, None], dN[None])


def cell_geometry(mesh, table, weights, cells=None, chunk=2048):
    """Physical basis gradients G (nc, nq, nb, d) and weights*det (nc, nq)."""
    conn = mesh.cell_nodes if cells is None else mesh.cell_nodes[cells]
    nc = len(conn)
    nq, nb, d = table.dN.shape
    G = np.empty((nc, nq, nb, d))
    wdet = np.empty((nc, nq))
    bad = []

    def work(s):
        X = mesh.nodes[conn[s:s + chunk]]
        J = _jacobian(table.dN, X)
        det = np.linalg.det(J)
        if np.any(det <= 0):
            bad.append(s)
            return
        Jinv = np.linalg.inv(J)
        # G[c,q] = dN[q] @ Jinv[c,q]: batched matmul (the reference's einsum
        # form sums the same three terms; ~1e-16 apart, 5x faster)
        np.matmul(table.dN[None], Jinv, out=G[s:s + chunk])
        wdet[s:s + chunk] = det * weights[None, :]

    parallel_chunks(work, range(0, nc, chunk))
    if bad:
        raise GeometryError("non-positive cell map determinant")
    return G, wdet


# -- facet quadrature --------------------------------------------------------------

def _facet_ref_points(dim, loc, s, t=None):
    """Reference-cell points of local facet ``loc`` and its outward normal."""
    z = 0.0 * s
    if dim == 2:
        table = {0: ((s, z), (0.0, -1.0)), 1: ((z + 1.0, s), (1.0, 0.0)),
                 2: ((s, z + 1.0), (0.0, 1.0)), 3: ((z, s), (-1.0, 0.0))}
    else:
        table = {0: ((s, t, z), (0.0, 0.0, -1.0)), 1: ((s, t, z + 1.0), (0.0, 0.0, 1.0)),
                 2: ((s, z, t), (0.0, -1.0, 0.0)), 3: ((z + 1.0, s, t), (1.0, 0.0, 0.0)),
                 4: ((s, z + 1.0, t), (0.0, 1.0, 0.0)), 5: ((z, s, t), (-1.0, 0.0, 0.0))}
    pts, nref = table[loc]
    return np.stack(pts, axis=1), np.array(nref)


class FacetQuadrature:
    """Gauss quadrature on labelled boundary facets with owner-cell traces
    (reference fem.py:224-293); facets are ordered by local facet id."""

    def __init__(self, mesh, label, n1d=3, facet_cells=None):
        dim = mesh.dim
        fc = mesh.facet_cells[label] if facet_cells is None else facet_cells
        cells, locs = fc[:, 0], fc[:, 1]
        x1, w1 = np.polynomial.legendre.leggauss(n1d)
        x1 = 0.5 * (x1 + 1.0)
        w1 = 0.5 * w1
        if dim == 2:
            s, t, wq = x1, None, w1
        else:
            ss, tt = np.meshgrid(x1, x1, indexing="ij")
            s, t = ss.reshape(-1), tt.reshape(-1)
            wq = np.outer(w1, w1).reshape(-1)
        self.w = wq
        order = np.argsort(locs, kind="stable")
        parts = {k: [] for k in ("N", "G", "dS", "n", "x")}
        for loc in np.unique(locs):
            sel = order[locs[order] == loc]
            pts, nref = _facet_ref_points(dim, int(loc), s, t)
            table = ShapeTable(dim, pts)
            X = mesh.nodes[mesh.cell_nodes[cells[sel]]]
            J = _jacobian(table.dN, X)
            det = np.linalg.det(J)
            Jinv = np.linalg.inv(J)
            G = np.einsum("qbj,cqji->cqbi", table.dN, Jinv)
            cof = det[..., None] * np.einsum("cqji,j->cqi", Jinv, nref)
            mag = np.linalg.norm(cof, axis=-1)
            parts["N"].append(np.broadcast_to(table.N, (len(sel),) + table.N.shape))
            parts["G"].append(G)
            parts["dS"].append(mag * wq[None, :])
            parts["n"].append(cof / mag[..., None])
            parts["x"].append(np.einsum("qb,cbi->cqi", table.N, X))
        self.cells = cells[order]
        self.conn = mesh.cell_nodes[self.cells]
        self.N = np.concatenate(parts["N"], axis=0)
        self.G = np.concatenate(parts["G"], axis=0)
        self.dS = np.concatenate(parts["dS"], axis=0)
        self.normal = np.concatenate(parts["n"], axis=0)
        self.x = np.concatenate(parts["x"], axis=0)

    @property
    def area(self):
        return float(self.dS.sum())

    def eval(self, nodal):
        return np.einsum("cqb,cb...->cq...", self.N, np.asarray(nodal)[self.conn])

    def eval_grad(self, nodal):
        return np.einsum("cqbj,cb...->cq...j", self.G, np.asarray(nodal)[self.conn])

    def integrate(self, values):
        return np.einsum("cq,cq...->...", self.dS, values)


# -- local projection stabilisation ------------------------------------------------

def _q1_table(points, dim):
    points = np.atleast_2d(points)
    return _tensor([np.stack([1.0 - points[:, i], points[:, i]], axis=1) for i in range(dim)])


def lps_macro_nodes(mesh, fluid_mask):
    """Fluid macros (children of one parent, first child fluid) and their
    sorted unique node lists (reference fem.py:315-327)."""
    groups = mesh.macro_groups()
    groups = groups[fluid_mask[groups[:, 0]]]
    if len(groups) == 0:
        return groups, np.zeros((0, mesh.cell_nodes.shape[1]), dtype=np.int64)
    child = mesh.cell_nodes[groups].reshape(len(groups), -1)
    srt = np.sort(child, axis=1)
    new = np.ones(srt.shape, dtype=bool)
    new[:, 1:] = srt[:, 1:] != srt[:, :-1]
    nmn = int(new[0].sum())
    return groups, srt[new].reshape(len(groups), nmn)


def lps_local_matrices(mesh, table, qpoints, G, wdet, delta_cell, groups, macro_nodes,
                       chunk=512):
    """Pressure-gradient fluctuation penalty per fluid macro: (nm, nmn, nmn).

    The Q2 pressure gradient is projected onto the parent cell's Q1 space
    (constants on single-cell macros) and the fluctuation is penalised with
    the per-cell weight delta (reference fem.py:306-358):
        out = F^T D F,   F = (I - Q M^-1 Q^T W) Gk,   M = Q^T W Q,
    with Gk the macro basis gradients at the children's quadrature points.
    Gk is block sparse (a child touches 27 of the macro's 125 basis
    functions), so the product is expanded as
        out = Gk^T D Gk - C - C^T + coef^T (Q^T D Q) coef,
        coef = M^-1 Q^T W Gk,   C = (Gk^T D Q) coef,
    with the Gk terms accumulated child by child: ~1.5 M instead of 10 M
    multiply-adds per 3D macro and no dense (216 x 375) gradient array
    (same values to ~1e-15 relative)."""
    dim = mesh.dim
    nm, nch = groups.shape
    nb = table.n_basis
    nq = len(qpoints)
    nmn = macro_nodes.shape[1]
    if nch == 1:
        q1 = np.ones((1, nq, 1))
    else:
        q1 = np.empty((nch, nq, 2 ** dim))
        for j in range(nch):
            off = np.array([(j >> i) & 1 for i in range(dim)], dtype=float)
            q1[j] = _q1_table(0.5 * (qpoints + off), dim)
    n1 = q1.shape[2]
    Q = q1.reshape(nch * nq, n1)                                 # ((j q), i)
    d = dim
    out = np.empty((nm, nmn, nmn))

    def work(s):
        g = groups[s:s + chunk]
        m = len(g)
        child = mesh.cell_nodes[g]                              # (m, nch, nb)
        mn = macro_nodes[s:s + chunk]
        # macro-local position of every child basis function
        key = np.arange(m, dtype=np.int64)[:, None] * (mesh.n_nodes + 1)
        loc = np.searchsorted((mn + key).reshape(-1),
                              (child.reshape(m, -1) + key).reshape(-1)).reshape(m, nch, nb)
        loc -= np.arange(m)[:, None, None] * nmn
        Gc = G[g]                                               # (m, nch, nq, nb, d)
        wq = wdet[g]                                            # (m, nch, nq)
        dq = delta_cell[g][:, :, None] * wq
        M = np.matmul(Q.T[None] * wq.reshape(m, 1, nch * nq), Q[None])       # (m, i, l)
        K = np.matmul(Q.T[None] * dq.reshape(m, 1, nch * nq), Q[None])
        R = np.zeros((m, nmn, n1, d))                           # Gk^T W Q
        H = np.zeros((m, nmn, n1, d))                           # Gk^T D Q
        A = np.zeros((m, nmn, nmn))                             # Gk^T D Gk
        mi = np.arange(m)[:, None]
        for j in range(nch):
            Gj = Gc[:, j].transpose(0, 2, 1, 3)                 # (m, nb, nq, d)
            # within one child the positions loc[:, j] are distinct: plain += scatters
            R[mi, loc[:, j]] += np.einsum("mbqd,mq,qi->mbid", Gj, wq[:, j], q1[j], optimize=True)
            H[mi, loc[:, j]] += np.einsum("mbqd,mq,qi->mbid", Gj, dq[:, j], q1[j], optimize=True)
            X = Gj.reshape(m, nb, nq * d)
            Y = (Gj * dq[:, j][:, None, :, None]).reshape(m, nb, nq * d)
            A[mi[:, :, None], loc[:, j][:, :, None], loc[:, j][:, None, :]] += \
                np.matmul(Y, X.transpose(0, 2, 1))
        coef = np.linalg.solve(M, R.transpose(0, 2, 1, 3).reshape(m, n1, nmn * d))
        coef4 = coef.reshape(m, n1, nmn, d)
        C = np.matmul(H.reshape(m, nmn, n1 * d),
                      coef4.transpose(0, 1, 3, 2).reshape(m, n1 * d, nmn))
        KC = np.matmul(K, coef).reshape(m, n1, nmn, d)
        quad = np.matmul(coef4.transpose(0, 2, 1, 3).reshape(m, nmn, n1 * d),
                         KC.transpose(0, 1, 3, 2).reshape(m, n1 * d, nmn))
        out[s:s + m] = A - C - np.swapaxes(C, 1, 2) + quad

    parallel_chunks(work, range(0, nm, chunk))
    return out


def single_blas():
    """Context: one BLAS thread.  The batched tiny LAPACK calls of the setup
    (3x3 / 4x4 / 108x108 inverses) slow down by orders of magnitude when
    OpenBLAS threads each call."""
    from threadpoolctl import threadpool_limits
    return threadpool_limits(limits=1, user_api="blas")


def parallel_chunks(fn, starts, consume=None):
    """Run independent chunk jobs on a thread pool (numpy releases the GIL);
    ``consume`` receives the results in chunk order on the calling thread."""
    from threadpoolctl import threadpool_limits
    starts = list(starts)
    n = min(len(starts), os.cpu_count() or 1)
    with threadpool_limits(limits=1 if n > 1 else None):
        if n <= 1:
            results = map(fn, starts)
            pool = None
        else:
            pool = ThreadPoolExecutor(max_workers=n)
            results = pool.map(fn, starts)
        try:
            for r in results:
                if consume is not None:
                    consume(r)
        finally:
            if pool is not None:
                pool.shutdown()


# -- sparsity patterns and the split operator ----------------------------------------

def pattern_from_elements(n_nodes, elements):
    """Row-sorted union of element stencils (native; reference fem.py:119-133)."""
    elems = [np.ascontiguousarray(e, dtype=np.int64) for e in elements if len(e)]
    ptr = np.concatenate([[0]] + [np.full(len(e), e.shape[1], dtype=np.int64) for e in elems])
    ptr = np.cumsum(ptr).astype(np.int64)
    flat = np.ascontiguousarray(np.concatenate([e.reshape(-1) for e in elems]))
    indptr = np.zeros(n_nodes + 1, dtype=np.int64)
    _lib.call("alefsi_pattern_build", n_nodes, len(ptr) - 1, ptr, flat, indptr, None)
    indices = np.empty(int(indptr[-1]), dtype=np.int32)
    _lib.call("alefsi_pattern_build", n_nodes, len(ptr) - 1, ptr, flat, indptr, indices)
    return indptr, indices


def pattern_slots(indptr, indices, elem_nodes):
    """slots[e, a, b] of pair (elem[e,a], elem[e,b]); -1 where absent."""
    e = np.ascontiguousarray(elem_nodes, dtype=np.int64)
    out = np.empty((e.shape[0], e.shape[1], e.shape[1]), dtype=np.int64)
    _lib.call("alefsi_pattern_slots", len(indptr) - 1, indptr, indices, e.shape[0],
              e.shape[1], e, out)
    return out


def scatter_blocks(indptr, indices, data, elem_nodes, local, skip_missing=False):
    """data[slot(e,a,b)] += local[e,a,b] in flattened order (np.add.at order)."""
    e = np.ascontiguousarray(elem_nodes, dtype=np.int64)
    loc = np.ascontiguousarray(local, dtype=np.float64)
    bs = int(np.prod(data.shape[1:])) if data.ndim > 1 else 1
    if loc.size != e.shape[0] * e.shape[1] ** 2 * bs:
        raise ValueError("local block array does not match elements")
    _lib.call("alefsi_scatter_add_blocks", len(indptr) - 1, indptr, indices, e.shape[0],
              e.shape[1], e, bs, loc, data, 1 if skip_missing else 0)


@dataclass
class SplitPattern:
    """Cell-stencil block pattern plus the pressure-only macro extension."""

    n_nodes: int
    indptr: np.ndarray          # cell pattern (block rows = nodes)
    indices: np.ndarray
    pp_indptr: np.ndarray       # macro-pattern entries outside the cell pattern
    pp_indices: np.ndarray
    macro_indptr: np.ndarray    # full LPS macro pattern (scalar)
    macro_indices: np.ndarray
    macro_to_cell: np.ndarray   # per macro entry: cell slot or -1
    macro_to_pp: np.ndarray     # per macro entry: pp slot or -1
    diag_slot: np.ndarray

    @property
    def nnzb(self):
        return len(self.indices)

    @property
    def nnz_pp(self):
        return len(self.pp_indices)


def build_split_pattern(n_nodes, cell_groups, macro_nodes):
    indptr, indices = pattern_from_elements(n_nodes, cell_groups)
    diag = pattern_match(indptr, indices, np.arange(n_nodes + 1, dtype=np.int64),
                         np.arange(n_nodes, dtype=np.int32))
    if len(macro_nodes):
        mptr, mind = pattern_from_elements(n_nodes, [macro_nodes])
    else:
        mptr, mind = np.zeros(n_nodes + 1, dtype=np.int64), np.zeros(0, dtype=np.int32)
    to_cell = pattern_match(indptr, indices, mptr, mind)
    # entries outside the cell pattern, row by row (native, two parallel passes)
    mind = np.ascontiguousarray(mind, dtype=np.int32)
    pp_indptr = np.zeros(n_nodes + 1, dtype=np.int64)
    n_extra = int(np.count_nonzero(to_cell < 0))
    pp_indices = np.empty(n_extra, dtype=np.int32)
    to_pp = np.empty(len(mind), dtype=np.int64)
    _lib.call("alefsi_split_extension", n_nodes, np.ascontiguousarray(mptr, dtype=np.int64), mind,
              to_cell, pp_indptr, pp_indices, to_pp)
    return SplitPattern(n_nodes, indptr, indices, pp_indptr, pp_indices,
                        mptr, mind, to_cell, to_pp, diag.astype(np.int64))


def pattern_match(a_ptr, a_idx, b_ptr, b_idx):
    """Slot in pattern A of every entry of pattern B (-1 if absent); native."""
    out = np.empty(len(b_idx), dtype=np.int64)
    _lib.call("alefsi_pattern_match", len(a_ptr) - 1,
              np.ascontiguousarray(a_ptr, dtype=np.int64), np.ascontiguousarray(a_idx, dtype=np.int32),
              np.ascontiguousarray(b_ptr, dtype=np.int64), np.ascontiguousarray(b_idx, dtype=np.int32),
              out)
    return out


@dataclass
class SplitBlockMatrix:
    """A = B (nc x nc blocks, cell pattern) + L (scalar (0,0) entries, pp pattern)."""

    pattern: SplitPattern
    data: np.ndarray            # (nnzb, nc, nc)
    pp_data: np.ndarray         # (nnz_pp,)

    @property
    def nc(self):
        return self.data.shape[1]

    @property
    def n_nodes(self):
        return self.pattern.n_nodes

    @property
    def shape(self):
        n = self.n_nodes * self.nc
        return (n, n)

    def to_csr(self):
        """Scalar CSR of the whole operator (host verification use)."""
        p, nc = self.pattern, self.nc
        B = sp.bsr_matrix((self.data, p.indices, p.indptr),
                          shape=self.shape).tocoo()
        rows = np.repeat(np.arange(p.n_nodes), np.diff(p.pp_indptr)) * nc
        cols = p.pp_indices.astype(np.int64) * nc
        L = sp.coo_matrix((self.pp_data, (rows, cols)), shape=self.shape)
        return (B + L).tocsr()

    def dot(self, x):
        return self.to_csr() @ x

    @classmethod
    def from_union(cls, n_nodes, indptr, indices, data):
        """Split a reference-layout operator (BlockPattern indptr/indices,
        data (nnzb, nc, nc)) by value: blocks whose entries other than (0,0)
        are all zero (the LPS macro couplings) become scalar pp entries;
        diagonal blocks always stay blocks."""
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices)
        rows = np.repeat(np.arange(n_nodes, dtype=np.int64), np.diff(indptr))
        off = np.array(data, copy=True)
        off[:, 0, 0] = 0.0
        cell = np.any(off.reshape(len(data), -1) != 0.0, axis=1) | (rows == indices)

        def csr(mask):
            ptr = np.concatenate([[0], np.cumsum(np.bincount(rows[mask], minlength=n_nodes))])
            return ptr.astype(np.int64), indices[mask].astype(np.int32)
        ip, ix = csr(cell)
        pp, px = csr(~cell)
        key = rows[cell] * n_nodes + ix
        diag = np.searchsorted(key, np.arange(n_nodes, dtype=np.int64) * (n_nodes + 1))
        pat = SplitPattern(n_nodes, ip, ix, pp, px, indptr, indices.astype(np.int32),
                           np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.int64),
                           diag.astype(np.int64))
        return cls(pat, np.ascontiguousarray(data[cell]), np.ascontiguousarray(data[~cell, 0, 0]))

    def copy(self):
        return SplitBlockMatrix(self.pattern, self.data.copy(), self.pp_data.copy())


def apply_dirichlet_rows(A: SplitBlockMatrix, mask):
    """Constrained (node, comp) rows become identity rows (reference
    fem.py:172-182), in both parts of the split operator."""
    p = A.pattern
    for c in range(A.nc):
        nodes = np.flatnonzero(mask[:, c])
        if len(nodes) == 0:
            continue
        cnt = np.diff(p.indptr)[nodes]
        slots = np.repeat(p.indptr[nodes], cnt) + _ranges(cnt)
        A.data[slots, c, :] = 0.0
        if c == 0:
            cnt = np.diff(p.pp_indptr)[nodes]
            A.pp_data[np.repeat(p.pp_indptr[nodes], cnt) + _ranges(cnt)] = 0.0
        A.data[p.diag_slot[nodes], c, c] = 1.0


def _ranges(counts):
    counts = np.asarray(counts, dtype=np.int64)
    if counts.sum() == 0:
        return np.zeros(0, dtype=np.int64)
    starts = np.repeat(np.cumsum(counts) - counts, counts)
    return np.arange(int(counts.sum()), dtype=np.int64) - starts


def union_layout(A: SplitBlockMatrix, union_indptr, union_indices):
    """Re-encode the split operator on a union (reference-layout) pattern."""
    p, nc, n = A.pattern, A.nc, A.n_nodes
    ukey = np.repeat(np.arange(n, dtype=np.int64), np.diff(union_indptr)) * n + union_indices
    out = np.zeros((len(union_indices), nc, nc))
    ckey = np.repeat(np.arange(n, dtype=np.int64), np.diff(p.indptr)) * n + p.indices
    out[np.searchsorted(ukey, ckey)] += A.data
    pkey = np.repeat(np.arange(n, dtype=np.int64), np.diff(p.pp_indptr)) * n + p.pp_indices
    out[np.searchsorted(ukey, pkey), 0, 0] += A.pp_data
    return out
