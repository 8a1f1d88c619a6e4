"""Q2 grid transfer between nested levels.

Host-side construction of the prolongation of reference linsolve.py:183-216:
every fine node takes the coarse Q2 interpolation weights of the first
(lowest-index) fine cell that contains it; restriction is the transpose.
The matrices are built once per hierarchy and applied on the device
(``csrc/device_kernels.cu: transfer_kernel``).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .fem import ShapeTable


def _lattice_points(dim):
    t = np.array([0.0, 0.5, 1.0])
    idx = np.indices((3,) * dim).reshape(dim, -1)
    return np.stack([t[idx[dim - 1 - i]] for i in range(dim)], axis=1)   # x fastest


def prolongation(coarse, fine):
    """Scalar Q2 interpolation matrix (fine nodes x coarse nodes), CSR."""
    dim = coarse.dim
    kids = 2 ** dim
    ref = _lattice_points(dim)
    nb = fine.cell_nodes.shape[1]
    owner = np.full(fine.n_nodes, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(owner, fine.cell_nodes.reshape(-1),
                  np.repeat(np.arange(len(fine.cells), dtype=np.int64), nb))
    rows, cols, vals = [], [], []
    cn = coarse.cell_nodes
    for j in range(kids):
        off = np.array([(j >> i) & 1 for i in range(dim)], dtype=float)
        W = ShapeTable(dim, 0.5 * (ref + off)).N          # W[fine lattice pt, coarse basis]
        fcells = np.arange(len(coarse.cells), dtype=np.int64) * kids + j
        fn = fine.cell_nodes[fcells]
        keep = owner[fn] == fcells[:, None]
        ci_, fi_ = np.nonzero(keep)
        nz = np.abs(W) > 1e-14
        for fi in range(nb):
            sel = fi_ == fi
            if not sel.any():
                continue
            for cb in np.flatnonzero(nz[fi]):
                rows.append(fn[ci_[sel], fi])
                cols.append(cn[ci_[sel], cb])
                vals.append(np.full(int(sel.sum()), W[fi, cb]))
    P = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(fine.n_nodes, coarse.n_nodes))
    P.sum_duplicates()
    P.sort_indices()
    return P
