"""Nested quad/hex meshes, dof classification, Vanka patches and coloring.

Host-side mirror of the reference's mesh module (reference
pkg/src/alefsi/mesh.py).  Everything here is integer index work that has to
be bit-exact with the reference: node numbering (vertices, then edge
midpoints, face centres and cell centres, each in the lexicographic order of
their sorted vertex tuples; mesh.py:103-156), uniform refinement
(mesh.py:246-294), dof classification (mesh.py:418-437), patch construction
(mesh.py:483-510) and the greedy coloring (mesh.py:522-556, run natively in
``csrc/host_index.cpp``).

Besides the reference API this module builds the structured channel/box
meshes used by the benchmark workloads (``box_mesh``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FLUID = 0
SOLID = 1

INFLOW = "inflow"
OUTFLOW = "outflow"
WALL = "wall"
CYLINDER = "cylinder"
SOLID_DIRICHLET = "solid_dirichlet"

NODE_FLUID = 0
NODE_INTERFACE = 1
NODE_SOLID = 2

ONE_ELEMENT = "one"
MULTI_ELEMENT = "multi"     # 4 elements in 2d, 8 in 3d

# reference-cell vertex coordinates (v0=(0,0) v1=(1,0) v2=(1,1) v3=(0,1); z=1 copies)
_REF_VERTS = {
    2: np.array([[0, 0], [1, 0], [1, 1], [0, 1]]),
    3: np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                 [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]]),
}
# local edges and faces (vertex tuples) — reference mesh.py:38-43
LOCAL_EDGES = {
    2: [(0, 1), (1, 2), (2, 3), (3, 0)],
    3: [(0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
        (0, 4), (1, 5), (2, 6), (3, 7)],
}
LOCAL_FACES_3D = [(0, 1, 2, 3), (4, 5, 6, 7), (0, 1, 5, 4),
                  (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7)]
_QUAD_EDGES = [(0, 1), (1, 2), (2, 3), (3, 0)]


class MeshError(Exception):
    pass


class MeshIntegrityError(MeshError):
    pass


def _lattice_map(dim):
    """For each of the 3^d lattice positions (x fastest): (kind, local id).

    kind 0 = vertex, 1 = edge, 2 = face, 3 = cell centre.  Derived from the
    reference-cell geometry: a lattice point at 2*p is the centroid of the
    entity whose vertices average to p.
    """
    ref = _REF_VERTS[dim]
    out = []
    for flat in range(3 ** dim):
        pos = np.array([(flat // 3 ** i) % 3 for i in range(dim)]) / 2.0
        n_mid = int(np.sum(pos == 0.5))
        if n_mid == 0:
            hit = [v for v in range(len(ref)) if np.all(ref[v] == pos)]
            out.append((0, hit[0]))
        elif n_mid == dim:
            out.append((3, 0))
        elif n_mid == 1:
            hit = [e for e, (a, b) in enumerate(LOCAL_EDGES[dim])
                   if np.all((ref[a] + ref[b]) / 2.0 == pos)]
            out.append((1, hit[0]))
        else:
            hit = [f for f, vs in enumerate(LOCAL_FACES_3D)
                   if np.all(ref[list(vs)].mean(axis=0) == pos)]
            out.append((2, hit[0]))
    return out


_LATTICE = {d: _lattice_map(d) for d in (2, 3)}


def _unique_sorted_tuples(conn):
    """Unique rows of row-sorted int tuples in lexicographic order + inverse."""
    rows = np.sort(np.asarray(conn, dtype=np.int64), axis=1)
    order = np.lexsort(rows.T[::-1])
    srt = rows[order]
    new = np.ones(len(srt), dtype=bool)
    new[1:] = np.any(srt[1:] != srt[:-1], axis=1)
    uniq = srt[new]
    ids_sorted = np.cumsum(new) - 1
    inverse = np.empty(len(rows), dtype=np.int64)
    inverse[order] = ids_sorted
    return uniq, inverse


def _lookup_tuples(table, queries):
    """Row index of each (row-sorted) query tuple in a lexicographic table."""
    q = np.sort(np.asarray(queries, dtype=np.int64).reshape(-1, table.shape[1]), axis=1)
    if len(q) == 0:
        return np.zeros(0, dtype=np.int64)
    allrows = np.concatenate([table, q])
    order = np.lexsort(allrows.T[::-1])
    srt = allrows[order]
    is_table = order < len(table)
    new = np.ones(len(srt), dtype=bool)
    new[1:] = np.any(srt[1:] != srt[:-1], axis=1)
    group = np.cumsum(new) - 1
    # table id per group (tables have unique rows)
    gid = np.full(group[-1] + 1, -1, dtype=np.int64)
    gid[group[is_table]] = order[is_table]
    res = np.empty(len(q), dtype=np.int64)
    res[order[~is_table] - len(table)] = gid[group[~is_table]]
    if np.any(res < 0):
        raise MeshError("facet entity not found in mesh")
    return res


@dataclass(frozen=True)
class CircleProjector:
    """Radial projection onto a circle (2d) or a z-aligned cylinder (3d)."""

    cx: float
    cy: float
    radius: float

    def __call__(self, points):
        points = np.array(points, dtype=float, copy=True)
        c = np.array([self.cx, self.cy])
        d = points[:, :2] - c
        points[:, :2] = c + self.radius * d / np.linalg.norm(d, axis=1)[:, None]
        return points


class MeshLevel:
    """One level: bilinear cell connectivity plus the derived Q2 node set."""

    def __init__(self, dim, vertices, cells, cell_subdomain, facets,
                 projectors=None, parent_cell=None, level=0):
        self.dim = int(dim)
        self.vertices = np.asarray(vertices, dtype=float)
        self.cells = np.asarray(cells, dtype=np.int64)
        self.cell_subdomain = np.asarray(cell_subdomain, dtype=np.int8)
        nfv = 2 ** (self.dim - 1)
        self.facets = {lab: np.asarray(f, dtype=np.int64).reshape(-1, nfv)
                       for lab, f in facets.items() if len(f)}
        self.projectors = dict(projectors or {})
        self.parent_cell = (np.asarray(parent_cell, dtype=np.int64) if parent_cell is not None
                            else np.full(len(self.cells), -1, dtype=np.int64))
        self.level = level
        self._entities()
        self._nodes()
        self._facet_info()

    # -- entities ------------------------------------------------------------
    def _entities(self):
        c = self.cells
        le = LOCAL_EDGES[self.dim]
        conn = np.concatenate([c[:, list(e)] for e in le], axis=0)
        self.edges, inv = _unique_sorted_tuples(conn)
        self.cell_edges = inv.reshape(len(le), -1).T.copy()
        if self.dim == 3:
            conn = np.concatenate([c[:, list(f)] for f in LOCAL_FACES_3D], axis=0)
            self.faces, inv = _unique_sorted_tuples(conn)
            self.cell_faces = inv.reshape(len(LOCAL_FACES_3D), -1).T.copy()
        else:
            self.faces = np.zeros((0, 4), dtype=np.int64)
            self.cell_faces = np.zeros((len(c), 0), dtype=np.int64)

    def _lattice(self):
        nv, ne, nf = len(self.vertices), len(self.edges), len(self.faces)
        cols = []
        for kind, lid in _LATTICE[self.dim]:
            if kind == 0:
                cols.append(self.cells[:, lid])
            elif kind == 1:
                cols.append(self.cell_edges[:, lid] + nv)
            elif kind == 2:
                cols.append(self.cell_faces[:, lid] + nv + ne)
            else:
                cols.append(np.arange(len(self.cells), dtype=np.int64) + nv + ne + nf)
        return np.stack(cols, axis=1)

    @staticmethod
    def _centroid(pts):
        # sequential sum in vertex order, then divide (matches np.mean on
        # a short middle axis)
        acc = pts[:, 0].copy()
        for i in range(1, pts.shape[1]):
            acc = acc + pts[:, i]
        return acc / pts.shape[1]

    def _nodes(self):
        parts = [self.vertices, self._centroid(self.vertices[self.edges])]
        if self.dim == 3:
            parts.append(self._centroid(self.vertices[self.faces]))
        parts.append(self._centroid(self.vertices[self.cells]))
        nodes = np.concatenate(parts, axis=0)
        for label, proj in self.projectors.items():
            if label in self.facets:
                ids = self._curved_node_ids(self.facets[label])
                if len(ids):
                    nodes[ids] = proj(nodes[ids])
        self.nodes = nodes
        self.n_nodes = len(nodes)
        self.cell_nodes = self._lattice()

    def edge_ids(self, pairs):
        return _lookup_tuples(self.edges, pairs)

    def face_ids(self, quads):
        return _lookup_tuples(self.faces, quads)

    def _facet_entity_nodes(self, f):
        nv, ne = len(self.vertices), len(self.edges)
        if self.dim == 2:
            return [nv + self.edge_ids(f)]
        ids = [nv + self.edge_ids(f[:, [a, b]]) for a, b in _QUAD_EDGES]
        ids.append(nv + ne + self.face_ids(f))
        return ids

    def _curved_node_ids(self, f):
        return np.unique(np.concatenate(self._facet_entity_nodes(f)))

    def _facet_info(self):
        self.facet_cells = {}
        self.boundary_nodes = {}
        ent = self.cell_edges if self.dim == 2 else self.cell_faces
        n_ent = len(self.edges) if self.dim == 2 else len(self.faces)
        # first (local facet, cell) occurrence in local-facet-major order
        owner = np.full((n_ent, 2), -1, dtype=np.int64)
        for loc in range(ent.shape[1])[::-1]:
            cells = np.arange(len(self.cells))[::-1]
            owner[ent[cells, loc], 0] = cells
            owner[ent[cells, loc], 1] = loc
        for label, f in self.facets.items():
            ids = self.edge_ids(f) if self.dim == 2 else self.face_ids(f)
            self.facet_cells[label] = owner[ids].copy()
            self.boundary_nodes[label] = np.unique(np.concatenate(
                [f.reshape(-1)] + self._facet_entity_nodes(f)))

    # -- helpers ---------------------------------------------------------------
    def nodes_of_label(self, *labels):
        parts = [self.boundary_nodes[l] for l in labels if l in self.boundary_nodes]
        if not parts:
            return np.zeros(0, dtype=np.int64)
        return np.unique(np.concatenate(parts))

    def macro_groups(self):
        """Cells grouped by parent; the coarsest level uses single cells."""
        if self.parent_cell[0] < 0:
            return np.arange(len(self.cells), dtype=np.int64)[:, None]
        order = np.argsort(self.parent_cell, kind="stable")
        return order.reshape(-1, 2 ** self.dim)


def refine(mesh: MeshLevel) -> MeshLevel:
    """Uniform refinement: Q2 nodes become the fine vertices; the 2^d children
    of a cell are contiguous, x-index fastest (reference mesh.py:246-294)."""
    d = mesh.dim
    lat = mesh._lattice().reshape((-1,) + (3,) * d)      # [..., z, y, x]
    kids = []
    if d == 2:
        for b in (0, 1):
            for a in (0, 1):
                kids.append(np.stack([lat[:, b, a], lat[:, b, a + 1],
                                      lat[:, b + 1, a + 1], lat[:, b + 1, a]], axis=1))
    else:
        for c in (0, 1):
            for b in (0, 1):
                for a in (0, 1):
                    kids.append(np.stack([
                        lat[:, c, b, a], lat[:, c, b, a + 1],
                        lat[:, c, b + 1, a + 1], lat[:, c, b + 1, a],
                        lat[:, c + 1, b, a], lat[:, c + 1, b, a + 1],
                        lat[:, c + 1, b + 1, a + 1], lat[:, c + 1, b + 1, a]], axis=1))
    nk = 2 ** d
    cells = np.stack(kids, axis=1).reshape(len(mesh.cells) * nk, -1)
    parent = np.repeat(np.arange(len(mesh.cells), dtype=np.int64), nk)
    sub = np.repeat(mesh.cell_subdomain, nk)
    nv, ne = len(mesh.vertices), len(mesh.edges)
    facets = {}
    for label, f in mesh.facets.items():
        if d == 2:
            m = nv + mesh.edge_ids(f)
            facets[label] = np.concatenate([np.stack([f[:, 0], m], axis=1),
                                            np.stack([m, f[:, 1]], axis=1)])
        else:
            e = [nv + mesh.edge_ids(f[:, [a, b]]) for a, b in _QUAD_EDGES]
            fc = nv + ne + mesh.face_ids(f)
            facets[label] = np.concatenate([
                np.stack([f[:, 0], e[0], fc, e[3]], axis=1),
                np.stack([e[0], f[:, 1], e[1], fc], axis=1),
                np.stack([fc, e[1], f[:, 2], e[2]], axis=1),
                np.stack([e[3], fc, e[2], f[:, 3]], axis=1)])
    return MeshLevel(d, mesh.nodes, cells, sub, facets, projectors=mesh.projectors,
                     parent_cell=parent, level=mesh.level + 1)


@dataclass
class MeshHierarchy:
    levels: list

    @property
    def dim(self):
        return self.levels[0].dim

    @property
    def finest(self):
        return self.levels[-1]

    def __len__(self):
        return len(self.levels)


def build_hierarchy(coarse: MeshLevel, level: int) -> MeshHierarchy:
    levels = [coarse]
    for _ in range(level):
        levels.append(refine(levels[-1]))
    return MeshHierarchy(levels)


def box_mesh(lengths, cells_per_dim) -> MeshLevel:
    """Structured channel [0,Lx]x[0,Ly](x[0,Lz]) with inflow at x=0, outflow at
    x=Lx and walls elsewhere; vertices lexicographic with x fastest.  All
    cells are fluid (solid tags are set per level by ``tag_solid_box``)."""
    L = [float(v) for v in lengths]
    n = [int(v) for v in cells_per_dim]
    dim = len(n)
    axes = [np.linspace(0.0, L[i], n[i] + 1) for i in range(dim)]
    grids = np.meshgrid(*axes[::-1], indexing="ij")
    verts = np.stack([g.reshape(-1) for g in grids[::-1]], axis=1)
    shape = [n[i] + 1 for i in range(dim)]

    def vid(*ijk):
        out = 0
        for i in reversed(range(dim)):
            out = out * shape[i] + ijk[i]
        return out

    facets = {INFLOW: [], OUTFLOW: [], WALL: []}
    if dim == 2:
        j, i = np.meshgrid(np.arange(n[1]), np.arange(n[0]), indexing="ij")
        i, j = i.reshape(-1), j.reshape(-1)
        cells = np.stack([vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)], axis=1)
        jj = np.arange(n[1])
        facets[INFLOW] = np.stack([vid(0, jj + 1), vid(0, jj)], axis=1)
        facets[OUTFLOW] = np.stack([vid(n[0], jj), vid(n[0], jj + 1)], axis=1)
        ii = np.arange(n[0])
        bot = np.stack([vid(ii, 0), vid(ii + 1, 0)], axis=1)
        top = np.stack([vid(ii + 1, n[1]), vid(ii, n[1])], axis=1)
        facets[WALL] = np.stack([bot, top], axis=1).reshape(-1, 2)
    else:
        k, j, i = np.meshgrid(np.arange(n[2]), np.arange(n[1]), np.arange(n[0]), indexing="ij")
        i, j, k = i.reshape(-1), j.reshape(-1), k.reshape(-1)
        cells = np.stack([vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k), vid(i, j + 1, k),
                          vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i + 1, j + 1, k + 1),
                          vid(i, j + 1, k + 1)], axis=1)
        kk, jj = [a.reshape(-1) for a in np.meshgrid(np.arange(n[2]), np.arange(n[1]), indexing="ij")]

        def xface(x):
            return np.stack([vid(x, jj, kk), vid(x, jj + 1, kk), vid(x, jj + 1, kk + 1),
                             vid(x, jj, kk + 1)], axis=1)
        facets[INFLOW] = xface(0)
        facets[OUTFLOW] = xface(n[0])
        kk, ii = [a.reshape(-1) for a in np.meshgrid(np.arange(n[2]), np.arange(n[0]), indexing="ij")]

        def yface(y):
            return np.stack([vid(ii, y, kk), vid(ii + 1, y, kk), vid(ii + 1, y, kk + 1),
                             vid(ii, y, kk + 1)], axis=1)
        ywalls = np.stack([yface(0), yface(n[1])], axis=1).reshape(-1, 4)
        jj, ii = [a.reshape(-1) for a in np.meshgrid(np.arange(n[1]), np.arange(n[0]), indexing="ij")]

        def zface(z):
            return np.stack([vid(ii, jj, z), vid(ii + 1, jj, z), vid(ii + 1, jj + 1, z),
                             vid(ii, jj + 1, z)], axis=1)
        zwalls = np.stack([zface(0), zface(n[2])], axis=1).reshape(-1, 4)
        facets[WALL] = np.concatenate([ywalls, zwalls])
    sub = np.zeros(len(cells), dtype=np.int8)
    return MeshLevel(dim, verts, cells, sub, facets)


def tag_solid_box(mesh: MeshLevel, lo, hi):
    """Tag cells whose centre lies strictly inside the box (lo, hi) as solid."""
    cen = MeshLevel._centroid(mesh.vertices[mesh.cells])
    inside = np.all((cen > np.asarray(lo)) & (cen < np.asarray(hi)), axis=1)
    mesh.cell_subdomain = np.where(inside, SOLID, FLUID).astype(np.int8)
    return mesh


# -- dof classification ----------------------------------------------------------

@dataclass
class DofClassification:
    node_class: np.ndarray
    pressure_active: np.ndarray

    def count(self, kind):
        return int(np.sum(self.node_class == kind))


def classify_dofs(mesh: MeshLevel) -> DofClassification:
    """Fluid / interface / solid node labels from cell adjacency
    (reference mesh.py:418-437)."""
    fl = np.zeros(mesh.n_nodes, dtype=bool)
    so = np.zeros(mesh.n_nodes, dtype=bool)
    fl[mesh.cell_nodes[mesh.cell_subdomain == FLUID].reshape(-1)] = True
    so[mesh.cell_nodes[mesh.cell_subdomain == SOLID].reshape(-1)] = True
    if not np.all(fl | so):
        raise MeshIntegrityError("orphan nodes without cell adjacency")
    cls = np.full(mesh.n_nodes, NODE_FLUID, dtype=np.int8)
    cls[so] = NODE_SOLID
    cls[fl & so] = NODE_INTERFACE
    centre = mesh.cell_nodes[:, mesh.cell_nodes.shape[1] // 2]
    if np.any(cls[centre] == NODE_INTERFACE):
        raise MeshIntegrityError("interface cuts through a cell interior")
    return DofClassification(cls, cls != NODE_SOLID)


# -- Vanka patches and coloring ----------------------------------------------------

@dataclass
class PatchSet:
    """Dof-index patches; ``groups`` holds (node_array, subdomain) pairs with a
    homogeneous patch size per group (reference mesh.py:446-480)."""

    n_comp: int
    groups: list = field(default_factory=list)

    def add(self, nodes, subdomain):
        if len(nodes):
            self.groups.append((np.asarray(nodes, dtype=np.int64), int(subdomain)))

    @property
    def n_patches(self):
        return sum(len(g) for g, _ in self.groups)

    def patch_nodes(self):
        for g, _ in self.groups:
            yield from g

    def dof_groups(self):
        out = []
        for g, sub in self.groups:
            out.append(((g[:, :, None] * self.n_comp + np.arange(self.n_comp)).reshape(len(g), -1),
                        sub))
        return out

    def sizes(self):
        return [g.shape[1] * self.n_comp for g, _ in self.groups]


def build_patches(mesh: MeshLevel, strategy, n_comp, per_subdomain=None) -> PatchSet:
    """One-element or 2^d-element (children of one parent) patches per
    subdomain (reference mesh.py:483-510)."""
    per_subdomain = per_subdomain or {FLUID: strategy, SOLID: strategy}
    ps = PatchSet(n_comp=n_comp)
    for sub in (FLUID, SOLID):
        strat = per_subdomain.get(sub, strategy)
        cells = np.flatnonzero(mesh.cell_subdomain == sub)
        if len(cells) == 0:
            continue
        if strat == ONE_ELEMENT or mesh.parent_cell[0] < 0:
            ps.add(mesh.cell_nodes[cells], sub)
        elif strat == MULTI_ELEMENT:
            groups = mesh.macro_groups()
            keep = np.isin(groups[:, 0], cells)
            nodes = np.sort(mesh.cell_nodes[groups[keep]].reshape(int(keep.sum()), -1), axis=1)
            if len(nodes):
                new = np.ones(nodes.shape, dtype=bool)
                new[:, 1:] = nodes[:, 1:] != nodes[:, :-1]
                per_row = new.sum(axis=1)
                if np.any(per_row != per_row[0]):
                    raise MeshError("macro patches of differing size")
                nodes = nodes[new].reshape(len(nodes), per_row[0])
            ps.add(nodes, sub)
        else:
            raise ValueError(f"unknown patch strategy {strat!r}")
    return ps


@dataclass
class Coloring:
    color: np.ndarray
    n_colors: int

    def patches_of_color(self, c):
        return np.flatnonzero(self.color == c)


def color_patches(patchset: PatchSet) -> Coloring:
    """Greedy first-fit coloring (reference mesh.py:522-556), run natively."""
    from . import _lib
    rows = [g for g, _ in patchset.groups]
    n = sum(len(g) for g in rows)
    if n == 0:
        return Coloring(color=np.zeros(0, dtype=np.int64), n_colors=0)
    sizes = np.concatenate([np.full(len(g), g.shape[1] * patchset.n_comp, dtype=np.int64)
                            for g in rows])
    ptr = np.concatenate([[0], np.cumsum(np.concatenate(
        [np.full(len(g), g.shape[1], dtype=np.int64) for g in rows]))]).astype(np.int64)
    flat = np.ascontiguousarray(np.concatenate([g.reshape(-1) for g in rows]), dtype=np.int64)
    n_nodes = int(flat.max()) + 1
    color = np.empty(n, dtype=np.int64)
    nc = np.zeros(1, dtype=np.int64)
    _lib.call("alefsi_color_patches", n, ptr, flat, sizes, n_nodes, color, nc)
    return Coloring(color=color, n_colors=int(nc[0]))
