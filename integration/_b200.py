"""Reference-side binding of the B200 path: the module a maintainer adds to
the reference package as ``alefsi/_b200.py``.

It binds ``libalefsi_b200.so`` with ctypes (C ABI of
``include/alefsi_b200.h``) and replaces the bodies of the reference's
``LinearStack.build_momentum`` / ``solve_momentum`` (reference
newton.py:134-157): the reference keeps assembling the condensed Jacobian
with ``model.momentum_jacobian_data`` and building its patch sets and
prolongations; the operator hierarchy, the Vanka factorisation, the
V-cycle and GMRES run on the GPU.  Depends on numpy and ctypes only (no
torch, no import of this repository's Python package).

    import alefsi.newton, _b200
    _b200.install(alefsi.newton)          # patches LinearStack in place
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB_DEFAULT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "paper_1904_02401_b200", "libalefsi_b200.so")
lib = C.CDLL(os.environ.get("ALEFSI_B200_LIB", _LIB_DEFAULT))
i32, i64, f64, p = C.c_int32, C.c_int64, C.c_double, C.c_void_p
lib.alefsi_mg_create.argtypes = [i32, i32, i32, i32, f64, p]
lib.alefsi_mg_destroy.argtypes = [p]
lib.alefsi_mg_set_matrix.argtypes = [p, i32, i64, i64, p, p, p, i64, p, p, p]
lib.alefsi_mg_set_patches.argtypes = [p, i32, i32, p, p, p]
lib.alefsi_mg_set_prolongation.argtypes = [p, i32, i64, i64, i64, p, p, p]
lib.alefsi_mg_set_constrained.argtypes = [p, i32, p]
lib.alefsi_mg_factorize.argtypes = [p]
lib.alefsi_mg_use_graph.argtypes = [p, i32]
lib.alefsi_gmres.argtypes = [p, p, p, f64, f64, i32, i32, p, p, p]
lib.alefsi_last_error.restype = C.c_char_p

ERR_SINGULAR, ERR_NOT_CONVERGED = 3, 4


def _ok(rc):
    if rc:
        raise RuntimeError(lib.alefsi_last_error().decode())


def _ptr(a):
    return a.ctypes.data


def split(pattern, data):
    """Reference (BlockPattern, data (nnzb, nc, nc)) -> the library's split
    layout: blocks with any entry besides (0,0) (and every diagonal block)
    stay nc x nc blocks, the rest are LPS pressure couplings and move to the
    scalar (p, p) extension.  An exact re-encoding."""
    off = data.copy()
    off[:, 0, 0] = 0.0
    cell = np.any(off.reshape(len(data), -1) != 0.0, axis=1)
    indptr = np.asarray(pattern.indptr, dtype=np.int64)
    indices = np.asarray(pattern.indices)
    rows = np.repeat(np.arange(pattern.n_nodes), np.diff(indptr))
    cell |= rows == indices

    def csr(mask):
        ptr = np.concatenate([[0], np.cumsum(np.bincount(rows[mask], minlength=pattern.n_nodes))])
        return ptr.astype(np.int64), np.ascontiguousarray(indices[mask], dtype=np.int32)
    ip, ix = csr(cell)
    pp, px = csr(~cell)
    return (ip, ix, np.ascontiguousarray(data[cell], dtype=np.float64), pp, px,
            np.ascontiguousarray(data[~cell, 0, 0], dtype=np.float64))


class B200MgSolver:
    """Replaces MgSolver + VankaSmoother.factorize (reference linsolve.py:120-270)."""

    def __init__(self, levels_data, smoothers, transfers, constrained, nu_pre, nu_post, omega):
        nc = levels_data[0][1].shape[1]
        self.h = C.c_void_p()
        _ok(lib.alefsi_mg_create(len(levels_data), nc, nu_pre, nu_post, omega, C.byref(self.h)))
        for l, (pattern, data) in enumerate(levels_data):
            ip, ix, d, pp, px, pd = split(pattern, data)
            _ok(lib.alefsi_mg_set_matrix(self.h, l, pattern.n_nodes, len(ix), _ptr(ip), _ptr(ix),
                                         _ptr(d), len(px), _ptr(pp), _ptr(px), _ptr(pd)))
            mask = np.ascontiguousarray(constrained[l], dtype=np.uint8)
            _ok(lib.alefsi_mg_set_constrained(self.h, l, _ptr(mask)))
            if l == 0:
                continue
            groups = [g for g, _ in smoothers[l].patchset.groups]
            n_p = np.array([len(g) for g in groups], dtype=np.int64)
            npn = np.array([g.shape[1] for g in groups], dtype=np.int32)
            flat = np.ascontiguousarray(np.concatenate([g.ravel() for g in groups]),
                                        dtype=np.int64)
            _ok(lib.alefsi_mg_set_patches(self.h, l, len(groups), _ptr(n_p), _ptr(npn),
                                          _ptr(flat)))
            P = transfers[l].tocsr()
            P.sort_indices()
            ind = P.indptr.astype(np.int64)
            ix2 = P.indices.astype(np.int32)
            val = P.data.astype(np.float64)
            _ok(lib.alefsi_mg_set_prolongation(self.h, l, P.shape[0], P.shape[1], P.nnz,
                                               _ptr(ind), _ptr(ix2), _ptr(val)))
        _ok(lib.alefsi_mg_use_graph(self.h, 1))
        rc = lib.alefsi_mg_factorize(self.h)
        if rc == ERR_SINGULAR:
            raise SingularPatch(lib.alefsi_last_error().decode())
        _ok(rc)

    def gmres(self, b, rel_tol, max_iter, abs_tol=0.0):
        """Replaces linsolve.gmres (reference linsolve.py:41-115); host buffers."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        res = np.zeros(max_iter + 1)
        its = np.zeros(1, np.int32)
        conv = np.zeros(1, np.int32)
        rc = lib.alefsi_gmres(self.h, _ptr(b), _ptr(x), rel_tol, abs_tol, max_iter, 1,
                              _ptr(res), _ptr(its), _ptr(conv))
        if rc not in (0, ERR_NOT_CONVERGED):
            _ok(rc)
        return x, res[: its[0] + 1], int(its[0]), bool(conv[0])

    def close(self):
        if self.h:
            lib.alefsi_mg_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SingularPatch(RuntimeError):
    pass


def install(newton):
    """Patch the reference's ``newton.LinearStack`` (module passed in) so that
    build_momentum / solve_momentum run on the GPU.  Returns the originals."""
    linsolve, model = newton.linsolve, newton.model
    orig = (newton.LinearStack.build_momentum, newton.LinearStack.solve_momentum)

    def build_momentum(self, U, U_prev, k, theta):
        problem = self.problem
        levels_data = []
        for l, lvl in enumerate(problem.levels):
            data = model.momentum_jacobian_data(lvl, problem.mats, problem.flags, k, theta,
                                                problem.restrict_state(U, l),
                                                problem.restrict_state(U_prev, l))
            levels_data.append((lvl.pattern, data))
        old = getattr(self, "mom_b200", None)
        if old is not None:
            old.close()
        try:
            self.mom_b200 = B200MgSolver(
                levels_data, self.mom_smoothers, self.transfers,
                [lvl.momentum_dirichlet.reshape(-1) for lvl in problem.levels],
                self.cfg.nu_pre, self.cfg.nu_post, self.cfg.omega)
        except SingularPatch as exc:
            raise linsolve.SolverError(f"singular Vanka patch block: {exc}") from exc
        self.mom_mg = self.mom_b200      # newton_solve tests `stack.mom_mg is None`

    def solve_momentum(self, b):
        x, res, its, conv = self.mom_b200.gmres(b, self.cfg.momentum_rel_tol, self.cfg.max_iter)
        stats = linsolve.KrylovStats(iterations=its, initial_residual=float(res[0]),
                                     final_residual=float(res[-1]),
                                     residuals=[float(r) for r in res], converged=conv)
        if not conv:
            raise linsolve.SolverError(
                f"GMRES stalled at {stats.final_residual:.3e} after {its} iterations", stats)
        return x, stats

    newton.LinearStack.build_momentum = build_momentum
    newton.LinearStack.solve_momentum = solve_momentum
    return orig
