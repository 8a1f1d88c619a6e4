"""Python handle over the device-resident multigrid hierarchy (C ABI).

``DeviceMgSolver`` owns one ``alefsi_mg`` handle: per-level split block
operators, Vanka patch tables and their inverses, Q2 transfer operators and
the GMRES Krylov basis, all resident in HBM.  Vectors may be numpy arrays
(host; copied in and out by the library, the end-to-end path) or CUDA
tensors (device-resident, no copies).
"""

from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass, field

import numpy as np

from . import _lib


class SolverError(Exception):
    """Raised when GMRES misses its tolerance or a patch is singular
    (reference linsolve.py:25-28)."""

    def __init__(self, message, stats=None):
        super().__init__(message)
        self.stats = stats


@dataclass
class KrylovStats:
    iterations: int = 0
    initial_residual: float = 0.0
    final_residual: float = 0.0
    elapsed: float = 0.0
    converged: bool = True
    residuals: list = field(default_factory=list)


def _is_device(a):
    return hasattr(a, "is_cuda") and a.is_cuda


class DeviceMgSolver:
    """V-cycle preconditioner + GMRES over a device level hierarchy.

    ``levels`` are dicts with keys ``matrix`` (fem.SplitBlockMatrix),
    ``patches`` (mesh.PatchSet; None on level 0), ``P`` (scipy CSR
    prolongation from the coarser level; None on level 0) and
    ``constrained`` (bool per dof)."""

    def __init__(self, levels, nu_pre=2, nu_post=2, omega=0.8, use_graph=False, stream=None,
                 factorize=True, nc=None):
        lib = _lib.load()
        self.n_levels = len(levels)
        self.nc = nc if nc is not None else levels[0]["matrix"].nc
        self.nu_pre, self.nu_post, self.omega = nu_pre, nu_post, omega
        h = C.c_void_p()
        _lib.call("alefsi_mg_create", self.n_levels, self.nc, nu_pre, nu_post, float(omega),
                  C.byref(h))
        self._h = h
        self._lib = lib
        self._stream_bound = stream is not None
        if stream is None and "torch" in sys.modules:
            # enqueue on torch's current stream so device tensors passed in are
            # ordered after the work that produced them.  Without torch loaded
            # (host-array callers such as the time loop) the library keeps its
            # own stream and torch is bound on first use of a device tensor.
            self._bind_torch_stream()
        elif stream is not None:
            _lib.call("alefsi_mg_set_stream", h, C.c_void_p(int(stream)))
        self.ndofs = []
        self._groups = {}
        self._device_outflow = set()     # levels whose outflow blocks are assembled on device
        self._device_tail = set()        # levels whose residual tail runs on device
        for l, lv in enumerate(levels):
            self._set_level(l, lv)
        _lib.call("alefsi_mg_use_graph", h, 1 if use_graph else 0)
        if factorize:
            self.factorize()

    def _bind_torch_stream(self):
        if self._stream_bound:
            return
        import torch
        if torch.cuda.is_available():
            _lib.call("alefsi_mg_set_stream", self._h,
                      C.c_void_p(int(torch.cuda.current_stream().cuda_stream)))
        self._stream_bound = True

    # -- setup ------------------------------------------------------------------
    def _set_level(self, l, lv):
        A = lv.get("matrix")
        if A is None:          # structure only: the operator is assembled on the device
            p = lv["pattern"]
            _lib.call("alefsi_mg_set_pattern", self._h, l, p.n_nodes, p.nnzb,
                      np.ascontiguousarray(p.indptr, dtype=np.int64),
                      np.ascontiguousarray(p.indices, dtype=np.int32), p.nnz_pp,
                      np.ascontiguousarray(p.pp_indptr, dtype=np.int64),
                      np.ascontiguousarray(p.pp_indices, dtype=np.int32))
            self.ndofs.append(p.n_nodes * self.nc)
        else:
            p = A.pattern
            _lib.call("alefsi_mg_set_matrix", self._h, l, p.n_nodes, p.nnzb,
                      np.ascontiguousarray(p.indptr, dtype=np.int64),
                      np.ascontiguousarray(p.indices, dtype=np.int32),
                      np.ascontiguousarray(A.data, dtype=np.float64), p.nnz_pp,
                      np.ascontiguousarray(p.pp_indptr, dtype=np.int64),
                      np.ascontiguousarray(p.pp_indices, dtype=np.int32),
                      np.ascontiguousarray(A.pp_data, dtype=np.float64))
            self.ndofs.append(p.n_nodes * A.nc)
        mask = np.ascontiguousarray(np.asarray(lv["constrained"]).reshape(-1), dtype=np.uint8)
        _lib.call("alefsi_mg_set_constrained", self._h, l, mask)
        if l == 0:
            return
        groups = [g for g, _ in lv["patches"].groups]
        n_p = np.array([len(g) for g in groups], dtype=np.int64)
        self._groups[l] = [(len(g), g.shape[1] * self.nc) for g in groups]
        npn = np.array([g.shape[1] for g in groups], dtype=np.int32)
        flat = np.ascontiguousarray(np.concatenate([g.reshape(-1) for g in groups]),
                                    dtype=np.int64)
        _lib.call("alefsi_mg_set_patches", self._h, l, len(groups), n_p, npn, flat)
        P = lv["P"].tocsr()
        _lib.call("alefsi_mg_set_prolongation", self._h, l, P.shape[0], P.shape[1], P.nnz,
                  np.ascontiguousarray(P.indptr, dtype=np.int64),
                  np.ascontiguousarray(P.indices, dtype=np.int32),
                  np.ascontiguousarray(P.data, dtype=np.float64))

    def factorize(self):
        _lib.call("alefsi_mg_factorize", self._h)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.call("alefsi_mg_destroy", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self, level):
        out = np.zeros(8, dtype=np.int64)
        _lib.call("alefsi_mg_info", self._h, level, out)
        return dict(zip(["n_nodes", "ndof", "nnzb", "nnz_pp", "n_groups", "y_size",
                         "inverse_doubles", "ld"], out.tolist()))

    def kernel_launches(self):
        out = np.zeros(1, dtype=np.int64)
        _lib.call("alefsi_kernel_stats", self._h, out)
        return int(out[0])

    KINDS = ["spmv", "vanka_apply", "vanka_gather", "restrict", "prolong", "coarse", "krylov"]

    def profile(self, on=True):
        """Toggle live CUDA-event timing of every kernel on the launch stream."""
        _lib.call("alefsi_mg_profile", self._h, 1 if on else 0)

    def profile_read(self, reset=True):
        """{(kind, finest): (launches, total_ms)} since the last reset."""
        counts = np.zeros(14, dtype=np.int64)
        ms = np.zeros(14, dtype=np.float64)
        _lib.call("alefsi_mg_profile_read", self._h, counts, ms, 1 if reset else 0)
        out = {}
        for i in range(14):
            out[(self.KINDS[i % 7], bool(i // 7))] = (int(counts[i]), float(ms[i]))
        return out

    def inverses(self, level, group):
        """Stored inverses of one patch group: (n_patches, np, np), row-major."""
        n_p, npd = self._groups[level][group]
        ld = npd + (npd % 2)
        out = np.empty(n_p * npd * ld, dtype=np.float64)
        _lib.call("alefsi_mg_get_inverses", self._h, level, group, out)
        return out.reshape(n_p, npd, ld)[:, :, :npd].transpose(0, 2, 1)

    # -- application --------------------------------------------------------------
    def dot(self, b):
        """One V-cycle (MgSolver.dot, reference linsolve.py:238-255)."""
        if _is_device(b):
            import torch
            self._bind_torch_stream()
            z = torch.empty_like(b)
            _lib.call("alefsi_mg_apply", self._h, b, z, 0)
            return z
        b = np.ascontiguousarray(b, dtype=np.float64)
        z = np.empty_like(b)
        _lib.call("alefsi_mg_apply", self._h, b, z, 1)
        return z

    __call__ = dot

    def gmres(self, b, rel_tol=1e-4, abs_tol=0.0, max_iter=200, x_out=None, raise_on_fail=True):
        """Right-preconditioned GMRES (reference linsolve.py:41-115)."""
        import time
        t0 = time.perf_counter()
        res = np.zeros(max_iter + 1, dtype=np.float64)
        its = np.zeros(1, dtype=np.int32)
        conv = np.zeros(1, dtype=np.int32)
        if _is_device(b):
            import torch
            self._bind_torch_stream()
            x = x_out if x_out is not None else torch.empty_like(b)
            host = 0
        else:
            b = np.ascontiguousarray(b, dtype=np.float64)
            x = x_out if x_out is not None else np.empty_like(b)
            host = 1
        try:
            _lib.call("alefsi_gmres", self._h, b, x, float(rel_tol), float(abs_tol), int(max_iter),
                      host, res, its, conv)
            err = None
        except _lib.NativeError as exc:
            if exc.code != 4:        # ALEFSI_ERR_NOT_CONVERGED
                raise
            err = exc
        n = int(its[0])
        stats = KrylovStats(iterations=n, initial_residual=float(res[0]),
                            final_residual=float(res[n]), residuals=res[:n + 1].tolist(),
                            converged=bool(conv[0]), elapsed=time.perf_counter() - t0)
        if err is not None and raise_on_fail:
            tol = max(rel_tol * stats.initial_residual, abs_tol)
            raise SolverError(f"GMRES stalled at {stats.final_residual:.3e} (tol {tol:.3e}) "
                              f"after {stats.iterations} iterations", stats)
        return x, stats

    # -- single kernels (parity tests, micro-benchmarks; device tensors) ------------
    def spmv(self, level, x, b=None, y=None):
        self._bind_torch_stream()
        import torch
        y = torch.empty_like(x) if y is None else y
        _lib.call("alefsi_mg_spmv", self._h, level, x, b if b is not None else None, y)
        return y

    def set_sell(self, level, lanes_per_row):
        """Re-lay a 2D level's SpMV copy out as sliced ELL with 1, 2 or 4
        lanes per row (0: CSR half-warp kernel); see alefsi_mg_set_sell."""
        _lib.call("alefsi_mg_set_sell", self._h, level, int(lanes_per_row))

    def set_apply_split(self, level, split):
        """Vanka apply form of a level: -1 default, 0 unsplit, 1 column-split
        (alefsi_mg_set_apply_split)."""
        _lib.call("alefsi_mg_set_apply_split", self._h, level, int(split))

    def sweep(self, level, x, b):
        self._bind_torch_stream()
        _lib.call("alefsi_mg_vanka_sweep", self._h, level, x, b)
        return x

    def restrict(self, level, r_fine, out):
        self._bind_torch_stream()
        _lib.call("alefsi_mg_restrict", self._h, level, r_fine, out)
        return out

    def prolong_add(self, level, x_coarse, x_fine):
        self._bind_torch_stream()
        _lib.call("alefsi_mg_prolong_add", self._h, level, x_coarse, x_fine)
        return x_fine

    def coarse_solve(self, b, x):
        self._bind_torch_stream()
        _lib.call("alefsi_mg_coarse_solve", self._h, b, x)
        return x

    def reserve(self, max_iter):
        _lib.call("alefsi_gmres_workspace", self._h, int(max_iter))

    # -- device assembly of the condensed Jacobian -----------------------------------
    def asm_setup(self, level, lvl):
        """Upload cell topology, geometry, colour groups, LPS entries and the
        Dirichlet mask of one LevelData for device assembly."""
        from . import mesh as mm
        m = lvl.mesh
        d = lvl.dim
        groups, kinds = [], []
        for cells, kind in ((lvl.fluid_cells, 0), (lvl.solid_cells, 1)):
            if len(cells) == 0:
                continue
            ps = mm.PatchSet(n_comp=1)
            ps.add(m.cell_nodes[cells], 0)
            col = mm.color_patches(ps)
            for c in range(col.n_colors):
                groups.append(cells[col.color == c])
                kinds.append(kind)
        gptr = np.concatenate([[0], np.cumsum([len(g) for g in groups])]).astype(np.int64)
        gcells = np.ascontiguousarray(np.concatenate(groups), dtype=np.int32)
        p = lvl.pattern
        _lib.call("alefsi_mg_asm_setup", self._h, level, d, len(m.cells),
                  np.ascontiguousarray(m.cell_nodes, dtype=np.int32),
                  np.ascontiguousarray(m.nodes, dtype=np.float64), len(groups), gptr,
                  np.asarray(kinds, dtype=np.int32), gcells, len(p.macro_to_cell),
                  np.ascontiguousarray(p.macro_to_cell, dtype=np.int64),
                  np.ascontiguousarray(p.macro_to_pp, dtype=np.int64),
                  np.ascontiguousarray(lvl.lps_macro_vals, dtype=np.float64),
                  np.ascontiguousarray(lvl.momentum_dirichlet.reshape(-1), dtype=np.uint8))
        t = lvl.table
        _lib.call("alefsi_mg_asm_tables", self._h, d, t.N.shape[0],
                  np.ascontiguousarray(t.N), np.ascontiguousarray(t.dN),
                  np.ascontiguousarray(lvl.quad_weights))
        fq = lvl.outflow
        if fq is not None and len(fq.cells):
            # slot reduction plan in np.add.at order (model._outflow_blocks)
            from . import fem
            sl = fem.pattern_slots(p.indptr, p.indices, fq.conn).reshape(-1)
            uniq, inv = np.unique(sl, return_inverse=True)
            contrib = np.argsort(inv, kind="stable").astype(np.int64)
            uptr = np.concatenate([[0], np.cumsum(np.bincount(inv, minlength=len(uniq)))])
            _lib.call("alefsi_mg_asm_outflow", self._h, level, len(fq.cells), fq.N.shape[1],
                      np.ascontiguousarray(fq.conn, dtype=np.int32),
                      np.ascontiguousarray(fq.cells, dtype=np.int64),
                      np.ascontiguousarray(fq.N, dtype=np.float64),
                      np.ascontiguousarray(fq.G, dtype=np.float64),
                      np.ascontiguousarray(fq.dS, dtype=np.float64),
                      np.ascontiguousarray(fq.normal, dtype=np.float64), len(uniq),
                      np.ascontiguousarray(uniq, dtype=np.int64), uptr.astype(np.int64), contrib)
            self._device_outflow.add(level)
        # residual tail: outflow rows per node (np.add.at order) and LPS CSR
        L = lvl.lps_csr()
        onodes = np.zeros(0, dtype=np.int64)
        ouptr = np.zeros(1, dtype=np.int64)
        ocontrib = np.zeros(0, dtype=np.int64)
        if level in self._device_outflow:
            onodes, inv = np.unique(fq.conn.reshape(-1), return_inverse=True)
            ocontrib = np.argsort(inv, kind="stable").astype(np.int64)
            ouptr = np.concatenate([[0], np.cumsum(np.bincount(inv, minlength=len(onodes)))])
        _lib.call("alefsi_mg_asm_residual_tables", self._h, level,
                  np.ascontiguousarray(L.indptr, dtype=np.int64),
                  np.ascontiguousarray(L.indices, dtype=np.int32),
                  np.ascontiguousarray(L.data, dtype=np.float64), len(onodes),
                  np.ascontiguousarray(onodes, dtype=np.int64), ouptr.astype(np.int64), ocontrib)
        self._device_tail.add(level)

    def asm_momentum(self, level, lvl, mats, k, theta, U, U_prev):
        """Assemble the condensed Jacobian of one level on the device (cells,
        outflow facets, LPS, Dirichlet rows); refactorise afterwards."""
        from . import fem, model
        d = lvl.dim
        nc = d + 1
        slots = np.zeros(0, dtype=np.int64)
        vals = np.zeros((0, nc, nc))
        if lvl.outflow is not None and level not in self._device_outflow:
            with fem.single_blas():
                local = model._outflow_blocks(lvl.outflow, U, mats, k, theta, d)
            if getattr(lvl, "_outflow_slots", None) is None:    # state independent
                sl = fem.pattern_slots(lvl.pattern.indptr, lvl.pattern.indices,
                                       lvl.outflow.conn).reshape(-1)
                lvl._outflow_slots = np.unique(sl, return_inverse=True)
            slots, inv = lvl._outflow_slots
            vals = np.zeros((len(slots), nc, nc))
            np.add.at(vals, inv, local.reshape(-1, nc, nc))
        params = np.array([mats.rho_f, mats.mu_f, mats.rho_s, mats.mu_s, mats.lam_s, k, theta])
        _lib.call("alefsi_mg_asm_momentum", self._h, level, params,
                  np.ascontiguousarray(U, dtype=np.float64),
                  np.ascontiguousarray(U_prev, dtype=np.float64), len(slots),
                  np.ascontiguousarray(slots, dtype=np.int64),
                  np.ascontiguousarray(vals, dtype=np.float64))

    def asm_residual(self, level, lvl, mats, flags, k, theta, U, U_prev, which=0):
        """Cell parts of the theta residual (which=0) or of the explicit
        previous-state forces (which=1) evaluated on the device."""
        d = lvl.dim
        f = list(mats.body_force) + [0.0] * (3 - len(mats.body_force))
        params = np.array([mats.rho_f, mats.mu_f, mats.rho_s, mats.mu_s, mats.lam_s, k, theta,
                           f[0], f[1], f[2], 0.0 if flags.extension_model == "harmonic" else 1.0,
                           flags.ext_mu, flags.ext_lam, 1.0 if flags.ext_volume_scaling else 0.0])
        out = np.zeros((lvl.n_nodes, 1 + 2 * d if which == 0 else d))
        _lib.call("alefsi_mg_asm_residual", self._h, level, params,
                  None if U is None else np.ascontiguousarray(U, dtype=np.float64),
                  np.ascontiguousarray(U_prev, dtype=np.float64), which, out)
        return out

    def matrix_data(self, level, pattern):
        data = np.empty((pattern.nnzb, self.nc, self.nc))
        pp = np.empty(pattern.nnz_pp)
        _lib.call("alefsi_mg_get_matrix", self._h, level, data, pp)
        return data, pp

    # -- construction from a workload case -------------------------------------------
    @classmethod
    def from_case(cls, case, wl, **kw):
        return cls(case.mg_levels(), nu_pre=wl.nu_pre, nu_post=wl.nu_post, omega=wl.omega, **kw)
