"""Continuum kinematics and the condensed momentum Jacobian.

Host-side mirror of the reference's model module (reference
pkg/src/alefsi/model.py).  ``momentum_jacobian`` assembles the reduced
velocity-pressure Jacobian of reference model.py:297-381 (deformation
derivatives dropped, solid deformation condensed onto the velocity through
u_n = u_{n-1} + k theta v_n + k (1-theta) v_{n-1}) directly into the split
block layout of ``fem.SplitBlockMatrix``, processing cells in chunks so the
3D 4.3M-dof level fits in host memory.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fem


class InvertedElementError(Exception):
    pass


@dataclass
class MaterialParams:
    rho_f: float = 1.0e3
    nu_f: float = 1.0e-3
    rho_s: float = 1.0e3
    mu_s: float = 2.0e6
    lam_s: float = 8.0e6
    body_force: tuple = (0.0, 0.0)

    def __post_init__(self):
        for name in ("rho_f", "nu_f", "rho_s", "mu_s", "lam_s"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    @property
    def mu_f(self):
        return self.rho_f * self.nu_f

    def density_scaled(self):
        """Same problem divided by rho_f (reference model.py:44-54)."""
        r = self.rho_f
        return MaterialParams(rho_f=1.0, nu_f=self.nu_f, rho_s=self.rho_s / r,
                              mu_s=self.mu_s / r, lam_s=self.lam_s / r,
                              body_force=self.body_force), r


def _fields(G, N, Uc, d):
    """Values and gradients of v (comps 1..d) and u (comps d+1..2d) at qpoints."""
    v = np.einsum("qb,cbi->cqi", N, Uc[:, :, 1:1 + d])
    u = np.einsum("qb,cbi->cqi", N, Uc[:, :, 1 + d:])
    gv = np.einsum("cqbj,cbi->cqij", G, Uc[:, :, 1:1 + d], optimize=True)
    gu = np.einsum("cqbj,cbi->cqij", G, Uc[:, :, 1 + d:], optimize=True)
    return v, u, gv, gu


def _fluid_kin(gu):
    F = gu + np.eye(gu.shape[-1])
    J = np.linalg.det(F)
    if np.any(J <= 0):
        raise InvertedElementError(f"fluid cell inverted, min J = {np.min(J):g}")
    return F, J, np.linalg.inv(F)


def _fluid_blocks(G, N, wdet, Uc, Upc, mats, k, theta):
    """Local (c, b, a, nc, nc) blocks of the fluid rows: row test function b,
    column trial function a (reference model.py:303-337)."""
    C, nq, nb, d = G.shape
    nc = d + 1
    v, u, gv, gu = _fields(G, N, Uc, d)
    _, up, _, gup = _fields(G, N, Upc, d)
    F, J, Fi = _fluid_kin(gu)
    Fp, Jp, _ = _fluid_kin(gup)
    Jbar = 0.5 * (J + Jp)
    w = np.einsum("cqij,cqj->cqi", np.linalg.inv(0.5 * (F + Fp)), u - up)
    Fiv = np.einsum("cqij,cqj->cqi", Fi, v)
    FiTG = np.einsum("cqmi,cqam->cqai", Fi, G, optimize=True)        # (F^-T grad phi_a)_i
    K = Fi @ np.swapaxes(Fi, -1, -2)
    gvFi = gv @ Fi
    rho, mu, kt = mats.rho_f, mats.mu_f, k * theta

    out = np.zeros((C, nb, nb, nc, nc))
    coef = ((-0.5 * rho * Jbar)[..., None] * np.einsum("cqam,cqm->cqa", G, w)
            + (kt * rho * J)[..., None] * np.einsum("cqam,cqm->cqa", G, Fiv))
    wN = wdet[:, :, None] * N[None]                                    # (c, q, b)
    diag = np.matmul(np.swapaxes(wN, 1, 2), coef)
    diag += np.matmul(np.swapaxes((wdet * rho * Jbar)[:, :, None] * N[None], 1, 2), N[None])
    GK = np.einsum("cqbl,cqlm->cqbm", G, K, optimize=True) * (wdet * kt * mu * J)[:, :, None, None]
    diag += np.matmul(GK.transpose(0, 2, 1, 3).reshape(C, nb, nq * d),
                      G.transpose(0, 1, 3, 2).reshape(C, nq * d, nb))
    for i in range(d):
        out[:, :, :, 1 + i, 1 + i] += diag
    # transported-gradient convection: N_b N_a (grad v F^-1)_ij
    NN = (N[:, :, None] * N[:, None, :]).reshape(nq, nb * nb)         # (q, b*a)
    X = ((wdet * kt * rho * J)[:, :, None, None] * gvFi).reshape(C, nq, d * d)
    out[:, :, :, 1:, 1:] += np.matmul(NN.T[None], X).reshape(C, nb, nb, d, d)
    # second viscous piece: FiTG[a,i] FiTG[b,j]
    A1 = ((wdet * kt * mu * J)[:, :, None, None] * FiTG).reshape(C, nq, nb * d)   # (b, j)
    A2 = FiTG.reshape(C, nq, nb * d)                                              # (a, i)
    V = np.matmul(np.swapaxes(A1, 1, 2), A2).reshape(C, nb, d, nb, d)             # b j a i
    out[:, :, :, 1:, 1:] += V.transpose(0, 1, 3, 4, 2)
    # pressure column (b, vel i; a, p): -k J N_a FiTG[b,i]
    P = ((wdet * (-k) * J)[:, :, None, None] * FiTG).reshape(C, nq, nb * d)
    out[:, :, :, 1:, 0] += np.matmul(np.swapaxes(P, 1, 2), N[None]).reshape(
        C, nb, d, nb).transpose(0, 1, 3, 2)
    # divergence row (b, p; a, vel j): k J N_b FiTG[a,j]
    D = ((wdet * k * J)[:, :, None, None] * FiTG).reshape(C, nq, nb * d)
    out[:, :, :, 0, 1:] += np.matmul(N.T[None], D).reshape(C, nb, nb, d)
    return out


def _solid_blocks(G, N, wdet, Uc, Upc, mats, k, theta):
    """Mass + condensed St. Venant-Kirchhoff tangent (reference model.py:339-361)."""
    C, nq, nb, d = G.shape
    nc = d + 1
    _, _, gv, _ = _fields(G, N, Uc, d)
    _, _, gvp, gup = _fields(G, N, Upc, d)
    g = gup + k * theta * gv + k * (1.0 - theta) * gvp
    F = g + np.eye(d)
    J = np.linalg.det(F)
    if np.any(J <= 0):
        raise InvertedElementError(f"min det(F) = {np.min(J):g}")
    E = 0.5 * (np.swapaxes(F, -1, -2) @ F - np.eye(d))
    tr = np.trace(E, axis1=-2, axis2=-1)
    Sig = 2.0 * mats.mu_s * E + mats.lam_s * tr[..., None, None] * np.eye(d)
    kt2 = (k * theta) ** 2
    out = np.zeros((C, nb, nb, nc, nc))
    mass = np.matmul(np.swapaxes((wdet * mats.rho_s)[:, :, None] * N[None], 1, 2), N[None])
    GS = np.einsum("cqas,cqsm->cqam", G, Sig, optimize=True) * (wdet * kt2)[:, :, None, None]
    sA = np.matmul(G.transpose(0, 2, 1, 3).reshape(C, nb, nq * d),
                   GS.transpose(0, 1, 3, 2).reshape(C, nq * d, nb))            # [b, a]
    for i in range(d):
        out[:, :, :, 1 + i, 1 + i] += mass + sA
    FG = np.einsum("cqim,cqam->cqai", F, G, optimize=True)
    FFt = F @ np.swapaxes(F, -1, -2)
    wm = (wdet * kt2 * mats.mu_s)[:, :, None, None]
    A1 = (wm * FG).reshape(C, nq, nb * d)
    A2 = FG.reshape(C, nq, nb * d)
    sB = np.matmul(np.swapaxes(A1, 1, 2), A2).reshape(C, nb, d, nb, d)         # b j a i
    out[:, :, :, 1:, 1:] += sB.transpose(0, 1, 3, 4, 2)
    GG = np.matmul(G.transpose(0, 1, 2, 3).reshape(C * nq, nb, d),
                   G.reshape(C * nq, nb, d).transpose(0, 2, 1)).reshape(C, nq, nb, nb)  # [a,b]
    X = (wdet * kt2 * mats.mu_s)[:, :, None, None] * FFt                           # (c,q,i,j)
    sC = np.einsum("cqab,cqij->cbaij", GG, X, optimize=True)
    out[:, :, :, 1:, 1:] += sC
    wl = (wdet * kt2 * mats.lam_s)[:, :, None, None]
    A1 = (wl * FG).reshape(C, nq, nb * d)                                          # (b, i)
    sD = np.matmul(np.swapaxes(A1, 1, 2), A2).reshape(C, nb, d, nb, d)           # b i a j
    out[:, :, :, 1:, 1:] += sD.transpose(0, 1, 3, 2, 4)
    return out


def _outflow_blocks(fq, U, mats, k, theta, d):
    """Implicit do-nothing correction (reference model.py:363-375)."""
    gu = fq.eval_grad(U[:, 1 + d:])
    _, J, Fi = _fluid_kin(gu)
    FiTG = np.einsum("cqmi,cqam->cqai", Fi, fq.G)
    Fin = np.einsum("cqmi,cqm->cqi", Fi, fq.normal)
    coef = -k * theta * mats.mu_f * J * fq.dS
    nf, nq, nb = fq.N.shape
    out = np.zeros((nf, nb, nb, d + 1, d + 1))
    out[:, :, :, 1:, 1:] = np.einsum("cq,cqb,cqai,cqj->cbaij", coef, fq.N, FiTG, Fin,
                                     optimize=True)
    return out


def momentum_jacobian(lvl, mats, flags, k, theta, U, U_prev, chunk=2048):
    """Reduced (p, v) Jacobian on one level in the split block layout."""
    with fem.single_blas():
        return _momentum_jacobian(lvl, mats, flags, k, theta, U, U_prev, chunk)


def _momentum_jacobian(lvl, mats, flags, k, theta, U, U_prev, chunk):
    d = lvl.dim
    nc = d + 1
    p = lvl.pattern
    A = fem.SplitBlockMatrix(p, np.zeros((p.nnzb, nc, nc)), np.zeros(p.nnz_pp))
    N = lvl.table.N
    conn_all = lvl.mesh.cell_nodes
    for cells, kernel in ((lvl.fluid_cells, _fluid_blocks), (lvl.solid_cells, _solid_blocks)):
        def work(s, cells=cells, kernel=kernel):
            c = cells[s:s + chunk]
            conn = conn_all[c]
            return conn, kernel(lvl.G[c], N, lvl.wdet[c], U[conn], U_prev[conn], mats, k, theta)

        def scatter(res):
            # in chunk order: same accumulation order as one sequential pass
            fem.scatter_blocks(p.indptr, p.indices, A.data, res[0], res[1])
        fem.parallel_chunks(work, range(0, len(cells), chunk), scatter)
    if lvl.outflow is not None:
        local = _outflow_blocks(lvl.outflow, U, mats, k, theta, d)
        fem.scatter_blocks(p.indptr, p.indices, A.data, lvl.outflow.conn, local)
    # pressure stabilisation into the (p, p) entries
    vals = k * lvl.lps_macro_vals
    inc = p.macro_to_cell >= 0
    np.add.at(A.data[:, 0, 0], p.macro_to_cell[inc], vals[inc])
    A.pp_data[p.macro_to_pp[~inc]] += vals[~inc]
    fem.apply_dirichlet_rows(A, lvl.momentum_dirichlet)
    return A
