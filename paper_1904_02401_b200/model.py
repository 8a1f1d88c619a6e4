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
    # same contraction order as the reference (model.py:119-131): the
    # Newton/GMRES iteration counts of the time loop are sensitive to the
    # last bit of the residual near the 1e-4 linear tolerance
    v = np.einsum("qb,cbi->cqi", N, Uc[:, :, 1:1 + d])
    u = np.einsum("qb,cbi->cqi", N, Uc[:, :, 1 + d:])
    gv = np.einsum("cqbj,cbi->cqij", G, Uc[:, :, 1:1 + d])
    gu = np.einsum("cqbj,cbi->cqij", G, Uc[:, :, 1 + d:])
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


def kinematics(grad_u):
    """F = I + grad u, J, F^-1, E (reference model.py:65-75)."""
    d = grad_u.shape[-1]
    F = grad_u + np.eye(d)
    J = np.linalg.det(F)
    if np.any(J <= 0):
        raise InvertedElementError(f"min det(F) = {np.min(J):g}")
    return F, J, np.linalg.inv(F), 0.5 * (np.swapaxes(F, -1, -2) @ F - np.eye(d))


def _svk(F, E, mats):
    """First Piola stress F Sigma of St. Venant-Kirchhoff (model.py:101-106)."""
    d = F.shape[-1]
    tr = np.trace(E, axis1=-2, axis2=-1)
    return F @ (2.0 * mats.mu_s * E + mats.lam_s * tr[..., None, None] * np.eye(d))


def deformation_update(U, U_prev, k, theta, nodes):
    """u_n = u_{n-1} + k theta v_n + k (1-theta) v_{n-1} on nodes (model.py:109-114)."""
    d = (U.shape[1] - 1) // 2
    U[nodes, 1 + d:] = (U_prev[nodes, 1 + d:] + k * theta * U[nodes, 1:1 + d]
                        + k * (1.0 - theta) * U_prev[nodes, 1:1 + d])


def _test(wdet, N, G, val, grad):
    """sum_q w (N_b val_i + G_b . grad_i) -> (c, b, i) (model.py:147-154)."""
    out = 0.0
    if val is not None:
        out = out + np.einsum("cq,qb,cqi->cbi", wdet, N, val)
    if grad is not None:
        out = out + np.einsum("cq,cqbj,cqij->cbi", wdet, G, grad)
    return out


def _qfields(lvl, cells, U):
    d = lvl.dim
    Uc = U[lvl.mesh.cell_nodes[cells]]
    N = lvl.table.N
    p = np.einsum("qb,cb->cq", N, Uc[:, :, 0])
    v, u, gv, gu = _fields(lvl.G[cells], N, Uc, d)
    return p, v, u, gv, gu


def outflow_correction(lvl, mats, U, X, scale=1.0):
    """Do-nothing correction -(mu J F^-T grad(v)^T F^-T n, phi) on the outflow
    facets (reference model.py:191-205)."""
    fq = lvl.outflow
    if fq is None:
        return
    d = lvl.dim
    gv = fq.eval_grad(U[:, 1:1 + d])
    gu = fq.eval_grad(U[:, 1 + d:])
    _, J, Fi = _fluid_kin(gu)
    FiT = np.swapaxes(Fi, -1, -2)
    t = np.einsum("cqij,cqj->cqi", FiT @ np.swapaxes(gv, -1, -2) @ FiT, fq.normal)
    local = np.einsum("cq,cqb,cqi->cbi", fq.dS, fq.N, -scale * mats.mu_f * J[..., None] * t)
    np.add.at(X, fq.conn, local)


def explicit_forces(lvl, mats, flags, U_prev):
    """A_F + A_S of the previous state (reference model.py:159-188)."""
    d = lvl.dim
    X = np.zeros((lvl.n_nodes, d))
    f = np.asarray(mats.body_force, dtype=float)

    def fluid_local(cells):
        _, v, _, gv, gu = _qfields(lvl, cells, U_prev)
        _, J, Fi = _fluid_kin(gu)
        gvFi = gv @ Fi
        conv = mats.rho_f * J[..., None] * np.einsum("cqij,cqj->cqi", gvFi, v)
        conv = conv - mats.rho_f * J[..., None] * f
        visc = mats.mu_f * J[..., None, None] * ((gvFi + np.swapaxes(gvFi, -1, -2))
                                                 @ np.swapaxes(Fi, -1, -2))
        return _test(lvl.wdet[cells], lvl.table.N, lvl.G[cells], conv, visc)

    def solid_local(cells):
        _, v, _, _, gu = _qfields(lvl, cells, U_prev)
        F, _, _, E = kinematics(gu)
        sval = -mats.rho_s * np.broadcast_to(f, v.shape)
        return _test(lvl.wdet[cells], lvl.table.N, lvl.G[cells], sval, _svk(F, E, mats))

    with fem.single_blas():
        _chunked_scatter(lvl, lvl.fluid_cells, fluid_local, X)
        _chunked_scatter(lvl, lvl.solid_cells, solid_local, X)
        outflow_correction(lvl, mats, U_prev, X)
    return X


def theta_residual(lvl, mats, flags, k, theta, U, U_prev, explicit=None, device=None):
    """Residual of one theta step with constrained rows zeroed
    (reference model.py:208-292).  Returns (R, explicit).

    ``device = (DeviceMgSolver, level)`` evaluates the cell integrals (the
    bulk of the work) on the GPU; facet, LPS, mass-relation and masking terms
    stay on the host."""
    with fem.single_blas():
        if device is None:
            return _theta_residual(lvl, mats, flags, k, theta, U, U_prev, explicit)
        mg, level = device
        tail = level in getattr(mg, "_device_tail", ())   # outflow + LPS terms on device
        if explicit is None:
            explicit = mg.asm_residual(level, lvl, mats, flags, k, theta, None, U_prev, which=1)
            if not tail:
                outflow_correction(lvl, mats, U_prev, explicit)
        R = mg.asm_residual(level, lvl, mats, flags, k, theta, U, U_prev, which=0)
        return _residual_tail(lvl, mats, k, theta, U, U_prev, explicit, R,
                              device_tail=tail), explicit


def _chunked_scatter(lvl, cells, fn, out, chunk=1024):
    """out[conn] += fn(cell chunk) over chunks computed on a thread pool and
    accumulated in chunk order (same order as one np.add.at over all cells)."""
    conn = lvl.mesh.cell_nodes

    def work(s):
        c = cells[s:s + chunk]
        return c, fn(c)

    def consume(res):
        np.add.at(out, conn[res[0]], res[1])
    fem.parallel_chunks(work, range(0, len(cells), chunk), consume)


def _theta_residual(lvl, mats, flags, k, theta, U, U_prev, explicit):
    d = lvl.dim
    n = lvl.n_nodes
    if explicit is None:
        explicit = explicit_forces(lvl, mats, flags, U_prev)
    R = np.zeros((n, 1 + 2 * d))
    f = np.asarray(mats.body_force, dtype=float)
    N = lvl.table.N

    def fluid_local(cells):
        wdet, G = lvl.wdet[cells], lvl.G[cells]
        p, v, u, gv, gu = _qfields(lvl, cells, U)
        _, vp, up, gvp, gup = _qfields(lvl, cells, U_prev)
        F, J, Fi = _fluid_kin(gu)
        Fp, Jp, _ = _fluid_kin(gup)
        Jbar = 0.5 * (J + Jp)
        w = np.einsum("cqij,cqj->cqi", np.linalg.inv(0.5 * (F + Fp)), u - up)
        gvFi = gv @ Fi
        mom_val = (mats.rho_f * Jbar[..., None] * (v - vp)
                   - mats.rho_f * Jbar[..., None] * np.einsum("cqij,cqj->cqi", 0.5 * (gv + gvp), w)
                   + k * theta * mats.rho_f * J[..., None]
                   * (np.einsum("cqij,cqj->cqi", gvFi, v) - f))
        FiT = np.swapaxes(Fi, -1, -2)
        mom_grad = (k * theta * mats.mu_f * J[..., None, None]
                    * (gvFi + np.swapaxes(gvFi, -1, -2)) @ FiT
                    - k * (J * p)[..., None, None] * FiT)
        div_val = k * (J * np.einsum("cqij,cqji->cq", gv, Fi))
        if flags.extension_model == "harmonic":
            ext_grad = k * gu
        else:
            eps = 0.5 * (gu + np.swapaxes(gu, -1, -2))
            tr = np.einsum("cqii->cq", eps)
            ext_grad = k * (2.0 * flags.ext_mu * eps + flags.ext_lam * tr[..., None, None] * np.eye(d))
            if flags.ext_volume_scaling:
                ext_grad = ext_grad * lvl.inv_cell_volume[cells][:, None, None, None]
        local = np.zeros((len(cells), N.shape[1], 1 + 2 * d))
        local[:, :, 0] = np.einsum("cq,qb,cq->cb", wdet, N, div_val)
        local[:, :, 1:1 + d] = _test(wdet, N, G, mom_val, mom_grad)
        local[:, :, 1 + d:] = _test(wdet, N, G, None, ext_grad)
        return local

    def solid_local(cells):
        wdet, G = lvl.wdet[cells], lvl.G[cells]
        _, v, _, gv, _ = _qfields(lvl, cells, U)
        _, vp, _, gvp, gup = _qfields(lvl, cells, U_prev)
        F, _, _, E = kinematics(gup + k * theta * gv + k * (1.0 - theta) * gvp)
        sval = mats.rho_s * (v - vp) - k * theta * mats.rho_s * f
        local = np.zeros((len(cells), N.shape[1], 1 + 2 * d))
        local[:, :, 1:1 + d] = _test(wdet, N, G, sval, k * theta * _svk(F, E, mats))
        return local

    _chunked_scatter(lvl, lvl.fluid_cells, fluid_local, R)
    _chunked_scatter(lvl, lvl.solid_cells, solid_local, R)
    return _residual_tail(lvl, mats, k, theta, U, U_prev, explicit, R), explicit


def _residual_tail(lvl, mats, k, theta, U, U_prev, explicit, R, device_tail=False):
    """Explicit theta part, outflow correction, LPS, velocity-deformation
    relation rows and constraint masking (reference model.py:277-292).
    ``device_tail``: the outflow and LPS terms are already in R (added by
    the device residual)."""
    d = lvl.dim
    n = lvl.n_nodes
    R[:, 1:1 + d] += k * (1.0 - theta) * explicit
    if not device_tail:
        Xc = np.zeros((n, d))
        outflow_correction(lvl, mats, U, Xc, scale=k * theta)
        R[:, 1:1 + d] += Xc
        R[:, 0] += k * (lvl.lps_csr() @ U[:, 0])
    # the deficit is formed only on the columns the relation rows touch
    cols, M = lvl.solid_mass_relation()
    Uc, Upc = U[cols], U_prev[cols]
    deficit = (Uc[:, 1 + d:] - Upc[:, 1 + d:] - k * theta * Uc[:, 1:1 + d]
               - k * (1.0 - theta) * Upc[:, 1:1 + d])
    R[lvl.relation_nodes, 1 + d:] = M @ deficit
    if R.flags.c_contiguous:
        R.reshape(-1)[lvl.residual_zero_flat()] = 0.0
    else:
        R[lvl.residual_zero_mask] = 0.0
    return R


def extension_operator(lvl, flags):
    """State-independent mesh-extension operator on the fluid cells
    (reference model.py:442-461), split layout with nc = d."""
    d = lvl.dim
    import dataclasses
    # cell-stencil blocks only: the extension has no LPS macro couplings
    p = dataclasses.replace(lvl.pattern, pp_indptr=np.zeros(lvl.n_nodes + 1, dtype=np.int64),
                            pp_indices=np.zeros(0, dtype=np.int32))
    A = fem.SplitBlockMatrix(p, np.zeros((p.nnzb, d, d)), np.zeros(0))
    cells = lvl.fluid_cells
    if len(cells) == 0:
        return A
    # Cell Gram products of the basis gradients as batched BLAS matrix
    # products over the (quadrature point, component) axis (reference
    # model.py:442-461 writes them as einsums; same terms, BLAS summation
    # order, ~1e-16 relative)
    wdet, G = lvl.wdet[cells], lvl.G[cells]
    nq, nb = G.shape[1], G.shape[2]
    if flags.extension_model == "harmonic":
        w = wdet
    else:
        scale = lvl.inv_cell_volume[cells] if flags.ext_volume_scaling else np.ones(len(cells))
        w = wdet * scale[:, None]
    local = np.empty((len(cells), nb, nb, d, d))
    chunk = 2048

    def work(s):
        Gc, wc = G[s:s + chunk], w[s:s + chunk]
        m = len(Gc)
        if flags.extension_model == "harmonic":
            X = np.ascontiguousarray(Gc.transpose(0, 2, 1, 3)).reshape(m, nb, nq * d)
            Y = (Gc * wc[:, :, None, None]).transpose(0, 2, 1, 3).reshape(m, nb, nq * d)
            gg = np.matmul(Y, X.transpose(0, 2, 1))                       # (c, b, a)
            local[s:s + m] = gg[..., None, None] * np.eye(d)
        else:
            X = Gc.reshape(m, nq, nb * d)                                  # (q, a i)
            Y = (Gc * wc[:, :, None, None]).reshape(m, nq, nb * d)         # (q, b j)
            T1 = np.matmul(Y.transpose(0, 2, 1), X).reshape(m, nb, d, nb, d)
            T1 = T1.transpose(0, 1, 3, 4, 2)                               # (c, b, a, i, j)
            gg = np.trace(T1, axis1=3, axis2=4)                            # (c, b, a)
            local[s:s + m] = (flags.ext_mu * gg[..., None, None] * np.eye(d)
                              + flags.ext_mu * T1 + flags.ext_lam * np.swapaxes(T1, -1, -2))

    fem.parallel_chunks(work, range(0, len(cells), chunk))
    fem.scatter_blocks(p.indptr, p.indices, A.data, lvl.mesh.cell_nodes[cells], local)
    return A


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
