"""Element matrices, assembly and prolongation (oracle; test infrastructure).

Forms (eq. CoupledFormu), restricted to a box of a Kuhn mesh:

* mass            (p, v)                         -> |K| mass22
* stiffness       (grad p, grad v)               -> |K| sum_kl (G_k . G_l) grad22
* deformation     2 nu eta (D(u), D(v))          (a_c_eta volume part)
* divergence      b_eta(v, p) = -eta (p, div v)
* convection      b_N_eta(w, u, v) = eta ((w . grad) u, v), plain form (C10)
* facet terms on Gamma: friction eta nu alpha sqrt(d)/sqrt(tr Pi) <P_tau u, P_tau v>
  with Pi = k_F I, i.e. eta nu alpha / sqrt(k_F); the interface
  loads (eta/rho) int p_F v.n_c and (eta nu alpha sqrt(k_F)/mu) int grad_tau p_F . P_tau v
  (P:203-204); the porous flux int v_F u.n_c.

Each is computed per element from its vertex coordinates (no use of the
translation invariance of Kuhn meshes), with the exact reference tensors of
poly.py, and assembled with scipy.sparse.
"""
from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np
import scipy.sparse as sp

from . import mesh as M
from .poly import edges, eval_p2, ftensors


def geometry(X: np.ndarray):
    """X (E, d+1, d) vertex coordinates -> (|K| (E,), grad lambda (E, d+1, d))."""
    d = X.shape[-1]
    J = np.transpose(X[:, 1:, :] - X[:, :1, :], (0, 2, 1))  # columns X_k - X_0
    det = np.linalg.det(J)
    vol = np.abs(det) / float(np.prod(range(1, d + 1)))
    Jinv = np.linalg.inv(J)  # rows: grad lambda_1..d
    G = np.empty((X.shape[0], d + 1, d))
    G[:, 1:, :] = Jinv
    G[:, 0, :] = -Jinv.sum(axis=1)
    return vol, G


def _coo(rows, cols, vals, shape):
    return sp.coo_matrix((vals.ravel(), (rows.ravel(), cols.ravel())), shape=shape).tocsr()


class BoxFEM:
    """All element-level data of one box (volume simplices + Gamma facets)."""

    def __init__(self, box: M.Box):
        self.box = box
        self.d = d = box.d
        p2, p1, gv, cell = box.simplices()
        self.p2, self.p1, self.cell = p2, p1, cell
        X = box.grid.coords(gv)
        self.vol, self.G = geometry(X)
        self.n2 = box.node_g.shape[0]
        self.n1 = box.vert_g.shape[0]
        self.T = ftensors(d)
        # Gamma facets inside the box
        self.facets = self._gamma_facets()

    # ---------------- volume forms ----------------
    def mass(self, coef=None) -> sp.csr_matrix:
        c = self.vol if coef is None else self.vol * coef
        Me = c[:, None, None] * self.T["mass22"][None]
        n = self.p2.shape[1]
        r = np.repeat(self.p2[:, :, None], n, axis=2)
        cc = np.repeat(self.p2[:, None, :], n, axis=1)
        return _coo(r, cc, Me, (self.n2, self.n2))

    def grad_products(self) -> np.ndarray:
        """(E, n2, n2, d, d): int dphi_i/dx_a dphi_j/dx_b."""
        # int dphi_i/dlam_k dphi_j/dlam_l * G[k,a] G[l,b]
        return np.einsum("ikjl,eka,elb->eijab", self.T["grad22"], self.G, self.G) * self.vol[:, None, None, None, None]

    def stiffness(self, coef=None) -> sp.csr_matrix:
        gp = self.grad_products()
        Ke = np.einsum("eijaa->eij", gp)
        if coef is not None:
            Ke = Ke * coef[:, None, None]
        n = self.p2.shape[1]
        r = np.repeat(self.p2[:, :, None], n, axis=2)
        cc = np.repeat(self.p2[:, None, :], n, axis=1)
        return _coo(r, cc, Ke, (self.n2, self.n2))

    def _vec_blocks(self, Be) -> sp.csr_matrix:
        """Be (E, n2, d, n2, d) element blocks [row node, row comp, col node, col comp] -> d*n2 square."""
        d, n = self.d, self.p2.shape[1]
        rows = (np.arange(d)[None, None, :] * self.n2 + self.p2[:, :, None])  # (E, n, d)
        R = np.broadcast_to(rows[:, :, :, None, None], Be.shape)
        C = np.broadcast_to(rows[:, None, None, :, :], Be.shape)
        return _coo(R, C, Be, (d * self.n2, d * self.n2))

    def deformation(self, nu_eta: float) -> sp.csr_matrix:
        """2 nu eta (D(u), D(v)): for u = phi_j e_b, v = phi_i e_a, D(u):D(v) = (delta_ab grad phi_i . grad phi_j
        + dphi_i/dx_b dphi_j/dx_a) / 2."""
        gp = self.grad_products()  # [e,i,j,a,b] = int d_a phi_i d_b phi_j
        E, n, d = gp.shape[0], gp.shape[1], self.d
        Be = np.zeros((E, n, d, n, d))
        lap = np.einsum("eijaa->eij", gp)
        for a in range(d):
            for b in range(d):
                # int d_b phi_i d_a phi_j = gp[e,i,j,b,a]
                Be[:, :, a, :, b] = nu_eta * ((lap if a == b else 0.0) + gp[:, :, :, b, a])
        return self._vec_blocks(Be)

    def vec_mass(self, coef: float) -> sp.csr_matrix:
        Me = (self.vol * coef)[:, None, None] * self.T["mass22"][None]
        return sp.block_diag([_coo(np.repeat(self.p2[:, :, None], Me.shape[1], 2),
                                   np.repeat(self.p2[:, None, :], Me.shape[1], 1), Me, (self.n2, self.n2))] * self.d).tocsr()

    def divergence(self, eta: float) -> sp.csr_matrix:
        """Bdiv[m, (b, j)] = eta int psi_m d_b phi_j  (n1 x d*n2).  b_eta(v, p) = -p^T Bdiv v."""
        # int psi_m dphi_j/dlam_l G[l,b]
        De = np.einsum("mjl,elb->emjb", self.T["div12"], self.G) * (eta * self.vol)[:, None, None, None]
        E, n1, n, d = De.shape
        R = np.broadcast_to(self.p1[:, :, None, None], De.shape)
        C = np.broadcast_to((np.arange(d)[None, None, None, :] * self.n2 + self.p2[:, None, :, None]), De.shape)
        return _coo(R, C, De, (self.n1, d * self.n2))

    def p1_mass_vector(self) -> np.ndarray:
        """m_k = int psi_k over the box (C6 multiplier row)."""
        out = np.zeros(self.n1)
        np.add.at(out, self.p1, self.vol[:, None] * self.T["mass1"][None, :])
        return out

    def _elem_vec(self, U: np.ndarray) -> np.ndarray:
        """U (d, n2) nodal vector field -> (E, d, n) element values."""
        return np.transpose(U[:, self.p2], (1, 0, 2))

    def convection(self, W: np.ndarray, eta: float) -> sp.csr_matrix:
        """eta ((w . grad) u, v) with wind w = W (d, n2) in P2: for u = phi_j e_b, v = phi_i e_a:
        delta_ab eta sum_c sum_m W_c,m int phi_i phi_m d_c phi_j."""
        We = self._elem_vec(W)  # (E, d, n)
        # int phi_i phi_m d_c phi_j = sum_l conv[i,m,j,l] G[l,c] |K|
        Ce = np.einsum("imjl,elc,ecm->eij", self.T["conv"], self.G, We) * (eta * self.vol)[:, None, None]
        E, n, d = Ce.shape[0], Ce.shape[1], self.d
        Be = np.zeros((E, n, d, n, d))
        for a in range(d):
            Be[:, :, a, :, a] = Ce
        return self._vec_blocks(Be)

    def convection_reaction(self, U: np.ndarray, eta: float) -> sp.csr_matrix:
        """eta ((e . grad) U, v) with fixed U (d, n2) in P2: for e = phi_j e_b, v = phi_i e_a:
        eta sum_m U_a,m int phi_i phi_j d_b phi_m."""
        Ue = self._elem_vec(U)  # (E, d, n)
        # int phi_i phi_j d_b phi_m = sum_l conv[i,j,m,l] G[l,b] |K|
        Te = np.einsum("ijml,elb,eam->eiajb", self.T["conv"], self.G, Ue) * (eta * self.vol)[:, None, None, None, None]
        return self._vec_blocks(Te)

    def convection_vector(self, U: np.ndarray, eta: float) -> np.ndarray:
        """eta ((U . grad) U, phi_i e_a) as a (d*n2,) vector."""
        return self.convection(U, eta) @ U.ravel()

    # ---------------- Gamma facets ----------------
    def _gamma_facets(self):
        box, d = self.box, self.d
        g_gamma = box.grid.gamma_g
        if not (2 * box.c0[-1] <= g_gamma <= 2 * box.c1[-1]):
            return None
        # (d-1)-dim Kuhn mesh of the face: cells over tangential axes, simplices over permutations of d-1 axes
        dt = d - 1
        lo = np.asarray(box.c0[:dt])
        hi = np.asarray(box.c1[:dt]) - 1
        fcells = M.lex_points(lo, hi)
        off = M.kuhn_offsets(dt)  # (S, dt+1, dt)
        verts = (fcells[:, None, None, :] + off[None]).reshape(-1, dt + 1, dt)
        eds = list(itertools.combinations(range(dt + 1), 2))
        gt = np.concatenate([2 * verts, np.stack([verts[:, a] + verts[:, b] for a, b in eds], axis=1)], axis=1)
        last = np.full(gt.shape[:-1] + (1,), g_gamma, dtype=np.int64)
        g_full = np.concatenate([gt, last], axis=-1)  # (F, n2f, d)
        idx = box.p2_index(g_full)
        X = box.grid.coords(np.concatenate([2 * verts, np.full(verts.shape[:-1] + (1,), g_gamma)], -1))[..., :dt]
        fvol, fG = geometry(X) if dt > 0 else (np.ones(len(verts)), np.zeros((len(verts), 1, 0)))
        fcell = np.repeat(fcells, off.shape[0], axis=0)
        return {"idx": idx, "vol": fvol, "G": fG, "cell": fcell, "T": ftensors(dt)}

    def facet_mass(self, coef=None) -> sp.csr_matrix:
        """int_{Gamma cap box} c phi_i phi_j (n2 x n2; zero rows off Gamma)."""
        f = self.facets
        if f is None:
            return sp.csr_matrix((self.n2, self.n2))
        c = f["vol"] if coef is None else f["vol"] * coef
        Me = c[:, None, None] * f["T"]["mass22"][None]
        n = f["idx"].shape[1]
        return _coo(np.repeat(f["idx"][:, :, None], n, 2), np.repeat(f["idx"][:, None, :], n, 1), Me, (self.n2, self.n2))

    def facet_tangential_grad(self, a: int, coef=None) -> sp.csr_matrix:
        """int_{Gamma cap box} c phi_i d_a phi_j, a a tangential axis (a < d-1)."""
        f = self.facets
        if f is None:
            return sp.csr_matrix((self.n2, self.n2))
        # int phi_i dphi_j/dlam_l G[l,a]: build from conv-free tensors: int phi_i dphi_j/dlam_l
        Tm = _facet_phi_dphi(self.d - 1)  # (n, n, dt+1)
        Te = np.einsum("ijl,el->eij", Tm, f["G"][:, :, a]) * (f["vol"] if coef is None else f["vol"] * coef)[:, None, None]
        n = f["idx"].shape[1]
        return _coo(np.repeat(f["idx"][:, :, None], n, 2), np.repeat(f["idx"][:, None, :], n, 1), Te, (self.n2, self.n2))


_PHI_DPHI = {}


def _facet_phi_dphi(d: int) -> np.ndarray:
    """(1/|K|) int phi_i dphi_j/dlam_l on a d-simplex (float)."""
    if d not in _PHI_DPHI:
        from .poly import p2_basis, poly_diff, poly_integral, poly_mul
        P2 = p2_basis(d)
        out = np.zeros((len(P2), len(P2), d + 1))
        for i, j, l in itertools.product(range(len(P2)), range(len(P2)), range(d + 1)):
            out[i, j, l] = float(poly_integral(poly_mul(P2[i], poly_diff(P2[j], l))))
        _PHI_DPHI[d] = out
    return _PHI_DPHI[d]


# ---------------- prolongation (nested meshes) ----------------
def _locate(gf: np.ndarray, R: int, ncoarse: tuple):
    """Fine half-grid points gf (N, d) on a mesh R times finer -> coarse cell (N, d), local coords as
    integer numerators over 2R (N, d)."""
    cell = np.minimum(gf // (2 * R), np.asarray(ncoarse) - 1)
    num = gf - 2 * R * cell
    return cell, num


def prolongation(coarse: M.Grid, fine_g: np.ndarray, R: int, degree: int) -> sp.csr_matrix:
    """Matrix evaluating a coarse P2 (degree 2) or P1 (degree 1) FE function of the whole region
    at fine half-grid points fine_g (N, d).  Exact: T_H and T_h are nested (C22)."""
    d = coarse.d
    cell, num = _locate(np.asarray(fine_g), R, coarse.n)
    xi = num / (2.0 * R)  # local coordinates in [0, 1]
    order = np.argsort(-xi, axis=1, kind="stable")  # pi: x_pi1 >= x_pi2 >= ...
    xs = np.take_along_axis(xi, order, axis=1)
    N = len(xi)
    lam = np.empty((N, d + 1))
    lam[:, 0] = 1.0 - xs[:, 0]
    for k in range(1, d):
        lam[:, k] = xs[:, k - 1] - xs[:, k]
    lam[:, d] = xs[:, d - 1]
    # simplex vertices (coarse vertex index) and P2 nodes
    verts = np.zeros((N, d + 1, d), dtype=np.int64)
    verts[:, 0] = cell
    for k in range(d):
        verts[:, k + 1] = verts[:, k]
        np.add.at(verts[:, k + 1], (np.arange(N), order[:, k]), 1)
    shape2 = np.asarray([2 * k + 1 for k in coarse.n])
    shape1 = np.asarray([k + 1 for k in coarse.n])
    if degree == 2:
        gnodes = [2 * verts[:, k] for k in range(d + 1)] + [verts[:, a] + verts[:, b] for a, b in edges(d)]
        cols = np.stack([M.lex_index(g, np.zeros(d, np.int64), shape2) for g in gnodes], axis=1)
        vals = eval_p2(d, lam)
        ncols = int(np.prod(shape2))
    else:
        cols = np.stack([M.lex_index(verts[:, k], np.zeros(d, np.int64), shape1) for k in range(d + 1)], axis=1)
        vals = lam
        ncols = int(np.prod(shape1))
    rows = np.repeat(np.arange(N)[:, None], cols.shape[1], axis=1)
    P = sp.coo_matrix((vals.ravel(), (rows.ravel(), cols.ravel())), shape=(N, ncols)).tocsr()
    P.eliminate_zeros()
    return P


def exact_prolong_weights(d: int, num: tuple, R: int) -> list[Fraction]:
    """Exact rational P2 weights of one fine point (tests)."""
    xi = [Fraction(v, 2 * R) for v in num]
    order = sorted(range(d), key=lambda a: -xi[a])
    xs = [xi[a] for a in order]
    lam = [1 - xs[0]] + [xs[k - 1] - xs[k] for k in range(1, d)] + [xs[d - 1]]
    from .poly import eval_p2_exact
    return eval_p2_exact(d, lam)
