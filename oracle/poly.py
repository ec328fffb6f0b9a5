"""Exact integration of P2/P1 Lagrange products on a d-simplex (oracle; test infrastructure).

Every form in the weak formulation (eq. CoupledFormu) restricted to
one simplex K is an integral of a product of Lagrange basis functions (and
their gradients) of degree <= 5.  Written in barycentric coordinates
lambda_0..lambda_d, each is a sum of monomials, integrated exactly by the
textbook formula

    int_K  prod_i lambda_i^{a_i} dx = d! |K| prod_i a_i! / (d + sum_i a_i)!

so the discrete problem does not depend on any quadrature rule.
Gradients use the chain rule grad(phi) = sum_k dphi/dlambda_k grad(lambda_k),
valid for any polynomial representation in (lambda_0..lambda_d).

All tensors here are exact rationals divided by |K| (dimensionless); fem.py
multiplies them by |K| and the constant grad(lambda_k) of each element.

Local node order (C23): vertices 0..d, then edge midpoints (a, b), a < b, in
lexicographic pair order.  Internal only.
"""
from __future__ import annotations

import itertools
from fractions import Fraction
from functools import lru_cache
from math import factorial

import numpy as np


def monomial_integral(alpha: tuple[int, ...]) -> Fraction:
    """(1/|K|) int_K prod lambda_i^alpha_i over a d-simplex, d = len(alpha) - 1."""
    d = len(alpha) - 1
    num = factorial(d)
    for a in alpha:
        num *= factorial(a)
    return Fraction(num, factorial(d + sum(alpha)))


# A polynomial in the d+1 barycentric coordinates: {exponent tuple: Fraction}.
Poly = dict


def _unit(d: int, i: int, p: int = 1) -> tuple[int, ...]:
    e = [0] * (d + 1)
    e[i] = p
    return tuple(e)


def poly_mul(p: Poly, q: Poly) -> Poly:
    out: Poly = {}
    for ea, ca in p.items():
        for eb, cb in q.items():
            e = tuple(x + y for x, y in zip(ea, eb))
            out[e] = out.get(e, Fraction(0)) + ca * cb
    return {e: c for e, c in out.items() if c != 0}


def poly_diff(p: Poly, k: int) -> Poly:
    """d/dlambda_k treating all d+1 barycentrics as independent."""
    out: Poly = {}
    for e, c in p.items():
        if e[k] == 0:
            continue
        e2 = list(e)
        e2[k] -= 1
        e2 = tuple(e2)
        out[e2] = out.get(e2, Fraction(0)) + c * e[k]
    return out


def poly_integral(p: Poly) -> Fraction:
    return sum((c * monomial_integral(e) for e, c in p.items()), Fraction(0))


def edges(d: int) -> list[tuple[int, int]]:
    return list(itertools.combinations(range(d + 1), 2))


def p2_basis(d: int) -> list[Poly]:
    """P2 Lagrange basis: vertex i -> lambda_i (2 lambda_i - 1); edge (a,b) -> 4 lambda_a lambda_b."""
    basis = []
    for i in range(d + 1):
        basis.append({_unit(d, i, 2): Fraction(2), _unit(d, i, 1): Fraction(-1)})
    for a, b in edges(d):
        e = [0] * (d + 1)
        e[a] = 1
        e[b] = 1
        basis.append({tuple(e): Fraction(4)})
    return basis


def p1_basis(d: int) -> list[Poly]:
    return [{_unit(d, i, 1): Fraction(1)} for i in range(d + 1)]


def _to_array(nested) -> np.ndarray:
    return np.array(nested, dtype=object)


@lru_cache(maxsize=None)
def tensors(d: int) -> dict[str, np.ndarray]:
    """Exact (Fraction) reference tensors, all divided by |K|.

    mass22[i,j]      = int phi_i phi_j
    grad22[i,k,j,l]  = int dphi_i/dlam_k dphi_j/dlam_l
    div12[m,j,l]     = int psi_m dphi_j/dlam_l            (psi = P1, phi = P2)
    conv[i,m,j,l]    = int phi_i phi_m dphi_j/dlam_l
    mass11[m,n]      = int psi_m psi_n
    mass1[m]         = int psi_m
    """
    P2 = p2_basis(d)
    P1 = p1_basis(d)
    n2, n1, nl = len(P2), len(P1), d + 1
    dP2 = [[poly_diff(phi, k) for k in range(nl)] for phi in P2]
    mass22 = [[poly_integral(poly_mul(P2[i], P2[j])) for j in range(n2)] for i in range(n2)]
    grad22 = [[[[poly_integral(poly_mul(dP2[i][k], dP2[j][l])) for l in range(nl)]
                for j in range(n2)] for k in range(nl)] for i in range(n2)]
    div12 = [[[poly_integral(poly_mul(P1[m], dP2[j][l])) for l in range(nl)]
              for j in range(n2)] for m in range(n1)]
    conv = [[[[poly_integral(poly_mul(poly_mul(P2[i], P2[m]), dP2[j][l])) for l in range(nl)]
              for j in range(n2)] for m in range(n2)] for i in range(n2)]
    mass11 = [[poly_integral(poly_mul(P1[m], P1[n])) for n in range(n1)] for m in range(n1)]
    mass1 = [poly_integral(P1[m]) for m in range(n1)]
    return {
        "mass22": _to_array(mass22),
        "grad22": _to_array(grad22),
        "div12": _to_array(div12),
        "conv": _to_array(conv),
        "mass11": _to_array(mass11),
        "mass1": _to_array(mass1),
    }


@lru_cache(maxsize=None)
def ftensors(d: int) -> dict[str, np.ndarray]:
    """Same tensors as float64 arrays."""
    return {k: v.astype(np.float64) for k, v in tensors(d).items()}


def eval_p2(d: int, lam: np.ndarray) -> np.ndarray:
    """Values of the P2 basis at barycentric points lam (..., d+1) -> (..., n2)."""
    cols = [lam[..., i] * (2.0 * lam[..., i] - 1.0) for i in range(d + 1)]
    cols += [4.0 * lam[..., a] * lam[..., b] for a, b in edges(d)]
    return np.stack(cols, axis=-1)


def eval_p2_exact(d: int, lam: list[Fraction]) -> list[Fraction]:
    vals = [lam[i] * (2 * lam[i] - 1) for i in range(d + 1)]
    vals += [4 * lam[a] * lam[b] for a, b in edges(d)]
    return vals
