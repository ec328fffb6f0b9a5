"""Structured nested Kuhn meshes, subdomain boxes, node classes and ownership (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: T_H and T_h are regular, nested, compatible on Gamma;
Algorithm 3 Step 2 divides each region into disjoint D_j and enlarges them to
Omega_j aligned with T_h (Ex1 layout P:1524-1538).  Readings
(DESIGN.md ledger): C3 ownership, C4/C5 node classes and precedence, C7
overlap = H clipped at the region boundary, C8 grid per region, C21
coordinates, C22 Kuhn/Freudenthal simplices.

Half-grid convention: a region meshed with n_a cells per axis has P2 nodes at
half-grid indices g_a in [0, 2 n_a] (x_a = lo_a + g_a * ((hi_a - lo_a) / (2 n_a)))
and P1 vertices at even g_a.  Numbering is lexicographic, x fastest.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

# node classes, precedence dir > art > gamma > int (C4, C5)
INT, GAMMA, ART, DIR = 0, 1, 2, 3


@dataclass(frozen=True)
class Grid:
    """One region ('p' porous, 'c' conduit) meshed with n[a] cells per axis."""

    region: str
    lo: tuple
    hi: tuple
    n: tuple

    @property
    def d(self) -> int:
        return len(self.n)

    @property
    def gamma_g(self) -> int:
        """Half-grid index of Gamma on the last axis: top of the porous box, bottom of the conduit box."""
        return 2 * self.n[-1] if self.region == "p" else 0

    def coords(self, g: np.ndarray) -> np.ndarray:
        """Physical coordinates of half-grid points g (..., d): x = lo + g * ((hi - lo) / (2 n)) (C21)."""
        g = np.asarray(g)
        out = np.empty(g.shape, dtype=np.float64)
        for a in range(self.d):
            step = (self.hi[a] - self.lo[a]) / (2 * self.n[a])
            out[..., a] = self.lo[a] + g[..., a] * step
        return out

    def n_p2(self) -> int:
        return int(np.prod([2 * k + 1 for k in self.n]))

    def n_p1(self) -> int:
        return int(np.prod([k + 1 for k in self.n]))

    def classify(self, g: np.ndarray, c0=None, c1=None) -> np.ndarray:
        """Node class of half-grid points g (..., d) in the box [c0, c1) (cells), precedence dir > art > Gamma > int.

        dir   = closure of the physical Dirichlet boundary dR \\ Gamma (C5);
        art   = remaining points on the closure of the artificial faces dOmega_j \\ dR (C4);
        Gamma = remaining points on Gamma;  int = the rest.
        """
        g = np.asarray(g)
        d = self.d
        cls = np.full(g.shape[:-1], INT, dtype=np.int64)
        on_gamma = g[..., d - 1] == self.gamma_g
        cls[on_gamma] = GAMMA
        if c0 is not None:
            art = np.zeros(g.shape[:-1], dtype=bool)
            for a in range(d):
                if c0[a] > 0:
                    art |= g[..., a] == 2 * c0[a]
                if c1[a] < self.n[a]:
                    art |= g[..., a] == 2 * c1[a]
            cls[art] = ART
        dirm = np.zeros(g.shape[:-1], dtype=bool)
        for a in range(d - 1):
            dirm |= (g[..., a] == 0) | (g[..., a] == 2 * self.n[a])
        far = 0 if self.region == "p" else 2 * self.n[-1]
        dirm |= g[..., d - 1] == far
        cls[dirm] = DIR
        return cls


def kuhn_permutations(d: int) -> list[tuple[int, ...]]:
    """Simplex types of a Kuhn cell, in itertools order (C22)."""
    return list(itertools.permutations(range(d)))


def kuhn_offsets(d: int) -> np.ndarray:
    """(d!, d+1, d) vertex offsets of the Kuhn simplices of the unit cell.

    Simplex pi = {x in cell : x_pi1 >= x_pi2 (>= x_pi3)}; vertices 0, e_pi1, e_pi1 + e_pi2, ... (C22).
    """
    perms = kuhn_permutations(d)
    out = np.zeros((len(perms), d + 1, d), dtype=np.int64)
    for s, pi in enumerate(perms):
        w = np.zeros(d, dtype=np.int64)
        for k in range(d):
            w = w.copy()
            w[pi[k]] += 1
            out[s, k + 1] = w
    return out


def lex_index(g: np.ndarray, lo: np.ndarray, shape: np.ndarray) -> np.ndarray:
    """Lexicographic (x fastest) index of integer points g (..., d) in the box lo + [0, shape)."""
    g = np.asarray(g)
    idx = np.zeros(g.shape[:-1], dtype=np.int64)
    stride = 1
    for a in range(g.shape[-1]):
        idx += (g[..., a] - lo[a]) * stride
        stride *= shape[a]
    return idx


def lex_points(lo, hi) -> np.ndarray:
    """All integer points of the closed box [lo, hi] in lexicographic order, x fastest: (N, d)."""
    axes = [np.arange(lo[a], hi[a] + 1) for a in range(len(lo))]
    mesh = np.meshgrid(*axes[::-1], indexing="ij")
    return np.stack([m.ravel() for m in mesh[::-1]], axis=-1).astype(np.int64)


@dataclass
class Box:
    """Cells [c0, c1) of a Grid, with local P2 (half-grid) and P1 (vertex) numbering."""

    grid: Grid
    c0: tuple
    c1: tuple
    node_g: np.ndarray = field(init=False)
    vert_g: np.ndarray = field(init=False)

    def __post_init__(self):
        c0 = np.asarray(self.c0)
        c1 = np.asarray(self.c1)
        self.node_g = lex_points(2 * c0, 2 * c1)
        self.vert_g = 2 * lex_points(c0, c1)

    @property
    def d(self) -> int:
        return self.grid.d

    @property
    def shape2(self) -> np.ndarray:
        return 2 * (np.asarray(self.c1) - np.asarray(self.c0)) + 1

    @property
    def shape1(self) -> np.ndarray:
        return np.asarray(self.c1) - np.asarray(self.c0) + 1

    def p2_index(self, g: np.ndarray) -> np.ndarray:
        return lex_index(g, 2 * np.asarray(self.c0), self.shape2)

    def p1_index(self, g: np.ndarray) -> np.ndarray:
        return lex_index(np.asarray(g) // 2, np.asarray(self.c0), self.shape1)

    def classes(self, whole_region: bool = False) -> np.ndarray:
        if whole_region:
            return self.grid.classify(self.node_g)
        return self.grid.classify(self.node_g, self.c0, self.c1)

    def on_artificial(self, g: np.ndarray) -> np.ndarray:
        """Points g on the closure of the artificial faces dOmega_j \\ dR, ignoring the class precedence
        (used for the pressure: Q_0^h of P:226 has compact support in Omega_j, reading C4)."""
        g = np.asarray(g)
        out = np.zeros(g.shape[:-1], dtype=bool)
        for a in range(self.d):
            if self.c0[a] > 0:
                out |= g[..., a] == 2 * self.c0[a]
            if self.c1[a] < self.grid.n[a]:
                out |= g[..., a] == 2 * self.c1[a]
        return out

    def cells(self) -> np.ndarray:
        return lex_points(np.asarray(self.c0), np.asarray(self.c1) - 1)

    def simplices(self):
        """Kuhn simplices of the box, cell-major (lexicographic) then permutation order.

        Returns (p2 local indices (E, n2), p1 local indices (E, d+1), vertex half-grid coords (E, d+1, d),
        cell index (E, d)).
        """
        d = self.d
        off = kuhn_offsets(d)  # (S, d+1, d)
        cells = self.cells()  # (Nc, d)
        verts = cells[:, None, None, :] + off[None, :, :, :]  # (Nc, S, d+1, d)
        verts = verts.reshape(-1, d + 1, d)
        gv = 2 * verts
        eds = list(itertools.combinations(range(d + 1), 2))
        ge = np.stack([verts[:, a] + verts[:, b] for a, b in eds], axis=1)
        g2 = np.concatenate([gv, ge], axis=1)
        p2 = self.p2_index(g2)
        p1 = self.p1_index(gv)
        cell_of = np.repeat(cells, off.shape[0], axis=0)
        return p2, p1, gv, cell_of


def region_grids(cfg: dict, which: str) -> tuple[Grid, Grid]:
    """(porous Grid, conduit Grid) at spacing which in {'h', 'H'}."""
    d = cfg["dim"]
    step = cfg[which]
    out = []
    for reg, lo, hi in (("p", cfg["porous_lo"], cfg["porous_hi"]), ("c", cfg["conduit_lo"], cfg["conduit_hi"])):
        n = tuple(int(round((hi[a] - lo[a]) / step)) for a in range(d))
        out.append(Grid(reg, tuple(lo), tuple(hi), n))
    return out[0], out[1]


@dataclass
class Subdomain:
    region: str
    index: tuple  # grid position (x fastest)
    core0: tuple
    core1: tuple
    box: Box

    @property
    def enclosed(self) -> bool:
        """Conduit box whose closure does not meet Gamma (C6)."""
        return self.box.c0[-1] > 0 if self.region == "c" else self.box.c1[-1] < self.box.grid.n[-1]


def subdomains(grid: Grid, m: tuple, overlap_cells: int) -> list[Subdomain]:
    """Algorithm 3 Step 2: cores D_j = equal blocks of cells, Omega_j = D_j enlarged by
    overlap_cells on every side, clipped at the region box (never across Gamma) (C7, C8)."""
    d = grid.d
    core = []
    for a in range(d):
        if grid.n[a] % m[a] != 0:
            raise ValueError("subdomain grid does not divide the fine mesh")
        core.append(grid.n[a] // m[a])
    out = []
    for pos in lex_points(np.zeros(d, dtype=np.int64), np.asarray(m) - 1):
        c0 = tuple(int(pos[a] * core[a]) for a in range(d))
        c1 = tuple(int((pos[a] + 1) * core[a]) for a in range(d))
        e0 = tuple(max(0, c0[a] - overlap_cells) for a in range(d))
        e1 = tuple(min(grid.n[a], c1[a] + overlap_cells) for a in range(d))
        out.append(Subdomain(grid.region, tuple(int(p) for p in pos), c0, c1, Box(grid, e0, e1)))
    return out


def owner(g: np.ndarray, grid: Grid, m: tuple) -> np.ndarray:
    """Owning subdomain (lexicographic index) of half-grid points g: per axis min(g // (2 core), m - 1) (C3)."""
    g = np.asarray(g)
    idx = np.zeros(g.shape[:-1], dtype=np.int64)
    stride = 1
    for a in range(grid.d):
        core = grid.n[a] // m[a]
        o = np.minimum(g[..., a] // (2 * core), m[a] - 1)
        idx += o * stride
        stride *= m[a]
    return idx
