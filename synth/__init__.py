"""Seeded synthetic inputs for the LGDM K/R assembly path (shared by tests, bench, smoke).

This module holds NONE of the method's arithmetic: it only builds structured meshes,
nodal fields and history values from a counter-based generator, so that the oracle
(``oracle/``) and the CUDA path (``paper_2301_06503_b200``) see identical inputs.
Everything is keyed by GLOBAL node / element / Gauss-point ids, so any z-slab (y-slab
for Q4) of a mesh sees exactly the values of the full mesh.

Recipe (BASELINE.json configs 0-4):
  * RNG: SplitMix64 finaliser of ``seed*K1 + stream*K2 + index``; U(0,1) from the top
    53 bits; N(0,1) by Box-Muller from two uniforms of paired streams.
  * seed = 2301065030 + config.
  * material (all configs): E=30000 MPa, nu=0.2, k=10, kappa0=1e-4, alpha=0.99,
    beta=300, c=l^2/2=2 mm^2 (l=2 mm), R=0.05, n(eta)=5, h=h_sigma=E (reading R-h),
    t=1 (1D: area 1 mm^2).
  * kappa_hist per GP = max(kappa0, U(0, 4e-4)).
  * displacement: uniaxial strain eps0=2e-4 along y (2D) / z (3D) plus a Gaussian
    strain band of peak 1e-3 (Delta=8e-4) and std-dev w (5 / 4 elements), integrated
    analytically with erf; config 2 adds a 45-degree band; N(0,(0.1 eps0 h_el)^2) noise
    on every displacement component.
  * ebar (nodal micro-equivalent strain) = nominal strain magnitude
    (eps0 + bands) * (1 + 0.05 z), z ~ N(0,1)  -- the "local strain" of BASELINE.json,
    taken as the nominal principal strain so that no constitutive law is evaluated here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import erf

BAR2, QUAD4, HEX8 = 1, 2, 3
# type -> (dim, nen, ndpn, ngp)
FAM = {1: (1, 2, 2, 2), 2: (2, 4, 3, 4), 3: (3, 8, 4, 8)}

MATERIAL = dict(E=30000.0, nu=0.2, k=10.0, kappa0=1e-4, alpha=0.99, beta=300.0,
                h=30000.0, h_sigma=30000.0, c=2.0, R=0.05, n=5.0, t=1.0)

_K1 = np.uint64(0x9E3779B97F4A7C15)
_K2 = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# RNG streams
S_UX, S_UY, S_UZ, S_EBAR, S_KAPPA, S_JITTER = 0, 2, 4, 6, 8, 10


def _mix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x.copy()
        x ^= x >> np.uint64(30)
        x *= _M1
        x ^= x >> np.uint64(27)
        x *= _M2
        x ^= x >> np.uint64(31)
    return x


def uniform(seed: int, stream: int, idx) -> np.ndarray:
    """Counter-based U[0,1): SplitMix64 finaliser of seed*K1 + stream*K2 + idx."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.uint64(seed) * _K1 + np.uint64(stream) * _K2 + idx
    return (_mix(x) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, stream: int, idx) -> np.ndarray:
    """Counter-based N(0,1) by Box-Muller from streams (stream, stream+1)."""
    u1 = uniform(seed, stream, idx)
    u2 = uniform(seed, stream + 1, idx)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


@dataclass
class Config:
    cid: int
    etype: int
    n: tuple            # elements per axis
    extent: float       # domain edge length (mm)
    name: str
    iterations: int = 1
    band2: bool = False
    seed: int = field(init=False)

    def __post_init__(self):
        self.seed = 2301065030 + self.cid

    @property
    def dim(self):
        return FAM[self.etype][0]

    @property
    def n_elems(self):
        return int(np.prod(self.n))

    @property
    def n_nodes(self):
        return int(np.prod([k + 1 for k in self.n]))

    @property
    def h_el(self):
        return self.extent / self.n[0]


CONFIGS = {
    0: Config(0, BAR2, (100,), 100.0, "bar2_100"),
    1: Config(1, QUAD4, (200, 200), 100.0, "q4_200x200"),
    2: Config(2, QUAD4, (1000, 1000), 100.0, "q4_1000x1000", iterations=10, band2=True),
    3: Config(3, HEX8, (100, 100, 100), 100.0, "hex8_100^3"),
    4: Config(4, HEX8, (200, 200, 200), 100.0, "hex8_200^3", iterations=10),
}


def small_config(etype: int, n: tuple, cid: int = 100, extent: float = None,
                 band2: bool = False) -> Config:
    """A small mesh with the generator of configs 0/1/3 (tests)."""
    ext = extent if extent is not None else (100.0 if etype == BAR2 else 100.0 * n[0] / 200.0)
    return Config(cid, etype, tuple(n), ext, f"small_{etype}_{'x'.join(map(str, n))}",
                  band2=band2)


@dataclass
class Mesh:
    etype: int
    coords: np.ndarray      # [nn, dim] float64
    conn: np.ndarray        # [ne, nen] int64, LOCAL node ids
    node_gid0: int          # global id of local node 0 (local nodes = contiguous global range)
    elem_gid: np.ndarray    # [ne] int64 global element ids
    n_global_nodes: int
    n_global_elems: int
    shape: tuple            # global elements per axis


def structured_mesh(cfg: Config, elem_layers=None) -> Mesh:
    """Structured mesh of cfg (x-fastest lexicographic ids; SURVEY 8c.1 local node order).

    ``elem_layers=(l0, l1)`` restricts to element layers [l0, l1) along the LAST axis
    (y for Q4, z for Hex8, x for the bar) and to the node layers [l0, l1] they touch.
    """
    n = cfg.n
    dim = cfg.dim
    h = cfg.extent / n[0]
    last = n[-1]
    l0, l1 = (0, last) if elem_layers is None else elem_layers
    assert 0 <= l0 < l1 <= last
    if dim == 1:
        gid = np.arange(l0, l1 + 1, dtype=np.int64)
        coords = (gid.astype(np.float64) * h)[:, None]
        e = np.arange(l0, l1, dtype=np.int64)
        conn = np.stack([e - l0, e - l0 + 1], axis=1)
        return Mesh(BAR2, coords, conn, l0, e, n[0] + 1, n[0], n)
    if dim == 2:
        nx, ny = n
        j = np.arange(l0, l1 + 1)
        i = np.arange(nx + 1)
        J, I = np.meshgrid(j, i, indexing="ij")
        coords = np.stack([I.ravel() * h, J.ravel() * h], axis=1).astype(np.float64)
        node_gid0 = l0 * (nx + 1)
        ej = np.arange(l0, l1)
        ei = np.arange(nx)
        EJ, EI = np.meshgrid(ej, ei, indexing="ij")
        EJ, EI = EJ.ravel().astype(np.int64), EI.ravel().astype(np.int64)
        base = EI + (nx + 1) * (EJ - l0)
        conn = np.stack([base, base + 1, base + nx + 2, base + nx + 1], axis=1)
        egid = EI + nx * EJ
        return Mesh(QUAD4, coords, conn, node_gid0, egid, (nx + 1) * (ny + 1), nx * ny, n)
    nx, ny, nz = n
    k = np.arange(l0, l1 + 1)
    j = np.arange(ny + 1)
    i = np.arange(nx + 1)
    K, J, I = np.meshgrid(k, j, i, indexing="ij")
    coords = np.stack([I.ravel() * h, J.ravel() * h, K.ravel() * h], axis=1).astype(np.float64)
    node_gid0 = l0 * (nx + 1) * (ny + 1)
    ek = np.arange(l0, l1)
    ej = np.arange(ny)
    ei = np.arange(nx)
    EK, EJ, EI = np.meshgrid(ek, ej, ei, indexing="ij")
    EK, EJ, EI = (a.ravel().astype(np.int64) for a in (EK, EJ, EI))
    sx, sy = 1, nx + 1
    sz = (nx + 1) * (ny + 1)
    base = EI + sy * EJ + sz * (EK - l0)
    bot = np.stack([base, base + sx, base + sx + sy, base + sy], axis=1)
    conn = np.concatenate([bot, bot + sz], axis=1)
    egid = EI + nx * (EJ + ny * EK)
    return Mesh(HEX8, coords, conn, node_gid0, egid, (nx + 1) * (ny + 1) * (nz + 1),
                nx * ny * nz, n)


def _band_potential(s, w, delta, s0):
    """Phi(s) = Delta w sqrt(pi/2) [erf(s/(sqrt2 w)) - erf(s0/(sqrt2 w))]; Phi' = Delta e^{-s^2/2w^2}."""
    r2w = math.sqrt(2.0) * w
    return delta * w * math.sqrt(math.pi / 2.0) * (erf(s / r2w) - erf(s0 / r2w))


def fields(cfg: Config, mesh: Mesh):
    """Nodal dofs [nn, ndpn] (node-interleaved) and kappa_hist [ne, ngp] for a mesh of cfg."""
    dim, nen, ndpn, ngp = FAM[cfg.etype]
    seed = cfg.seed
    nn = mesh.coords.shape[0]
    gid = np.arange(nn, dtype=np.uint64) + np.uint64(mesh.node_gid0)
    X = mesh.coords
    dofs = np.zeros((nn, ndpn))
    eps0, delta = 2e-4, 1e-3 - 2e-4
    h = cfg.h_el
    if dim == 1:
        x = X[:, 0]
        dofs[:, 0] = 3e-4 * x * (1.0 + 0.1 * normal(seed, S_UX, gid))
        dofs[:, 1] = 3e-4 * (1.0 + 0.05 * normal(seed, S_EBAR, gid))
    else:
        ax = dim - 1                      # loading axis: y (2D) or z (3D)
        w = (5.0 if dim == 2 else 4.0) * h
        jit = uniform(seed, S_JITTER, np.arange(3, dtype=np.uint64))
        c = cfg.extent / 2.0 + (jit[0] - 0.5) * h
        s = X[:, ax] - c
        dofs[:, ax] = eps0 * X[:, ax] + _band_potential(s, w, delta, -c)
        strain_nom = eps0 + delta * np.exp(-s * s / (2.0 * w * w))
        if cfg.band2 and dim == 2:
            xc = cfg.extent / 2.0 + (jit[1] - 0.5) * h
            yc = cfg.extent / 2.0 + (jit[2] - 0.5) * h
            nvec = np.array([-1.0, 1.0]) / math.sqrt(2.0)
            s2 = (X[:, 0] - xc) * nvec[0] + (X[:, 1] - yc) * nvec[1]
            phi2 = _band_potential(s2, w, delta, 0.0)
            dofs[:, 0] += nvec[0] * phi2
            dofs[:, 1] += nvec[1] * phi2
            strain_nom = strain_nom + delta * np.exp(-s2 * s2 / (2.0 * w * w))
        sd = 0.1 * eps0 * h
        for comp, st in zip(range(dim), (S_UX, S_UY, S_UZ)):
            dofs[:, comp] += sd * normal(seed, st, gid)
        dofs[:, dim] = strain_nom * (1.0 + 0.05 * normal(seed, S_EBAR, gid))
    gp = (mesh.elem_gid.astype(np.uint64)[:, None] * np.uint64(ngp) +
          np.arange(ngp, dtype=np.uint64)[None, :])
    kappa = np.maximum(MATERIAL["kappa0"], 4e-4 * uniform(seed, S_KAPPA, gp))
    return dofs, kappa


def distort(mesh: Mesh, amount: float, seed: int = 7) -> np.ndarray:
    """Coordinates with interior nodes moved by up to amount*h (det J stays > 0 for < 0.25)."""
    X = mesh.coords.copy()
    dim = X.shape[1]
    lo, hi = X.min(axis=0), X.max(axis=0)
    h = (hi[0] - lo[0]) / mesh.shape[0]
    interior = np.all((X > lo + 1e-9) & (X < hi - 1e-9), axis=1)
    gid = np.arange(X.shape[0], dtype=np.uint64) + np.uint64(mesh.node_gid0)
    for k in range(dim):
        d = (uniform(seed, 20 + 2 * k, gid) - 0.5) * 2.0 * amount * h
        X[:, k] = np.where(interior, X[:, k] + d, X[:, k])
    return X


def sample_nodes(n_nodes: int, count: int, seed: int) -> np.ndarray:
    """Distinct sampled node ids (sorted) for sampled-row parity at full size."""
    u = uniform(seed, 30, np.arange(count * 2, dtype=np.uint64))
    ids = np.unique((u * n_nodes).astype(np.int64))[:count]
    return np.sort(ids)


# ---------------------------------------------------------------------------------------
# Mixed-order meshes: BAR3 (quadratic u, linear ebar) and QUAD8
# (serendipity u, bilinear ebar).  Local node order: corners first (bar: x-, x+; quad:
# counter-clockwise), then midsides (bar: centre; quad: (0,-1), (1,0), (0,1), (-1,0)).
# Global nodes are the points of the half-spacing lattice that belong to an element
# (QUAD8 has no element-centre node), numbered x-fastest.  The flat dof vector lists, per
# node in id order, its displacement components and then, for corner nodes only, ebar.
# ---------------------------------------------------------------------------------------
BAR3, QUAD8 = 4, 5
# type -> (dim, nenu, nene, ngp)
MFAM = {4: (1, 3, 2, 3), 5: (2, 8, 4, 9)}


@dataclass
class MixedMesh:
    etype: int
    coords: np.ndarray      # [nn, dim]
    conn: np.ndarray        # [ne, nenu]
    corner: np.ndarray      # [nn] bool: node carries ebar
    shape: tuple


def mixed_mesh(etype: int, n: tuple, extent: float = 100.0) -> MixedMesh:
    h = extent / n[0]
    if etype == BAR3:
        ne = n[0]
        coords = (np.arange(2 * ne + 1, dtype=np.float64) * (h / 2.0))[:, None]
        e = np.arange(ne, dtype=np.int64)
        conn = np.stack([2 * e, 2 * e + 2, 2 * e + 1], axis=1)
        corner = np.arange(2 * ne + 1) % 2 == 0
        return MixedMesh(etype, coords, conn, corner, tuple(n))
    nx, ny = n
    I, J = np.meshgrid(np.arange(2 * nx + 1), np.arange(2 * ny + 1), indexing="xy")
    I, J = I.ravel(), J.ravel()                       # x fastest
    keep = ~((I % 2 == 1) & (J % 2 == 1))
    ids = -np.ones(I.size, dtype=np.int64)
    ids[keep] = np.arange(int(keep.sum()))
    lat = lambda i, j: ids[i + (2 * nx + 1) * j]      # noqa: E731
    coords = np.stack([I[keep] * (h / 2.0), J[keep] * (h / 2.0)], axis=1).astype(np.float64)
    corner = (I[keep] % 2 == 0) & (J[keep] % 2 == 0)
    EJ, EI = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    i0, j0 = 2 * EI.ravel(), 2 * EJ.ravel()
    conn = np.stack([lat(i0, j0), lat(i0 + 2, j0), lat(i0 + 2, j0 + 2), lat(i0, j0 + 2),
                     lat(i0 + 1, j0), lat(i0 + 2, j0 + 1), lat(i0 + 1, j0 + 2),
                     lat(i0, j0 + 1)], axis=1).astype(np.int64)
    return MixedMesh(etype, coords, conn, corner, tuple(n))


def mixed_fields(mesh: MixedMesh, cid: int = 200):
    """Flat dof vector (per node: u comps, then ebar for corner nodes) and kappa_hist
    [ne, ngp], drawn with the recipe of ``fields`` for the equal-order family of the same
    dimension (evaluated at the mixed mesh's nodes)."""
    dim, nenu, nene, ngp = MFAM[mesh.etype]
    eq = BAR2 if dim == 1 else QUAD4
    ext = float(mesh.coords[:, 0].max() - mesh.coords[:, 0].min())
    cfg = Config(cid, eq, tuple(mesh.shape), ext, "mixed")
    ne = mesh.conn.shape[0]
    proxy = Mesh(eq, mesh.coords, mesh.conn[:, :nene], 0, np.arange(ne, dtype=np.int64),
                 mesh.coords.shape[0], ne, mesh.shape)
    nodal, _ = fields(cfg, proxy)
    cnt = dim + mesh.corner.astype(np.int64)            # dofs per node
    start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    dofs = np.zeros(int(cnt.sum()))
    for c in range(dim):
        dofs[start + c] = nodal[:, c]
    dofs[start[mesh.corner] + dim] = nodal[mesh.corner, dim]
    gp = (np.arange(ne, dtype=np.uint64)[:, None] * np.uint64(ngp) +
          np.arange(ngp, dtype=np.uint64)[None, :])
    kappa = np.maximum(MATERIAL["kappa0"], 4e-4 * uniform(cfg.seed, S_KAPPA, gp))
    return dofs, kappa


def sen_mesh(etype: int, n: tuple, extent: float = 100.0, notch: float = 0.5) -> MixedMesh:
    """Side-edge-notched plate (SPEC default geometry: a square plate with an edge slit
    at mid-height of length notch * extent from x = 0).  QUAD8 (n = (nx, ny), ny even): the slit
    runs along the element-row boundary y = extent / 2; its nodes (x < notch * extent, the tip
    excluded) are duplicated so that the elements above the slit use the copies (appended at
    the end of the node list).  Pure geometry, no method arithmetic."""
    assert etype == QUAD8 and n[1] % 2 == 0
    mesh = mixed_mesh(etype, n, extent)
    X = mesh.coords
    ymid = extent / 2.0
    xt = notch * extent
    on_slit = (np.abs(X[:, 1] - ymid) < 1e-9) & (X[:, 0] < xt - 1e-9)
    slit_ids = np.nonzero(on_slit)[0]
    new_id = {int(g): X.shape[0] + k for k, g in enumerate(slit_ids)}
    conn = mesh.conn.copy()
    above = X[mesh.conn[:, :4], 1].mean(axis=1) > ymid            # elements above the slit
    for e in np.nonzero(above)[0]:
        for a in range(conn.shape[1]):
            g = int(conn[e, a])
            if g in new_id:
                conn[e, a] = new_id[g]
    coords = np.vstack([X, X[slit_ids]])
    corner = np.concatenate([mesh.corner, mesh.corner[slit_ids]])
    return MixedMesh(etype, coords, conn, corner, tuple(n))

