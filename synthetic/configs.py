"""Seeded input recipes for the five BASELINE.json configs (and scaled-down
variants of the same recipes for tests).

Conventions:
  * node id  = i + (nx+1)*(j + (ny+1)*k)       (x fastest; k = 0 in 2D)
  * dof id   = dim*node + c                     (component fastest)
  * element  = ex + nx*(ey + ny*ez)             (x fastest), density in that order
  * h = 1 (unit elements), E0 = 1, Emin = 1e-9, p = 3, nu = 0.3
  * y is "up"; a downward load is along -y.

Nothing here computes any part of the method: these are the inputs.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
import numpy as np


@dataclass
class Problem:
    name: str
    dim: int
    nel: tuple            # elements per axis (len == dim)
    sub: tuple            # elements per subdomain per axis (len == dim)
    fixed: np.ndarray     # uint8[ndof], 1 = homogeneous Dirichlet
    density: np.ndarray   # float64[prod(nel)], x fastest
    rhs: np.ndarray       # float64[ndof] nodal loads
    E0: float = 1.0
    Emin: float = 1e-9
    p: float = 3.0
    nu: float = 0.3
    h: float = 1.0
    rtol: float = 1e-10
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def nnodes_axis(self):
        return tuple(n + 1 for n in self.nel)

    @property
    def nnodes(self):
        return int(np.prod(self.nnodes_axis))

    @property
    def ndof(self):
        return self.dim * self.nnodes

    @property
    def nelem(self):
        return int(np.prod(self.nel))

    @property
    def nsub_axis(self):
        return tuple(n // s for n, s in zip(self.nel, self.sub))

    def with_density(self, rho):
        return replace(self, density=np.ascontiguousarray(rho, dtype=np.float64))


def _node(nel, i, j, k=0):
    nnx, nny = nel[0] + 1, nel[1] + 1
    return i + nnx * (j + nny * k)


def _box_mean(a):
    """Mean over the in-bounds 3^d neighbourhood (d = a.ndim)."""
    pad = np.pad(a, 1)
    ones = np.pad(np.ones_like(a), 1)
    s = np.zeros_like(a)
    c = np.zeros_like(a)
    for off in np.ndindex(*([3] * a.ndim)):
        sl = tuple(slice(o, o + n) for o, n in zip(off, a.shape))
        s += pad[sl]
        c += ones[sl]
    return s / c


def _smoothed_uniform(rng, nel):
    shape = tuple(reversed(nel))          # (nz,) ny, nx  -> x fastest when raveled
    raw = rng.uniform(0.01, 1.0, size=shape)
    return np.ascontiguousarray(_box_mean(raw).ravel())


def _clamp_x0(dim, nel):
    nn = tuple(n + 1 for n in nel)
    fixed = np.zeros(dim * int(np.prod(nn)), dtype=np.uint8)
    if dim == 2:
        for j in range(nn[1]):
            nd = _node(nel, 0, j)
            fixed[2 * nd:2 * nd + 2] = 1
    else:
        for k in range(nn[2]):
            for j in range(nn[1]):
                nd = _node(nel, 0, j, k)
                fixed[3 * nd:3 * nd + 3] = 1
    return fixed


def _right_edge_traction(nel, total=-1.0):
    """Consistent nodal loads of a uniform downward traction on x = nx with
    resultant `total` (interior nodes total/ny, the two corners total/(2ny))."""
    nx, ny = nel
    f = np.zeros(2 * (nx + 1) * (ny + 1))
    for j in range(ny + 1):
        w = 0.5 if j in (0, ny) else 1.0
        f[2 * _node(nel, nx, j) + 1] = total * w / ny
    return f


def _c1(nel=(32, 16), sub=(16, 8), seed=1):
    nx, ny = nel
    fixed = _clamp_x0(2, nel)
    rho = np.full(nx * ny, 0.5)
    f = np.zeros(2 * (nx + 1) * (ny + 1))
    f[2 * _node(nel, nx, ny // 2) + 1] = -1.0      # right-edge midpoint, downward
    return dict(fixed=fixed, density=rho, rhs=f)


def _c2(nel=(256, 128), sub=(32, 32), seed=2):
    rng = np.random.default_rng(seed)
    return dict(fixed=_clamp_x0(2, nel), density=_smoothed_uniform(rng, nel),
                rhs=_right_edge_traction(nel))


def _c3(nel=(1024, 512), sub=(32, 32), seed=3, ndisks=None, rmin=None, rmax=None):
    nx, ny = nel
    scale = nx / 1024.0
    ndisks = 160 if ndisks is None else ndisks
    rmin = 8.0 * scale if rmin is None else rmin
    rmax = 40.0 * scale if rmax is None else rmax
    rng = np.random.default_rng(seed)
    cx = rng.uniform(0, nx, size=ndisks)
    cy = rng.uniform(0, ny, size=ndisks)
    rr = rng.uniform(rmin, rmax, size=ndisks)
    ex = np.arange(nx) + 0.5
    ey = np.arange(ny) + 0.5
    X, Y = np.meshgrid(ex, ey)              # shape (ny, nx)
    solid = np.zeros((ny, nx), dtype=bool)
    for a, b, r in zip(cx, cy, rr):
        solid |= (X - a) ** 2 + (Y - b) ** 2 <= r * r
    rho = np.where(solid, 1.0, 1e-3).ravel()
    nn = 2 * (nx + 1) * (ny + 1)
    fixed = np.zeros(nn, dtype=np.uint8)
    for j in range(ny + 1):                      # symmetry rollers: u_x = 0 on x = 0
        fixed[2 * _node(nel, 0, j)] = 1
    fixed[2 * _node(nel, nx, 0) + 1] = 1         # roller at bottom-right: u_y = 0
    f = np.zeros(nn)
    f[2 * _node(nel, 0, ny) + 1] = -1.0          # unit load at top-left, downward
    return dict(fixed=fixed, density=np.ascontiguousarray(rho), rhs=f)


def _c4(nel=(96, 48, 48), sub=(12, 12, 12), seed=4):
    nx, ny, nz = nel
    rng = np.random.default_rng(seed)
    fixed = _clamp_x0(3, nel)
    f = np.zeros(3 * (nx + 1) * (ny + 1) * (nz + 1))
    for k in range(nz + 1):                      # line x = nx, y = 0, all z; resultant -1
        w = 0.5 if k in (0, nz) else 1.0
        f[3 * _node(nel, nx, 0, k) + 1] = -w / nz
    return dict(fixed=fixed, density=_smoothed_uniform(rng, nel), rhs=f)


def _c5(nel=(2048, 1024), sub=(32, 32), seed=5):
    return _c2(nel=nel, sub=sub, seed=seed)


_RECIPES = {
    "c1": (_c1, 2, (32, 16), (16, 8), 1),
    "c2": (_c2, 2, (256, 128), (32, 32), 2),
    "c3": (_c3, 2, (1024, 512), (32, 32), 3),
    "c4": (_c4, 3, (96, 48, 48), (12, 12, 12), 4),
    "c5": (_c5, 2, (2048, 1024), (32, 32), 5),
}


def config_names():
    return list(_RECIPES)


def make_config(name: str, nel=None, sub=None, seed=None, **kw) -> Problem:
    """Build config `name` (c1..c5).  `nel`/`sub`/`seed` override the BASELINE
    sizes to obtain scaled-down instances of the same recipe for tests."""
    fn, dim, nel0, sub0, seed0 = _RECIPES[name]
    nel = tuple(nel0 if nel is None else nel)
    sub = tuple(sub0 if sub is None else sub)
    seed = seed0 if seed is None else seed
    if len(nel) != dim or len(sub) != dim:
        raise ValueError("nel/sub must have length dim")
    d = fn(nel=nel, sub=sub, seed=seed, **kw)
    tag = name if (nel == nel0 and sub == sub0 and seed == seed0) else \
        f"{name}[{'x'.join(map(str, nel))}/{'x'.join(map(str, sub))}/s{seed}]"
    return Problem(name=tag, dim=dim, nel=nel, sub=sub, seed=seed, **d)


def paper_problem(inv_h: int, nsub: int) -> Problem:
    """The paper's test problem (Table 1 at PAPER.md:201-232):
    cantilever on Omega = (0,2) x (0,1), Q1 squares of edge h = 1/inv_h, clamped on x = 2 (all components),
    body force f = 0.75 downward, traction g = 1 on the free end x = 0 along its outward normal (-x)
    (reading R18: the text says "outward traction"; its extent is not stated), uniform material E = 1,
    nu = 0.3 (VTS with rho = 1: p = 1, Emin = 0), N = nsub subdomains as a sqrt(N) x sqrt(N) grid (R18),
    rtol 1e-6 (the paper's GMRES tolerance). Consistent nodal loads: body force f h^2/4 per element node,
    traction g h/2 per edge node."""
    q = int(round(nsub ** 0.5))
    if q * q != nsub:
        raise ValueError("nsub must be a perfect square")
    nel = (2 * inv_h, inv_h)
    nx, ny = nel
    if nx % q or ny % q:
        raise ValueError("sqrt(nsub) must divide the mesh")
    h = 1.0 / inv_h
    nn = 2 * (nx + 1) * (ny + 1)
    fixed = np.zeros(nn, dtype=np.uint8)
    for j in range(ny + 1):
        nd = _node(nel, nx, j)
        fixed[2 * nd:2 * nd + 2] = 1
    f = np.zeros(nn)
    cnt = np.zeros((ny + 1, nx + 1))          # elements touching each node
    cnt[:-1, :-1] += 1
    cnt[1:, :-1] += 1
    cnt[:-1, 1:] += 1
    cnt[1:, 1:] += 1
    f[1::2] = -0.75 * h * h / 4.0 * cnt.ravel()
    for j in range(ny + 1):
        w = 0.5 if j in (0, ny) else 1.0
        f[2 * _node(nel, 0, j)] += -1.0 * h * w
    return Problem(name=f"paper[h=1/{inv_h},N={nsub}]", dim=2, nel=nel, sub=(nx // q, ny // q), fixed=fixed,
                   density=np.ones(nx * ny), rhs=f, E0=1.0, Emin=0.0, p=1.0, nu=0.3, h=h, rtol=1e-6,
                   meta=dict(inv_h=inv_h, nsub=nsub))


def density_sequence_step(rho: np.ndarray, t: int, base_seed: int = 5000) -> np.ndarray:
    """Config-5 density evolution: rho <- clip(rho*(1+0.05*U[-1,1]), 1e-3, 1)
    with U drawn from default_rng(base_seed + t)."""
    rng = np.random.default_rng(base_seed + t)
    u = rng.uniform(-1.0, 1.0, size=rho.shape)
    return np.clip(rho * (1.0 + 0.05 * u), 1e-3, 1.0)
