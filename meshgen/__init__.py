"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module is the ONLY code both sides of the parity check share.  It holds
geometry, random draws and the hierarchy scaffold (the prolongations P_l are
*inputs* of the hot path: "P_1..P_H <- precompute multigrid hierarchy (V,F)",
PAPER.md Alg. 1 line 2).  It holds none of the method's arithmetic:
no Laplacian, no mass matrix, no Galerkin product, no colouring, no
relaxation.  Each side computes those from these arrays on its own.

Recipes follow BASELINE.json `configs` and SURVEY.md §8(d.2) / reading A22:

* RNG per config: ``numpy.random.default_rng(210413755 + config_id)``, drawn in
  the documented order (displacement, then jitter, then the right-hand side).
  Hierarchy scaffolds draw from a separate stream (seed + 7_000_000) so they
  never perturb the documented order.
* Icosphere: icosahedron, midpoint subdivision, projection to the unit sphere
  after every round (A22 i).
* Spherical-harmonic noise: 8 real orthonormal SH terms, l ~ U{1..6},
  m ~ U{-l..l}, coefficients N(0,1), g <- g / max|g|, v <- u (1 + 0.05 g)
  (A22 ii).
* Cylinder: r = 1, h = 4, 1024 x 1024 vertices, tangent jitter U(-0.3,0.3) h,
  boundary rings jittered in theta only, quads split along (i,j)-(i+1,j+1)
  (A22 iii).

Hierarchy scaffold (stand-in for the paper's successive self-parameterisation
builder, which is host precompute and not on the graded path; see DESIGN.md
"Inputs"): every P row holds the barycentric coordinates of a fine vertex in
the coarse triangle containing it (§4.5), so P has <= 3
non-negative entries per row summing to 1, exactly the structure the hot path
consumes.

* config 1: nested midpoint subdivision (BJ config 1): rows ``1`` or ``1/2,1/2``.
* spheres (configs 2, 4, 5): coarse level = randomly rotated icosphere of the
  next-lower subdivision, displaced by the same SH field; P by radial
  projection of each fine vertex onto the coarse surface (a bijection between
  star-shaped surfaces).
* cylinder (config 3): coarse level = a jittered (theta, z) grid of half the
  resolution per direction; P by barycentric location in the (theta, z) chart,
  which is an isometry of the cylinder, i.e. an intrinsic parameterisation.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 210413755
HIER_SEED_OFFSET = 7_000_000

# --------------------------------------------------------------------------
# icosphere


def icosahedron():
    t = (1.0 + math.sqrt(5.0)) / 2.0
    V = np.array(
        [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
         [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
         [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    V /= np.linalg.norm(V, axis=1, keepdims=True)
    F = np.array(
        [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
         [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
         [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
         [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    return V, F


def subdivide(V, F):
    """One round of midpoint subdivision, midpoints projected to the unit sphere.

    Returns (V', F', edges) where ``edges[e] = (a, b)`` (a < b) is the parent
    edge of new vertex ``len(V) + e``.  Old vertices keep their indices.
    """
    n = V.shape[0]
    e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]], axis=0)
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    key = lo * n + hi
    ukey, inv = np.unique(key, return_inverse=True)
    edges = np.stack([ukey // n, ukey % n], axis=1)
    mid = 0.5 * (V[edges[:, 0]] + V[edges[:, 1]])
    mid /= np.linalg.norm(mid, axis=1, keepdims=True)
    m = F.shape[0]
    ab = n + inv[:m]
    bc = n + inv[m:2 * m]
    ca = n + inv[2 * m:]
    a, b, c = F[:, 0], F[:, 1], F[:, 2]
    F2 = np.concatenate([
        np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
        np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], axis=0)
    return np.concatenate([V, mid], axis=0), F2, edges


def icosphere(k):
    """icosahedron midpoint-subdivided k times: 10*4^k + 2 vertices, 20*4^k faces."""
    V, F = icosahedron()
    for _ in range(k):
        V, F, _ = subdivide(V, F)
    return V, F


def icosphere_levels(k, k_min):
    """Nested icospheres k, k-1, ..., k_min with subdivision prolongations.

    Returns list of (V, F) fine->coarse and list of ELL-3 P (cols, w); P_l maps
    level l+1 (coarse) values to level l (fine) values.
    """
    meshes = []
    edges_of = {}
    V, F = icosahedron()
    meshes.append((V, F))
    for s in range(1, k + 1):
        V, F, E = subdivide(V, F)
        meshes.append((V, F))
        edges_of[s] = E
    levels = [meshes[s] for s in range(k, k_min - 1, -1)]
    Ps = []
    for s in range(k, k_min, -1):
        n_c = meshes[s - 1][0].shape[0]
        E = edges_of[s]
        n_f = n_c + E.shape[0]
        cols = np.zeros((n_f, 3), np.int32)
        w = np.zeros((n_f, 3), np.float64)
        cols[:n_c, 0] = np.arange(n_c)
        w[:n_c, 0] = 1.0
        cols[n_c:, 0] = E[:, 0]
        cols[n_c:, 1] = E[:, 1]
        w[n_c:, 0] = 0.5
        w[n_c:, 1] = 0.5
        # padding slots: column 0 with weight exactly 0 (contributes no structure, A9)
        Ps.append((cols, w))
    return levels, Ps


# --------------------------------------------------------------------------
# spherical-harmonic displacement (A22 ii)


def _real_sh(l, m, dirs):
    from scipy.special import lpmv
    z = np.clip(dirs[:, 2], -1.0, 1.0)
    phi = np.arctan2(dirs[:, 1], dirs[:, 0])
    am = abs(m)
    norm = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - am) / math.factorial(l + am))
    p = lpmv(am, l, z)
    if m > 0:
        return math.sqrt(2.0) * norm * p * np.cos(am * phi)
    if m < 0:
        return math.sqrt(2.0) * norm * p * np.sin(am * phi)
    return norm * p


@dataclass
class SHField:
    ls: np.ndarray
    ms: np.ndarray
    coef: np.ndarray
    scale: float = 1.0  # 1 / max|g| over the fine vertices

    def raw(self, dirs):
        g = np.zeros(dirs.shape[0])
        for l, m, c in zip(self.ls, self.ms, self.coef):
            g += c * _real_sh(int(l), int(m), dirs)
        return g

    def __call__(self, dirs):
        return self.raw(dirs) * self.scale


def draw_sh_field(rng, n_terms=8, lmax=6):
    ls = rng.integers(1, lmax + 1, size=n_terms)
    ms = np.array([rng.integers(-int(l), int(l) + 1) for l in ls])
    coef = rng.standard_normal(n_terms)
    return SHField(ls, ms, coef)


def displace(dirs, field_, amp=0.05):
    return dirs * (1.0 + amp * field_(dirs))[:, None]


# --------------------------------------------------------------------------
# cylinder (A22 iii)


def cylinder_grid(n_theta, n_z, height, rng=None, jitter=0.3, theta0=0.0):
    """Jittered (theta, z) grid on the unit-radius open cylinder.

    Returns V (n,3), F (m,3), theta (n,), z (n,). Vertex (i, j) has index
    j * n_theta + i, i around, j along the axis.
    """
    h_t = 2 * math.pi / n_theta
    h_z = height / (n_z - 1)
    i = np.tile(np.arange(n_theta), n_z)
    j = np.repeat(np.arange(n_z), n_theta)
    theta = theta0 + i * h_t
    z = j * h_z
    if rng is not None and jitter > 0:
        dt = rng.uniform(-jitter, jitter, size=theta.shape[0])
        dz = rng.uniform(-jitter, jitter, size=theta.shape[0])
        boundary = (j == 0) | (j == n_z - 1)
        dz[boundary] = 0.0
        theta = theta + dt * h_t
        z = z + dz * h_z
    V = np.stack([np.cos(theta), np.sin(theta), z], axis=1)
    ii, jj = np.meshgrid(np.arange(n_theta), np.arange(n_z - 1), indexing="xy")
    ii = ii.ravel()
    jj = jj.ravel()
    v00 = jj * n_theta + ii
    v10 = jj * n_theta + (ii + 1) % n_theta
    v11 = (jj + 1) * n_theta + (ii + 1) % n_theta
    v01 = (jj + 1) * n_theta + ii
    F = np.concatenate([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)], axis=0)
    return V, F, theta, z


# --------------------------------------------------------------------------
# scaffold prolongations


def _pick_best(lam_cands, valid):
    """SPEC decision: among candidate faces pick the one maximising the
    minimum barycentric coordinate; clamp negatives to 0 and renormalise."""
    mins = np.where(valid, lam_cands.min(axis=2), -np.inf)
    best = np.argmax(mins, axis=1)
    return best, mins[np.arange(mins.shape[0]), best]


def radial_prolongation(Vf, Vc, Fc, tol=1e-9):
    """Barycentric coordinates of the ray origin->Vf[i] through the coarse
    triangle it pierces.  Vc, Fc: a star-shaped closed coarse surface."""
    from scipy.spatial import cKDTree
    n_f = Vf.shape[0]
    uf = Vf / np.linalg.norm(Vf, axis=1, keepdims=True)
    uc = Vc / np.linalg.norm(Vc, axis=1, keepdims=True)
    n_c = Vc.shape[0]
    # vertex -> incident faces table
    fv = Fc.ravel()
    order = np.argsort(fv, kind="stable")
    counts = np.bincount(fv, minlength=n_c)
    maxval = counts.max()
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    table = -np.ones((n_c, maxval), np.int64)
    rank = np.arange(fv.shape[0]) - np.repeat(starts, counts)
    table[fv[order], rank] = order // 3
    tree = cKDTree(uc)

    cols = np.zeros((n_f, 3), np.int32)
    w = np.zeros((n_f, 3), np.float64)
    todo = np.arange(n_f)
    for k_nn in (1, 4, 16):
        if todo.size == 0:
            break
        _, nn = tree.query(uf[todo], k=k_nn)
        nn = nn.reshape(todo.size, k_nn)
        cand = table[nn].reshape(todo.size, -1)  # faces
        valid = cand >= 0
        cf = np.where(valid, cand, 0)
        A = Vc[Fc[cf, 0]]
        B = Vc[Fc[cf, 1]]
        C = Vc[Fc[cf, 2]]
        u = uf[todo][:, None, :]
        la = np.einsum("ijk,ijk->ij", u, np.cross(B, C))
        lb = np.einsum("ijk,ijk->ij", A, np.cross(u, C))
        lc = np.einsum("ijk,ijk->ij", A, np.cross(B, u))
        s = la + lb + lc
        valid &= s > 0
        ss = np.where(s > 0, s, 1.0)
        lam = np.stack([la / ss, lb / ss, lc / ss], axis=2)
        best, mn = _pick_best(lam, valid)
        ok = mn >= -tol
        sel = todo[ok]
        lam_b = lam[np.arange(todo.size), best][ok]
        lam_b = np.maximum(lam_b, 0.0)
        lam_b /= lam_b.sum(axis=1, keepdims=True)
        cols[sel] = Fc[cf[np.arange(todo.size), best][ok]]
        w[sel] = lam_b
        todo = todo[~ok]
    if todo.size:
        raise RuntimeError(f"radial_prolongation: {todo.size} fine vertices not located")
    return cols, w


def chart_prolongation(theta_f, z_f, theta_c, z_c, n_theta_c, n_z_c, Fc, tol=1e-9):
    """Barycentric location of fine (theta, z) points in a jittered coarse grid
    triangulation of the cylinder chart (periodic in theta)."""
    n_f = theta_f.shape[0]
    h_t = 2 * math.pi / n_theta_c
    h_z = (z_c.max() - z_c.min()) / (n_z_c - 1)
    ci = np.floor(theta_f / h_t).astype(np.int64)
    cj = np.clip(np.floor(z_f / h_z).astype(np.int64), 0, n_z_c - 2)
    ncell = n_theta_c * (n_z_c - 1)
    best_lam = np.full((n_f, 3), -np.inf)
    best_min = np.full(n_f, -np.inf)
    best_face = np.zeros(n_f, np.int64)
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            ii = (ci + di) % n_theta_c
            jj = cj + dj
            okc = (jj >= 0) & (jj <= n_z_c - 2)
            jj = np.clip(jj, 0, n_z_c - 2)
            cell = jj * n_theta_c + ii
            for half in (0, 1):
                f = cell + half * ncell
                tri = Fc[f]
                tt = theta_c[tri]
                tt = theta_f[:, None] + (np.mod(tt - theta_f[:, None] + math.pi, 2 * math.pi) - math.pi)
                zz = z_c[tri]
                x0, x1, x2 = tt[:, 0], tt[:, 1], tt[:, 2]
                y0, y1, y2 = zz[:, 0], zz[:, 1], zz[:, 2]
                det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)
                l1 = ((theta_f - x0) * (y2 - y0) - (x2 - x0) * (z_f - y0)) / det
                l2 = ((x1 - x0) * (z_f - y0) - (theta_f - x0) * (y1 - y0)) / det
                l0 = 1.0 - l1 - l2
                lam = np.stack([l0, l1, l2], axis=1)
                mn = lam.min(axis=1)
                better = okc & (mn > best_min)
                best_min = np.where(better, mn, best_min)
                best_lam[better] = lam[better]
                best_face = np.where(better, f, best_face)
    if np.any(best_min < -tol):
        raise RuntimeError("chart_prolongation: point outside the coarse chart")
    lam = np.maximum(best_lam, 0.0)
    lam /= lam.sum(axis=1, keepdims=True)
    return Fc[best_face].astype(np.int32), lam


# --------------------------------------------------------------------------
# configs


@dataclass
class Problem:
    """One synthetic workload (BASELINE.json configs[cid-1])."""
    cid: int
    name: str
    levels: list            # [(V_l, F_l)] fine -> coarse
    P: list                 # [(cols int32 [n_l,3], w f64 [n_l,3])], P[l]: level l+1 -> l
    mass_coeff: float       # A = mass_coeff * M + lap_coeff * L
    lap_coeff: float
    k: int
    rhs_kind: str           # "direct": B given; "mass": B = M @ F_rhs; "mcf": B = M_t X_t
    rhs: np.ndarray         # B (direct) or F_rhs (mass)
    rel_tol: float
    max_cycles: int
    steps: int = 1          # config 5: implicit MCF steps
    extra: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.levels[0][0].shape[0]

    @property
    def sizes(self):
        return [V.shape[0] for V, _ in self.levels]


def _random_rotation(rng):
    q, r = np.linalg.qr(rng.standard_normal((3, 3)))
    q = q * np.sign(np.diag(r))[None, :]
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def sphere_scaffold(Vf, Ff, k_fine, field_, rng_h, max_coarse=1000):
    """Coarse levels = rotated icospheres k-1, k-2, ... (displaced by the same
    field) until a level has <= max_coarse vertices; P by radial projection."""
    levels = [(Vf, Ff)]
    Ps = []
    s = k_fine
    Vprev = Vf
    while Vprev.shape[0] > max_coarse:
        s -= 1
        Vu, Fc = icosphere(s)
        R = _random_rotation(rng_h)
        Vu = Vu @ R.T
        Vc = displace(Vu, field_) if field_ is not None else Vu
        Ps.append(radial_prolongation(Vprev, Vc, Fc))
        levels.append((Vc, Fc))
        Vprev = Vc
    return levels, Ps


def _noisy_sphere(k, rng):
    Vu, F = icosphere(k)
    fld = draw_sh_field(rng)
    fld.scale = 1.0 / np.abs(fld.raw(Vu)).max()
    return displace(Vu, fld), F, fld


def mean_edge_length(V, F):
    e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]], axis=0)
    e = np.unique(np.sort(e, axis=1), axis=0)
    return float(np.linalg.norm(V[e[:, 0]] - V[e[:, 1]], axis=1).mean())


def make_config(cid, subdiv=None, grid=None, four_grids=False):
    """Build BASELINE.json config `cid` (1..5). `subdiv` / `grid` shrink the
    mesh for tests (same recipe, smaller resolution)."""
    rng = np.random.default_rng(BASE_SEED + cid)
    rng_h = np.random.default_rng(BASE_SEED + cid + HIER_SEED_OFFSET)
    if cid == 1:
        k = 4 if subdiv is None else subdiv
        kmin = max(k - (3 if four_grids else 2), 0)
        levels, Ps = icosphere_levels(k, kmin)
        n = levels[0][0].shape[0]
        b = rng.uniform(-1.0, 1.0, size=(n, 1))
        return Problem(1, f"icosphere({k}) nested", levels, Ps, 1.0, 1e-3, 1, "direct", b,
                       rel_tol=0.0, max_cycles=10)
    if cid in (2, 4, 5):
        k = {2: 7, 4: 9, 5: 8}[cid] if subdiv is None else subdiv
        V, F, fld = _noisy_sphere(k, rng)
        levels, Ps = sphere_scaffold(V, F, k, fld, rng_h)
        n = V.shape[0]
        if cid == 2:
            t = mean_edge_length(V, F) ** 2
            v = int(rng.integers(0, n))
            d = np.zeros((n, 1))
            d[v, 0] = 1.0
            return Problem(2, f"noisy sphere icosphere({k})", levels, Ps, 1.0, t, 1, "mass", d,
                           rel_tol=1e-10, max_cycles=100, extra={"source_vertex": v, "t": t})
        if cid == 4:
            f = V + rng.normal(0.0, 0.01, size=V.shape)
            return Problem(4, f"data smoothing icosphere({k}) k=3", levels, Ps, 1.0, 1e-4, 3,
                           "mass", f, rel_tol=1e-10, max_cycles=100)
        return Problem(5, f"implicit MCF icosphere({k}) 20 steps", levels, Ps, 1.0, 1e-3, 3,
                       "mcf", V.copy(), rel_tol=1e-8, max_cycles=100, steps=20)
    if cid == 3:
        nt, nz = (1024, 1024) if grid is None else grid
        height = 4.0
        V, F, th, z = cylinder_grid(nt, nz, height, rng=rng)
        levels = [(V, F)]
        Ps = []
        th_f, z_f = th, z
        nt_c, nz_c = nt, nz
        while th_f.shape[0] > 1000:
            nt_c //= 2
            nz_c //= 2
            Vc, Fc, th_c, z_c = cylinder_grid(nt_c, nz_c, height, rng=rng_h)
            Ps.append(chart_prolongation(np.mod(th_f, 2 * math.pi), z_f, np.mod(th_c, 2 * math.pi),
                                         z_c, nt_c, nz_c, Fc))
            levels.append((Vc, Fc))
            th_f, z_f = th_c, z_c
        b = rng.standard_normal((V.shape[0], 1))
        return Problem(3, f"open cylinder {nt}x{nz}", levels, Ps, 1.0, 1e-2, 1, "direct", b,
                       rel_tol=1e-10, max_cycles=100)
    raise ValueError(f"unknown config {cid}")
