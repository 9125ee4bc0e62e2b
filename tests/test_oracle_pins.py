"""Pins of the CPU oracle against what the paper and mathematics fix
(SURVEY.md §8(c.3)).  No GPU.  Each test names the property it pins and the
passage it comes from; none re-types the oracle's own formula.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import meshgen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _csr_from_dense(O, D):
    return O.Csr.from_scipy(sp.csr_matrix(np.asarray(D, dtype=np.float64)))


def _graph(O, n, edges):
    """Structural pattern with a unit diagonal and the given undirected edges."""
    rows = list(range(n)) + [a for a, b in edges] + [b for a, b in edges]
    cols = list(range(n)) + [b for a, b in edges] + [a for a, b in edges]
    S = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))
    return O.Csr.from_scipy(S)


# --------------------------------------------------------------------- a1 cotan / mass


def test_cotan_equilateral_worked_example(ora):
    g = GOLD["cotan_equilateral"]
    L = ora.cotan_laplacian(np.array(g["V"]), np.array(g["F"])).to_scipy().toarray()
    off = L[~np.eye(3, dtype=bool)]
    assert np.allclose(off, g["offdiag"], rtol=0, atol=1e-15)
    assert np.allclose(np.diag(L), g["diag"], rtol=0, atol=1e-15)


def test_cotan_unit_square_worked_example(ora):
    g = GOLD["cotan_unit_square"]
    L = ora.cotan_laplacian(np.array(g["V"]), np.array(g["F"])).to_scipy()
    i, j = g["diag_edge"]
    assert abs(L[i, j] - g["diag_edge_weight"]) < 1e-15
    assert L[i, j] == L[j, i]
    i, j = g["side_edge"]
    assert abs(L[i, j] - g["side_edge_weight"]) < 1e-15


def _fem_stiffness(V, F):
    """Independent textbook FEM stiffness  K_ij = sum_f area_f grad(phi_i).grad(phi_j)
    with hat-function gradients grad(phi_a) = (n x e_a) / (2 area), e_a the edge
    opposite corner a (not the cotangent formula)."""
    n = V.shape[0]
    rows, cols, vals = [], [], []
    for f in F:
        p = V[f]
        nrm = np.cross(p[1] - p[0], p[2] - p[0])
        area2 = np.linalg.norm(nrm)
        nhat = nrm / area2
        grads = []
        for a in range(3):
            e = p[(a + 2) % 3] - p[(a + 1) % 3]
            grads.append(np.cross(nhat, e) / area2)
        for a in range(3):
            for b in range(3):
                rows.append(f[a])
                cols.append(f[b])
                vals.append(0.5 * area2 * grads[a] @ grads[b])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n)).toarray()


@pytest.mark.parametrize("cid,kw", [(1, {"subdiv": 2}), (2, {"subdiv": 2}), (3, {"grid": (12, 9)})])
def test_cotan_equals_fem_stiffness(ora, cid, kw):
    V, F = meshgen.make_config(cid, **kw).levels[0]
    L = ora.cotan_laplacian(V, F).to_scipy().toarray()
    K = _fem_stiffness(V, F)
    assert np.abs(L - K).max() <= 1e-13 * np.abs(K).max()


@pytest.mark.parametrize("cid,kw", [(2, {"subdiv": 3}), (3, {"grid": (16, 12)})])
def test_cotan_invariants(ora, cid, kw):
    V, F = meshgen.make_config(cid, **kw).levels[0]
    L = ora.cotan_laplacian(V, F).to_scipy()
    D = L.toarray()
    assert np.abs(L @ np.ones(V.shape[0])).max() <= 1e-14 * np.abs(D).max()  # L 1 = 0
    assert np.array_equal(D, D.T)                                           # symmetric
    assert np.linalg.eigvalsh(D).min() >= -1e-10                            # PSD
    # 1-ring pattern: off-diagonals exactly the mesh edges
    e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])
    E = set(map(tuple, np.sort(e, axis=1).tolist()))
    Lc = sp.triu(L, 1).tocoo()
    assert set(zip(Lc.row.tolist(), Lc.col.tolist())) == E


def test_cotan_sphere_closed_form(ora):
    """-Delta_S x = 2x on the unit sphere: L X ~ 2 M X, M^-1-weighted error
    shrinking with h (lumped mass converges weakly, not pointwise)."""
    errs = []
    for k in (3, 4, 5):
        V, F = meshgen.icosphere(k)
        L = ora.cotan_laplacian(V, F).to_scipy()
        M = ora.lumped_mass(V, F)
        r = L @ V - 2 * M[:, None] * V
        errs.append(np.sqrt((r ** 2 / M[:, None]).sum()))
    assert errs[0] < 0.2
    assert errs[1] < errs[0] / 1.8 and errs[2] < errs[1] / 1.8


@pytest.mark.parametrize("cid,kw", [(2, {"subdiv": 4}), (3, {"grid": (30, 20)})])
def test_cotan_area_gradient_identity(ora, cid, kw):
    """L V is the gradient of the total area (the cotan formula's origin) and
    area is homogeneous of degree 2 in V, so sum_d V_d^T L V_d = 2 * area
    exactly, on any mesh, with or without boundary (Euler's theorem)."""
    V, F = meshgen.make_config(cid, **kw).levels[0]
    L = ora.cotan_laplacian(V, F).to_scipy()
    area = 0.5 * np.linalg.norm(np.cross(V[F[:, 1]] - V[F[:, 0]], V[F[:, 2]] - V[F[:, 0]]), axis=1).sum()
    assert abs((V * (L @ V)).sum() - 2 * area) <= 1e-12 * area


def test_mass_worked_example_and_trace(ora):
    g = GOLD["mass_area3"]
    M = ora.lumped_mass(np.array(g["V"]), np.array(g["F"]))
    assert np.allclose(M, g["M"], rtol=0, atol=1e-15)
    V, F = meshgen.make_config(3, grid=(20, 10)).levels[0]
    M = ora.lumped_mass(V, F)
    a = np.linalg.norm(V[F[:, 1]] - V[F[:, 0]], axis=1)
    b = np.linalg.norm(V[F[:, 2]] - V[F[:, 1]], axis=1)
    c = np.linalg.norm(V[F[:, 0]] - V[F[:, 2]], axis=1)
    s = (a + b + c) / 2
    heron = np.sqrt(s * (s - a) * (s - b) * (s - c)).sum()
    assert abs(M.sum() - heron) <= 1e-12 * heron
    assert (M > 0).all()
    V, F = meshgen.icosphere(6)
    assert abs(ora.lumped_mass(V, F).sum() - 4 * math.pi) < 4 * math.pi * 1e-3


# --------------------------------------------------------------------- P (input structure)


@pytest.mark.parametrize("cid,kw", [(1, {}), (2, {"subdiv": 5}), (3, {"grid": (64, 64)})])
def test_prolongation_structure(ora, cid, kw):
    p = meshgen.make_config(cid, **kw)
    for l, (c, w) in enumerate(p.P):
        P = ora.prolongation(p.sizes[l + 1], c, w).to_scipy()
        assert P.shape == (p.sizes[l], p.sizes[l + 1])
        assert (P.data > 0).all() and (P.data <= 1).all()
        assert np.abs(P @ np.ones(P.shape[1]) - 1).max() <= 1e-12     # partition of unity
        assert np.diff(P.indptr).max() <= 3


# --------------------------------------------------------------------- a2/a3 Galerkin


def test_galerkin_identity_cases(ora):
    rng = np.random.default_rng(0)
    n = 30
    B = rng.standard_normal((n, n))
    A = B @ B.T + n * np.eye(n)
    A[np.abs(A) < 2.0] = 0.0
    A = (A + A.T) / 2
    Ao = _csr_from_dense(ora, A)
    I = _csr_from_dense(ora, np.eye(n))
    assert np.array_equal(ora.galerkin(I, Ao).to_scipy().toarray(), A)     # P = I -> A
    P = np.zeros((n, 12))
    for i in range(n):
        cols = rng.choice(12, 3, replace=False)
        w = rng.dirichlet(np.ones(3))
        P[i, cols] = w
    Po = _csr_from_dense(ora, P)
    assert np.allclose(ora.galerkin(Po, I).to_scipy().toarray(), P.T @ P, atol=1e-15)   # A = I -> P^T P


@pytest.mark.parametrize("cid,kw", [(1, {}), (2, {"subdiv": 4}), (3, {"grid": (40, 30)})])
def test_galerkin_dense_and_invariants(ora, cid, kw):
    p = meshgen.make_config(cid, **kw)
    V, F = p.levels[0]
    L = ora.cotan_laplacian(V, F)
    M = ora.lumped_mass(V, F)
    A = ora.mass_plus_laplacian(L, M, p.mass_coeff, p.lap_coeff)
    c, w = p.P[0]
    P = ora.prolongation(p.sizes[1], c, w)
    Ac = ora.galerkin(P, A).to_scipy()
    Pd = P.to_scipy().toarray()
    dense = Pd.T @ A.to_scipy().toarray() @ Pd
    scale = np.abs(dense).max()
    assert np.abs(Ac.toarray() - dense).max() <= 1e-13 * scale                 # numpy dense P^T A P
    D = Ac.toarray()
    assert np.abs(D - D.T).max() <= 1e-13 * scale                              # reading A10
    np.linalg.cholesky(D)                                                       # SPD
    Lc = ora.galerkin(P, L).to_scipy()
    assert np.abs(Lc @ np.ones(Lc.shape[0])).max() <= 1e-13 * np.abs(Lc.data).max()   # (P^T L P) 1 = 0
    ones = np.ones(Ac.shape[0])
    assert abs(ones @ Ac @ ones - M.sum() * p.mass_coeff) <= 1e-12 * M.sum()   # 1^T A_c 1 = area
    # linearity  P^T (a L + b M) P = a P^T L P + b P^T M P  (App. D)
    Mo = _csr_from_dense(ora, np.diag(M))
    Mc = ora.galerkin(P, Mo).to_scipy()
    lin = p.lap_coeff * Lc + p.mass_coeff * Mc
    assert abs(lin - Ac).max() <= 1e-13 * scale


def test_galerkin_nested_pattern_is_coarse_one_ring(ora):
    """Nested subdivision P (rows 1 or 1/2,1/2): P^T A P has exactly the coarse
    1-ring pattern (reading A9: zero weights carry no structure)."""
    p = meshgen.make_config(1)
    V, F = p.levels[0]
    A, _ = ora.assemble(V, F, 1.0, 1e-3)
    for l in range(len(p.P)):
        c, w = p.P[l]
        Ac = ora.galerkin(ora.prolongation(p.sizes[l + 1], c, w), A)
        Vc, Fc = p.levels[l + 1]
        S = Ac.to_scipy()
        e = np.concatenate([Fc[:, [0, 1]], Fc[:, [1, 2]], Fc[:, [2, 0]]])
        E = set(map(tuple, np.sort(e, axis=1).tolist()))
        St = sp.triu(S, 1).tocoo()
        assert set(zip(St.row.tolist(), St.col.tolist())) == E
        assert (S.diagonal() != 0).all()
        assert S.nnz == Vc.shape[0] + 2 * len(E)
        A = Ac
    assert [4482, 1122] == [ora.MG(p.sizes, p.P, ora.assemble(V, F, 1, 1e-3)[0]).level(l)["nnz"] for l in (1, 2)]


# --------------------------------------------------------------------- colouring (Alg. 3)


def test_colouring_hand_traces(ora):
    for case in GOLD["colouring"]["cases"]:
        col, k = ora.greedy_colouring(_graph(ora, case["n"], case["edges"]))
        assert col.tolist() == case["colour"], case["name"]
        assert k == max(case["colour"]) + 1


def test_colouring_proper_random_patterns(ora):
    rng = np.random.default_rng(1)
    for t in range(1000):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(0, 3 * n))
        edges = [tuple(e) for e in rng.integers(0, n, size=(m, 2)) if e[0] != e[1]]
        G = _graph(ora, n, edges)
        col, k = ora.greedy_colouring(G)
        for a, b in edges:
            assert col[a] != col[b]
        deg = np.diff(G.to_scipy().indptr) - 1
        assert k <= (deg.max() if n else 0) + 1
        assert set(col.tolist()) == set(range(k))


def test_colouring_mesh_levels(ora):
    """Fine icosphere: 6 colours, cylinder grid: 4 colours (scratch counts)."""
    V, F = meshgen.icosphere(4)
    assert ora.greedy_colouring(ora.cotan_laplacian(V, F))[1] == 6
    V, F = meshgen.make_config(3, grid=(64, 64)).levels[0]
    assert ora.greedy_colouring(ora.cotan_laplacian(V, F))[1] == 4


# --------------------------------------------------------------------- Cholesky


def test_cholesky_worked_examples(ora):
    for key in ("chol_2I", "chol_2x2"):
        g = GOLD[key]
        L = ora.cholesky(np.array(g["A"]))
        x = ora.cholesky_solve(L, np.array(g["b"]))
        assert np.allclose(x, g["x"], rtol=0, atol=1e-15)
        if "L" in g:
            assert np.allclose(np.tril(L), g["L"], rtol=0, atol=1e-15)


def test_cholesky_random_spd_vs_numpy(ora):
    rng = np.random.default_rng(2)
    B = rng.standard_normal((100, 100))
    A = B @ B.T + 100 * np.eye(100)
    L = ora.cholesky(A)
    assert np.abs(np.tril(L) - np.linalg.cholesky(A)).max() <= 1e-13 * np.abs(L).max()
    b = rng.standard_normal(100)
    x = ora.cholesky_solve(L, b)
    assert np.linalg.norm(A @ x - b) <= 1e-12 * np.linalg.norm(b)
    with pytest.raises(np.linalg.LinAlgError):
        ora.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))


# --------------------------------------------------------------------- GS smoother


def test_gs_worked_examples(ora):
    g = GOLD["gs_2x2"]
    A = _csr_from_dense(ora, g["A"])
    col, k = ora.greedy_colouring(A)
    x = np.zeros(2)
    ora.gs_sweep(A, col, k, np.array(g["b"]), x)
    assert np.allclose(x, g["x"], rtol=0, atol=1e-15)
    D = np.diag([2.0, 4.0, 5.0])
    A = _csr_from_dense(ora, D)
    col, k = ora.greedy_colouring(A)
    x = np.zeros(3)
    ora.gs_sweep(A, col, k, np.array([2.0, 2.0, 10.0]), x)
    assert np.array_equal(x, [1.0, 0.5, 2.0])


def _gs_matrix_form(A, colour, b, x):
    """Textbook splitting form of one forward GS sweep in the colour-grouped
    order pi: with B = A[pi][:, pi] = D + Lo + U, x_pi <- (D + Lo)^{-1} (b_pi - U x_pi)."""
    import scipy.linalg as sla
    pi = np.lexsort((np.arange(len(colour)), colour))
    B = A[np.ix_(pi, pi)]
    lower = np.tril(B)
    upper = np.triu(B, 1)
    xp = sla.solve_triangular(lower, b[pi] - upper @ x[pi], lower=True)
    out = np.empty_like(x)
    out[pi] = xp
    return out


def test_gs_equals_splitting_form_and_decreases_energy_error(ora):
    p = meshgen.make_config(2, subdiv=3)
    V, F = p.levels[0]
    A, _ = ora.assemble(V, F, 1.0, 0.05)
    D = A.to_scipy().toarray()
    col, k = ora.greedy_colouring(A)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(D.shape[0])
    x = rng.standard_normal(D.shape[0])
    ref = _gs_matrix_form(D, col, b, x)
    y = x.copy()
    ora.gs_sweep(A, col, k, b, y)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    # theorem: a GS sweep strictly decreases the A-norm error on SPD matrices
    for t in range(100):
        n = 12
        Bm = rng.standard_normal((n, n))
        S = Bm @ Bm.T + 0.5 * np.eye(n)
        S[np.abs(S) < 0.8] = 0.0
        S = (S + S.T) / 2 + n * np.eye(n) * (np.linalg.eigvalsh((S + S.T) / 2).min() < 0.1)
        So = _csr_from_dense(ora, S)
        c, kc = ora.greedy_colouring(So)
        xs = np.linalg.solve(S, b[:n])
        x0 = rng.standard_normal(n)
        e0 = (x0 - xs) @ S @ (x0 - xs)
        x1 = x0.copy()
        ora.gs_sweep(So, c, kc, b[:n], x1)
        e1 = (x1 - xs) @ S @ (x1 - xs)
        assert e1 < e0


# --------------------------------------------------------------------- V-cycle


def _level_mats(ora, mg):
    mats = []
    for l in range(mg.n_levels):
        d = mg.level(l)
        mats.append((sp.csr_matrix((d["val"], d["col"], d["rowptr"]), shape=(d["n"], d["n"])).toarray(),
                     d["colour"]))
    return mats


def test_two_grid_error_propagator(ora):
    """Two-grid (H = 1) V-cycle equals the textbook operator
    E = S^mu2 (I - P A_c^{-1} P^T A) S^mu1 with S the colour-ordered GS error
    propagator (Alg. 2; pins readings A1 and A2)."""
    levels, Ps = meshgen.icosphere_levels(2, 1)
    V, F = levels[0]
    # perturb the fine vertex positions so A is not too regular
    A, _ = ora.assemble(V, F, 1.0, 0.3)
    sizes = [levels[0][0].shape[0], levels[1][0].shape[0]]
    mg = ora.MG(sizes, Ps, A, 2, 2)
    (Af, colf), (Ac, _) = _level_mats(ora, mg)
    n = Af.shape[0]
    Pd = ora.prolongation(sizes[1], *Ps[0]).to_scipy().toarray()
    pi = np.lexsort((np.arange(n), colf))
    Bp = Af[np.ix_(pi, pi)]
    Sp = np.eye(n) - np.linalg.solve(np.tril(Bp), Bp)
    S = np.empty_like(Sp)
    S[np.ix_(pi, pi)] = Sp
    CGC = np.eye(n) - Pd @ np.linalg.solve(Ac, Pd.T @ Af)
    E = S @ S @ CGC @ S @ S
    rng = np.random.default_rng(4)
    xs = rng.standard_normal(n)
    b = Af @ xs
    x0 = rng.standard_normal(n)
    x1 = x0.copy()
    mg.vcycle(b, x1)
    assert np.abs((x1 - xs) - E @ (x0 - xs)).max() <= 1e-13 * np.abs(x0 - xs).max()


def test_vcycle_special_cases(ora):
    p = meshgen.make_config(1, subdiv=2)
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, 1.0, 1e-2)
    n = V.shape[0]
    D = A.to_scipy().toarray()
    rng = np.random.default_rng(5)
    b = rng.standard_normal(n)
    xs = np.linalg.solve(D, b)
    # H = 0: one level -> direct solve (Alg. 2 else-branch)
    mg0 = ora.MG([n], [], A)
    x = rng.standard_normal(n)
    mg0.vcycle(b, x)
    assert np.abs(x - xs).max() <= 1e-12 * np.abs(xs).max()
    # mu = 0, H = 1, P = I -> exact
    eye = (np.tile(np.arange(n)[:, None], (1, 3)).astype(np.int32), np.tile([1.0, 0.0, 0.0], (n, 1)))
    mgI = ora.MG([n, n], [eye], A, 0, 0)
    x = rng.standard_normal(n)
    mgI.vcycle(b, x)
    assert np.abs(x - xs).max() <= 1e-12 * np.abs(xs).max()
    # exact solution is a fixed point; affine superposition from zero guess
    mg = ora.MG(p.sizes, p.P, A)
    x = xs.copy()
    mg.vcycle(b, x)
    assert np.abs(x - xs).max() <= 1e-13 * np.abs(xs).max()
    b2 = rng.standard_normal(n)
    x1, x2, x12 = np.zeros(n), np.zeros(n), np.zeros(n)
    mg.vcycle(b, x1)
    mg.vcycle(b2, x2)
    mg.vcycle(b + b2, x12)
    assert np.abs(x12 - x1 - x2).max() <= 1e-13 * np.abs(x12).max()


# --------------------------------------------------------------------- solve loop


def test_solve_special_cases(ora):
    p = meshgen.make_config(1, subdiv=3)
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, 1.0, 1e-3)
    mg = ora.MG([V.shape[0], p.sizes[1], p.sizes[2]], p.P, A)
    n = V.shape[0]
    X, hist, rc = mg.solve(np.zeros((n, 1)), rel_tol=1e-10, max_cycles=5)   # b = 0 -> cycle 0
    assert rc == 0 and hist.shape[0] == 1 and not X.any()
    b = np.random.default_rng(6).standard_normal((n, 1))
    X, hist, rc = mg.solve(b, rel_tol=2.0, max_cycles=5)                     # tol above rho_0
    assert rc == 0 and hist.shape[0] == 1 and hist[0, 0] == 1.0
    X, hist, rc = mg.solve(b, rel_tol=1e-30, max_cycles=3)                   # unreachable tol
    assert rc == 8 and hist.shape[0] == 4
    # b = M 1 -> x = 1 exactly (L 1 = 0)
    X, hist, rc = mg.solve(M[:, None], rel_tol=1e-13, max_cycles=30)
    assert rc == 0 and np.abs(X - 1).max() <= 1e-11


def test_config1_converges_to_dense_solve(ora):
    """BJ: a tiny-mesh solve converges to a dense direct solve to 1e-12; the
    residual decreases monotonically while above the rounding floor (A21)."""
    p = meshgen.make_config(1)
    V, F = p.levels[0]
    A, _ = ora.assemble(V, F, p.mass_coeff, p.lap_coeff)
    mg = ora.MG(p.sizes, p.P, A)
    X, hist, rc = mg.solve(p.rhs, rel_tol=0.0, max_cycles=p.max_cycles)
    assert rc == 0 and hist.shape[0] == 11
    xs = np.linalg.solve(A.to_scipy().toarray(), p.rhs)
    assert np.linalg.norm(X - xs) / np.linalg.norm(xs) <= 1e-12
    Ad = A.to_scipy()
    floor = 32 * 2.0 ** -53 * np.linalg.norm(abs(Ad) @ np.abs(X) + np.abs(p.rhs)) / np.linalg.norm(p.rhs)
    rho = hist[:, 0]
    for c in range(len(rho) - 1):
        if rho[c] > 10 * floor:
            assert rho[c + 1] < rho[c]


def test_energy_error_decreases_per_cycle(ora):
    p = meshgen.make_config(2, subdiv=4)
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, 1.0, 1e-2)
    mg = ora.MG(p.sizes, p.P, A)
    D = A.to_scipy()
    b = np.random.default_rng(7).standard_normal(V.shape[0])
    xs = sp.linalg.spsolve(D.tocsc(), b)
    x = np.zeros_like(b)
    e_prev = xs @ (D @ xs)
    for _ in range(4):
        mg.vcycle(b, x)
        e = (x - xs) @ (D @ (x - xs))
        assert e < e_prev
        e_prev = e


def test_sphere_eigenfunction_closed_form(ora):
    """Unit sphere, b = M Y_l -> x ~ Y_l / (1 + t l(l+1)), error O(h^2)."""
    t = 0.05
    errs = []
    for k in (3, 4, 5):
        levels, Ps = meshgen.icosphere_levels(k, max(k - 2, 1))
        V, F = levels[0]
        A, M = ora.assemble(V, F, 1.0, t)
        mg = ora.MG([m[0].shape[0] for m in levels], Ps, A)
        Y = V[:, 0] * V[:, 1]                      # a degree-2 harmonic (l = 2)
        X, hist, rc = mg.solve((M * Y)[:, None], rel_tol=1e-12, max_cycles=50)
        assert rc == 0
        e = X[:, 0] - Y / (1 + 6 * t)
        errs.append(np.sqrt((M * e * e).sum()))           # L2(M) error, O(h^2)
    assert errs[0] < 2e-3 and errs[1] < errs[0] / 3.5 and errs[2] < errs[1] / 3.5


def test_cylinder_neumann_closed_form(ora):
    """Open cylinder with natural BC: b = M cos(theta), t = 1e-2
    -> x ~ cos(theta) / (1 + t) (cos(theta) is Neumann-compatible)."""
    errs = []
    for g in ((32, 32), (64, 64), (128, 128)):
        p = meshgen.make_config(3, grid=g)          # jittered grid + its hierarchy
        V, F = p.levels[0]
        th = np.arctan2(V[:, 1], V[:, 0])
        A, M = ora.assemble(V, F, 1.0, 1e-2)
        B = (M * np.cos(th))[:, None]
        X, hist, rc = ora.MG(p.sizes, p.P, A).solve(B, rel_tol=1e-12, max_cycles=100)
        assert rc == 0
        xs = sp.linalg.spsolve(A.to_scipy().tocsc(), B[:, 0])
        assert np.abs(X[:, 0] - xs).max() <= 1e-10
        e = xs - np.cos(th) / 1.01
        errs.append(np.sqrt((M * e * e).sum()))
    assert errs[0] < 5e-3 and errs[1] < errs[0] / 2.5 and errs[2] < errs[1] / 2.5


def test_mcf_sphere_radius(ora):
    """Config-5 loop on a round sphere: radius follows r <- r / (1 + 2 dt / r^2)."""
    g = GOLD["mcf_sphere"]
    levels, Ps = meshgen.icosphere_levels(5, 3)
    V, F = levels[0]
    X, cycles = ora.mcf([m[0].shape[0] for m in levels], Ps, V, F, g["dt"], g["steps"], rel_tol=1e-10)
    r = np.linalg.norm(X, axis=1).mean()
    assert abs(r - g["radius"]) < 1e-3
    assert max(cycles) <= 10


# --------------------------------------------------------------------- f4: Jacobi smoother, symmetric V-cycle, MG-PCG


def test_jacobi_worked_example_and_splitting_form(ora):
    g = GOLD["jacobi_2x2"]
    A = _csr_from_dense(ora, g["A"])
    x = np.zeros(2)
    ora.jacobi_sweep(A, np.array(g["b"]), x, g["omega"])
    assert np.allclose(x, g["x1"], rtol=0, atol=1e-15)
    ora.jacobi_sweep(A, np.array(g["b"]), x, g["omega"])
    assert np.allclose(x, g["x2"], rtol=0, atol=1e-15)
    # splitting form x + omega D^{-1}(b - A x) on a random SPD matrix (numpy, independent)
    rng = np.random.default_rng(11)
    Q = rng.standard_normal((9, 9))
    D = Q @ Q.T + 9 * np.eye(9)
    A = _csr_from_dense(ora, D)
    b, x0 = rng.standard_normal((9, 2)), rng.standard_normal((9, 2))
    ref = x0 + 0.7 * (b - D @ x0) / np.diag(D)[:, None]
    y = x0.copy()
    ora.jacobi_sweep(A, b, y, 0.7)
    assert np.abs(y - ref).max() <= 1e-13 * np.abs(ref).max()


def _vcycle_operator(mg, n):
    """Dense matrix of the map b -> V(0, b) (zero initial guess)."""
    Mi = np.empty((n, n))
    for j in range(n):
        e = np.zeros((n, 1))
        e[j, 0] = 1.0
        z = np.zeros((n, 1))
        mg.vcycle(e, z)
        Mi[:, j] = z[:, 0]
    return Mi


def test_symmetric_vcycle_is_spd_preconditioner(ora):
    """Row f4: with the post-relaxation colours reversed (and Jacobi, whose
    sweep is symmetric), the V-cycle map b -> V(0, b) is symmetric positive
    definite, as CG needs; the default ascending post order is not symmetric."""
    p = meshgen.make_config(1, subdiv=3)                  # 642 -> 162 -> 42 (nested)
    V, F = p.levels[0]
    A, _ = ora.assemble(V, F, 1.0, 1e-2)
    n = V.shape[0]
    assert len(p.sizes) == 3
    mg = ora.MG(p.sizes, p.P, A)
    Mi = _vcycle_operator(mg, n)
    asym = np.abs(Mi - Mi.T).max() / np.abs(Mi).max()
    assert asym > 1e-6                                   # A2: not symmetric as a stand-alone solver
    for kind in (0, 1):
        mg.set_smoother(kind, 0.8, symmetric=True)
        Mi = _vcycle_operator(mg, n)
        assert np.abs(Mi - Mi.T).max() <= 1e-12 * np.abs(Mi).max()
        assert np.linalg.eigvalsh(0.5 * (Mi + Mi.T)).min() > 0


def test_pcg_special_cases_and_dense_solve(ora):
    p = meshgen.make_config(2, subdiv=4)
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, 1.0, 1e-2)
    n = V.shape[0]
    D = A.to_scipy().toarray()
    rng = np.random.default_rng(12)
    B = rng.standard_normal((n, 2))
    XS = np.linalg.solve(D, B)
    # one level: M^{-1} = A^{-1} -> PCG converges in one iteration
    X, hist, rc = ora.MG([n], [], A).pcg(B, rel_tol=1e-12, max_iters=5)
    assert rc == 0 and hist.shape[0] == 2
    assert np.linalg.norm(X - XS) / np.linalg.norm(XS) <= 1e-12
    # multigrid preconditioner (GS and Jacobi smoothers): dense solution to 1e-10
    for kind in (0, 1):
        mg = ora.MG(p.sizes, p.P, A).set_smoother(kind, 0.8)
        X, hist, rc = mg.pcg(B, rel_tol=1e-12, max_iters=60)
        assert rc == 0
        for c in range(2):
            assert np.linalg.norm(X[:, c] - XS[:, c]) / np.linalg.norm(XS[:, c]) <= 1e-10
        # the recursive residual ends within the tolerance; and the true residual agrees
        assert (hist[-1] <= 1e-12).all()
        tr = np.linalg.norm(B - D @ X, axis=0) / np.linalg.norm(B, axis=0)
        assert (tr <= 1e-11).all()
    # b = 0 -> converged at iteration 0
    X, hist, rc = ora.MG(p.sizes, p.P, A).pcg(np.zeros((n, 1)), rel_tol=1e-10, max_iters=5)
    assert rc == 0 and hist.shape[0] == 1 and not X.any()


def test_pcg_solved_column_stays_solved(ora):
    """Reading A27: a column whose residual is already zero (b = 0, x0 = 0)
    has nothing left for CG to do; with alpha = beta = 0 it stays exactly 0
    and the other columns follow exactly their single-column CG iterates
    (the columns of CG are independent)."""
    p = meshgen.make_config(2, subdiv=4)
    V, F = p.levels[0]
    A, _ = ora.assemble(V, F, 1.0, 1e-2)
    n = V.shape[0]
    b = np.random.default_rng(14).standard_normal((n, 1))
    mg = ora.MG(p.sizes, p.P, A)
    B3 = np.ascontiguousarray(np.concatenate([b, np.zeros((n, 1)), 3.0 * b], axis=1))
    X3, h3, rc = mg.pcg(B3, rel_tol=0.0, max_iters=4)
    X1, h1, _ = mg.pcg(b, rel_tol=0.0, max_iters=4)
    assert rc == 0 and np.all(np.isfinite(X3)) and not X3[:, 1].any()
    assert np.array_equal(X3[:, 0], X1[:, 0])
    assert np.linalg.norm(X3[:, 2] - 3.0 * X1[:, 0]) <= 1e-13 * np.linalg.norm(3.0 * X1[:, 0])
    assert np.all(h3[:, 1] == 0.0)


def test_pcg_energy_error_decreases(ora):
    """CG theory: the A-norm error decreases monotonically per iteration."""
    p = meshgen.make_config(3, grid=(48, 40))
    V, F = p.levels[0]
    A, _ = ora.assemble(V, F, 1.0, 1e-2)
    D = A.to_scipy().toarray()
    b = np.random.default_rng(13).standard_normal((V.shape[0], 1))
    xs = np.linalg.solve(D, b)
    mg = ora.MG(p.sizes, p.P, A)
    x = np.zeros_like(b)
    prev = float((xs - x).T @ D @ (xs - x))
    for it in range(1, 6):
        X, hist, rc = mg.pcg(b, rel_tol=0.0, max_iters=it)
        e = float((xs - X).T @ D @ (xs - X))
        assert e < prev
        prev = e


def test_jacobi_multigrid_converges(ora):
    """App. E: damped-Jacobi-smoothed V(2,2) still converges (each cycle
    contracts), more slowly than Gauss-Seidel."""
    p = meshgen.make_config(2, subdiv=4)
    V, F = p.levels[0]
    A, _ = ora.assemble(V, F, 1.0, 1e-2)
    b = np.random.default_rng(14).standard_normal((V.shape[0], 1))
    _, hg, _ = ora.MG(p.sizes, p.P, A).solve(b, rel_tol=0.0, max_cycles=6)
    _, hj, _ = ora.MG(p.sizes, p.P, A).set_smoother(1, 0.8).solve(b, rel_tol=0.0, max_cycles=6)
    assert (np.diff(hj[:, 0]) < 0).all()
    assert hj[-1, 0] > hg[-1, 0]


# --------------------------------------------------------------------- f2: Dirichlet reduction (App. B)


def test_dirichlet_no_constraints_is_identity(ora):
    p = meshgen.make_config(2, subdiv=4)
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, 1.0, 1e-2)
    b = np.random.default_rng(21).standard_normal((p.n, 1))
    X1, h1, _ = ora.MG(p.sizes, p.P, A).solve(b, rel_tol=0.0, max_cycles=4)
    X2, h2, _, _ = ora.dirichlet_solve(p.sizes, p.P, A, b, np.zeros((p.n, 1)), [], rel_tol=0.0, max_cycles=4)
    assert np.array_equal(X1, X2) and np.array_equal(h1, h2)


def test_dirichlet_all_known(ora):
    p = meshgen.make_config(1, subdiv=2)
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, 1.0, 1e-2)
    X0 = np.random.default_rng(22).standard_normal((p.n, 2))
    X, hist, rc, mg = ora.dirichlet_solve(p.sizes, p.P, A, np.ones((p.n, 2)), X0, np.arange(p.n))
    assert rc == 0 and hist.shape[0] == 0 and np.array_equal(X, X0) and mg is None


def test_dirichlet_matches_dense_constrained_solve(ora):
    """SPEC S:561 worked example: 10% random constraints; the reduced-system
    multigrid solution equals the dense solve of the constrained system."""
    p = meshgen.make_config(2, subdiv=4)
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, 1.0, 1e-2)
    rng = np.random.default_rng(23)
    known = np.sort(rng.choice(p.n, p.n // 10, replace=False))
    X0 = np.zeros((p.n, 2))
    X0[known] = rng.standard_normal((known.size, 2))
    B = M[:, None] * rng.standard_normal((p.n, 2))
    X, hist, rc, mg = ora.dirichlet_solve(p.sizes, p.P, A, B, X0, known, rel_tol=1e-12, max_cycles=60)
    assert rc == 0
    D = A.to_scipy().toarray()
    u = np.setdiff1d(np.arange(p.n), known)
    xu = np.linalg.solve(D[np.ix_(u, u)], B[u] - D[np.ix_(u, known)] @ X0[known])
    assert np.linalg.norm(X[u] - xu) / np.linalg.norm(xu) <= 1e-10
    assert np.array_equal(X[known], X0[known])
    # the full-system residual vanishes on the unknown rows
    r = B - D @ X
    assert np.abs(r[u]).max() <= 1e-9 * np.abs(B).max()


def test_dirichlet_zero_column_removal(ora):
    """constraining every child of a coarse vertex zeroes its column
    of P_{u:}; it must be removed (with its row of the next prolongation) so
    the reduced coarse operators have no zero rows and stay SPD."""
    p = meshgen.make_config(1, subdiv=3)                 # 642 -> 162 -> 42, nested P
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, 1.0, 1e-2)
    c0, w0 = p.P[0]
    J = 7
    children = np.nonzero(((c0 == J) & (w0 != 0.0)).any(axis=1))[0]
    u, rs, rP, keep = ora.dirichlet_reduce(p.sizes, p.P, children)
    assert rs[1] == p.sizes[1] - 1 and J not in keep[1]
    for l in range(len(rs) - 1):
        c, w = rP[l]
        assert c.shape == (rs[l], 3) and c.max() < rs[l + 1]
        assert np.allclose(w.sum(axis=1), 1.0)                    # dropped columns carried zero weight only
    X0 = np.zeros((p.n, 1))
    X, hist, rc, mg = ora.dirichlet_solve(p.sizes, p.P, A, M[:, None], X0, children, rel_tol=1e-12, max_cycles=60)
    assert rc == 0 and mg.status == 0
    for l in range(mg.n_levels):
        lv = mg.level(l)
        rows = np.repeat(np.arange(lv["n"]), np.diff(lv["rowptr"]))
        diag = lv["val"][lv["col"] == rows]
        assert diag.size == lv["n"] and (diag > 0).all()


# --------------------------------------------------------------------- f3: bilaplacian L M^-1 L


def test_bilaplacian_invariants_and_pattern(ora):
    """Q 1 = 0, symmetric PSD, pattern = the 2-ring."""
    p = meshgen.make_config(2, subdiv=3)
    V, F = p.levels[0]
    Q, M = ora.bilaplacian(V, F)
    Qs = Q.to_scipy()
    n = V.shape[0]
    assert np.abs(Qs @ np.ones(n)).max() <= 1e-10 * abs(Qs).max()
    assert abs(Qs - Qs.T).max() <= 1e-12 * abs(Qs).max()
    assert np.linalg.eigvalsh(Qs.toarray()).min() >= -1e-10 * abs(Qs).max()
    G = sp.csr_matrix((np.ones(3 * F.shape[0] * 2), (np.r_[F[:, 0], F[:, 1], F[:, 2], F[:, 1], F[:, 2], F[:, 0]],
                                                      np.r_[F[:, 1], F[:, 2], F[:, 0], F[:, 0], F[:, 1], F[:, 2]])),
                      shape=(n, n)) + sp.eye(n)
    two_ring = (G @ G).tocsr()
    two_ring.sort_indices()
    assert np.array_equal(two_ring.indptr, Qs.indptr) and np.array_equal(two_ring.indices, Qs.indices)


def test_bilaplacian_sphere_closed_form(ora):
    """Closed form on the unit sphere: -Delta z = 2 z, so int (Delta z)^2 =
    4 int z^2: the Rayleigh quotient z^T Q z / z^T M z -> 4 at O(h^2) (error
    ~4x smaller per subdivision; the pointwise strong form does not converge
    for cotan operators, the energy does)."""
    errs = []
    for k in (3, 4, 5):
        V, F = meshgen.icosphere(k)
        Q, M = ora.bilaplacian(V, F)
        z = V[:, 2]
        errs.append(abs(z @ (Q.to_scipy() @ z) / (z @ (M * z)) - 4.0))
    assert errs[0] / errs[1] > 3.5 and errs[1] / errs[2] > 3.5 and errs[2] < 1e-4


def test_bilaplacian_smoothing_solve(ora):
    """The data-smoothing system (alpha Q + (1 - alpha) M) x = (1 - alpha) M f
    (App. D eq. 1 with E_{Delta^2}) on the intrinsic hierarchy reaches the
    dense solution."""
    p = meshgen.make_config(2, subdiv=4)
    V, F = p.levels[0]
    alpha = 1e-4
    A, M = ora.assemble_bilaplacian(V, F, 1 - alpha, alpha)
    f = np.random.default_rng(41).standard_normal((p.n, 1))
    B = (1 - alpha) * M[:, None] * f
    X, hist, rc = ora.MG(p.sizes, p.P, A).solve(B, rel_tol=1e-11, max_cycles=200)
    assert rc == 0
    xs = np.linalg.solve(A.to_scipy().toarray(), B)
    assert np.linalg.norm(X - xs) / np.linalg.norm(xs) <= 1e-9
