"""GPU parity: the CUDA path (libmg through its C ABI) against the CPU oracle
on the same seeded inputs (SURVEY.md §8(c.4) tolerances).

Integer outputs (colourings, coarse CSR patterns) must be bit-exact; X within
1e-9 relative per column at the same cycle count; each cycle's residual norm
within 1e-8 relative plus the rounding floor tau_k (reading A20); coarse
operator values and M within 1e-12 row-normwise.
"""
import numpy as np
import pytest

import meshgen
from parity_util import (check_history, check_level_parity, check_x, gpu_solver, oracle_problem, oracle_rhs,
                         oracle_solve_tau, tau_floor)

pytestmark = pytest.mark.gpu

SMALL = [(1, {}), (1, {"four_grids": True}), (2, {"subdiv": 5}), (3, {"grid": (96, 80)}), (4, {"subdiv": 5}),
         (5, {"subdiv": 5})]


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2104_13755_b200 import build
    build.build()


def _gpu_rhs(S, p, n):
    if p.rhs_kind == "direct":
        return np.ascontiguousarray(p.rhs, np.float64)
    f = np.ascontiguousarray(p.rhs if p.rhs_kind == "mass" else p.levels[0][0], np.float64)
    B = np.empty_like(f)
    S.apply_mass(f, B)
    return B


@pytest.mark.parametrize("cid,kw", SMALL)
def test_assembly_galerkin_colouring(ora, cid, kw):
    p = meshgen.make_config(cid, **kw)
    A, M, mgo = oracle_problem(ora, p)
    S = gpu_solver(p)
    S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
    from paper_2104_13755_b200 import mg
    Mg = mg.mg_get_mass(S.ctx, p.n)
    assert np.abs(Mg - M).max() <= 1e-12 * np.abs(M).max()
    for l in range(len(p.sizes)):
        check_level_parity(S, mgo, l)
    nH = p.sizes[-1]
    Lg = mg.mg_get_coarse_factor(S.ctx, nH)
    Lo = np.tril(mgo.coarse_factor())
    assert np.abs(Lg - Lo).max() <= 1e-11 * np.abs(Lo).max()


@pytest.mark.parametrize("cid,kw", SMALL)
def test_solve_parity(ora, cid, kw):
    p = meshgen.make_config(cid, **kw)
    A, M, mgo = oracle_problem(ora, p)
    S = gpu_solver(p)
    if p.rhs_kind == "mcf":
        pytest.skip("config 5 loop covered by test_mcf_loop_parity")
    S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
    Bo = oracle_rhs(ora, p, M)
    Bg = _gpu_rhs(S, p, p.n)
    assert np.abs(Bg - Bo).max() <= 1e-12 * np.abs(Bo).max()
    Xo, ho, rco, tauo = oracle_solve_tau(mgo, A.to_scipy(), Bo, rel_tol=p.rel_tol, max_cycles=p.max_cycles)
    cyc_o = ho.shape[0] - 1
    # same cycle count: fixed-cycle mode on the GPU
    Xg = np.zeros_like(Bo)
    rc, cyc, hg = S.solve(Bo, Xg, rel_tol=0.0, max_cycles=cyc_o)
    assert cyc == cyc_o
    check_x(Xg, Xo)
    check_history(hg, ho, tauo)
    # own stopping rule: within +-1 cycle of the oracle
    Xg2 = np.zeros_like(Bo)
    rc2, cyc2, hg2 = S.solve(Bo, Xg2, rel_tol=p.rel_tol, max_cycles=p.max_cycles)
    assert rc2 == 0 and abs(cyc2 - cyc_o) <= 1


def test_matrix_from_csr_host_and_device(ora):
    import torch
    p = meshgen.make_config(2, subdiv=5)
    A, M, mgo = oracle_problem(ora, p)
    rp, col, val = A.arrays()
    rp32 = rp.astype(np.int32)
    B = np.random.default_rng(0).standard_normal((p.n, 2))
    Xo, ho, _, tauo = oracle_solve_tau(mgo, A.to_scipy(), B, rel_tol=0.0, max_cycles=6)
    outs = []
    for dev in (False, True):
        S = gpu_solver(p)
        if dev:
            S.set_matrix(torch.from_numpy(rp32).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda())
            Bt = torch.from_numpy(B).cuda()
            Xt = torch.zeros_like(Bt)
            rc, cyc, hg = S.solve(Bt, Xt, rel_tol=0.0, max_cycles=6)
            Xg = Xt.cpu().numpy()
        else:
            S.set_matrix(rp32, col, val)
            Xg = np.zeros_like(B)
            rc, cyc, hg = S.solve(B, Xg, rel_tol=0.0, max_cycles=6)
        for l in range(len(p.sizes)):
            check_level_parity(S, mgo, l)
        check_x(Xg, Xo)
        check_history(hg, ho, tauo)
        outs.append(Xg)
    assert np.array_equal(outs[0], outs[1])      # deterministic kernels: bitwise identical


def test_k_columns_are_independent_and_deterministic(ora):
    p = meshgen.make_config(3, grid=(64, 64))
    S = gpu_solver(p)
    S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
    rng = np.random.default_rng(1)
    B = rng.standard_normal((p.n, 4))
    X4 = np.zeros_like(B)
    S.solve(B, X4, rel_tol=0.0, max_cycles=5)
    for k in (1, 2, 3):
        Xk = np.zeros((p.n, k))
        S.solve(np.ascontiguousarray(B[:, :k]), Xk, rel_tol=0.0, max_cycles=5)
        assert np.array_equal(Xk, X4[:, :k])
    X4b = np.zeros_like(B)
    S.solve(B, X4b, rel_tol=0.0, max_cycles=5)
    assert np.array_equal(X4, X4b)


def test_mcf_loop_parity(ora):
    """Config 5 (implicit MCF, reading A15) on a small sphere: per step GPU
    assembly + Galerkin + factor + apply_mass + warm-started solve, run for
    the oracle's per-step cycle counts."""
    p = meshgen.make_config(5, subdiv=5)
    steps = 5
    V0, F = p.levels[0]
    Xo, cycles = ora.mcf(p.sizes, p.P, V0, F, p.lap_coeff, steps, rel_tol=p.rel_tol)
    S = gpu_solver(p)
    X = np.ascontiguousarray(V0, np.float64).copy()
    for t in range(steps):
        S.set_matrix_cotan(X, 1.0, p.lap_coeff)
        B = np.empty_like(X)
        S.apply_mass(X, B)
        Xn = X.copy()
        rc, cyc, h = S.solve(B, Xn, rel_tol=0.0, max_cycles=cycles[t])
        X = Xn
    check_x(X, Xo)
    # and with the GPU's own stopping rule: same positions to the solve tolerance
    S2 = gpu_solver(p)
    X2 = np.ascontiguousarray(V0, np.float64).copy()
    for t in range(steps):
        S2.set_matrix_cotan(X2, 1.0, p.lap_coeff)
        B = np.empty_like(X2)
        S2.apply_mass(X2, B)
        rc, cyc, h = S2.solve(B, X2, rel_tol=p.rel_tol, max_cycles=p.max_cycles)
        assert rc == 0 and abs(cyc - cycles[t]) <= 1
    assert np.abs(X2 - Xo).max() <= 1e-6 * np.abs(Xo).max()


# --------------------------------------------------------------------------- edge cases


def test_single_level_is_direct_solve(ora):
    levels, _ = meshgen.icosphere_levels(3, 3)
    V, F = levels[0]
    from paper_2104_13755_b200 import mg
    S = mg.Solver(levels, [])
    S.set_matrix_cotan(V, 1.0, 1e-2)
    A, M = ora.assemble(V, F, 1.0, 1e-2)
    b = np.random.default_rng(2).standard_normal((V.shape[0], 1))
    X = np.zeros_like(b)
    rc, cyc, h = S.solve(b, X, rel_tol=1e-12, max_cycles=3)
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    assert rc == 0 and cyc == 1
    assert np.linalg.norm(X - xs) <= 1e-12 * np.linalg.norm(xs)


def _fan_mesh(n_ring, closed, seed):
    """Apex (valence n_ring) over a jittered ring; closed: a second apex below
    (bipyramid), else an open disk whose ring edges are boundary edges."""
    rng = np.random.default_rng(seed)
    t = 2 * np.pi * (np.arange(n_ring) + 0.2 * rng.uniform(-1, 1, n_ring)) / n_ring
    ring = np.stack([np.cos(t), np.sin(t), 0.1 * rng.standard_normal(n_ring)], axis=1)
    V = [np.array([[0.05, -0.03, 0.8]]), ring]
    F = [(0, 1 + k, 1 + (k + 1) % n_ring) for k in range(n_ring)]
    if closed:
        V.append(np.array([[-0.02, 0.04, -0.9]]))
        b = n_ring + 1
        F += [(b, 1 + (k + 1) % n_ring, 1 + k) for k in range(n_ring)]
    return np.ascontiguousarray(np.concatenate(V), np.float64), np.asarray(F, np.int32)


@pytest.mark.parametrize("n_ring,closed", [(6, True), (7, True), (9, True), (14, True), (20, True), (9, False),
                                           (18, False)])
def test_cotan_long_rows(ora, n_ring, closed):
    """Rows of the 1-ring pattern longer than the 8 lanes of the assembly
    kernel (row-local opposite-vertex slots looked up through the columns),
    longer than 15 entries (index-table kernel), and boundary edges with a
    single opposite vertex: mass and the single-level direct solve against
    the oracle's assembly."""
    from paper_2104_13755_b200 import mg
    V, F = _fan_mesh(n_ring, closed, 5 + n_ring)
    S = mg.Solver([(V, F)], [])
    S.set_matrix_cotan(V, 1.0, 0.3)
    A, M = ora.assemble(V, F, 1.0, 0.3)
    Mg = mg.mg_get_mass(S.ctx, V.shape[0])
    assert np.abs(Mg - M).max() <= 1e-12 * np.abs(M).max()
    b = np.random.default_rng(3).standard_normal((V.shape[0], 2))
    X = np.zeros_like(b)
    rc, cyc, h = S.solve(b, X, rel_tol=1e-12, max_cycles=3)
    xs = np.linalg.solve(A.to_scipy().toarray(), b)
    assert rc == 0
    assert np.linalg.norm(X - xs) <= 1e-11 * np.linalg.norm(xs)
    S.close()


def test_zero_rhs_and_loose_tolerance(ora):
    p = meshgen.make_config(1)
    S = gpu_solver(p)
    S.set_matrix_cotan(p.levels[0][0], 1.0, 1e-3)
    Z = np.zeros((p.n, 1))
    X = np.zeros((p.n, 1))
    rc, cyc, h = S.solve(Z, X, rel_tol=1e-10, max_cycles=5)
    assert rc == 0 and cyc == 0 and not X.any()
    b = np.ones((p.n, 1))
    rc, cyc, h = S.solve(b, X, rel_tol=2.0, max_cycles=5)
    assert rc == 0 and cyc == 0 and h[0, 0] == 1.0
    from paper_2104_13755_b200 import mg
    rc, cyc, h = S.solve(b, X, rel_tol=1e-30, max_cycles=3)
    assert rc == mg.MG_NOT_CONVERGED and cyc == 3 and h.shape[0] == 4


def test_errors_are_reported():
    from paper_2104_13755_b200 import mg
    p = meshgen.make_config(1)
    ctx = mg.mg_create(0)
    try:
        with pytest.raises(mg.MGError) as e:
            mg.mg_solve(ctx, 1, np.zeros((p.n, 1)), np.zeros((p.n, 1)), 1e-8, 3)
        assert e.value.code == mg.MG_ERR_STATE
        bad = [(c, w.copy()) for c, w in p.P]
        bad[0][1][5, 0] += 1e-6
        with pytest.raises(mg.MGError) as e:
            mg.mg_hierarchy_load(ctx, p.levels, bad)
        assert e.value.code == mg.MG_ERR_INPUT and "row 5" in str(e.value)
        mg.mg_hierarchy_load(ctx, p.levels, p.P)
        with pytest.raises(mg.MGError) as e:
            mg.mg_set_matrix_cotan(ctx, p.levels[0][0], 1.0, -2.0)   # indefinite: coarse pivot fails
        assert e.value.code == mg.MG_ERR_NOT_SPD
        mg.mg_set_matrix_cotan(ctx, p.levels[0][0], 1.0, 1e-3)
        with pytest.raises(mg.MGError) as e:
            mg.mg_solve(ctx, 5, np.zeros((p.n, 5)), np.zeros((p.n, 5)), 1e-8, 3)
        assert e.value.code == mg.MG_ERR_INVALID_ARG
        b = np.ones((p.n, 1))
        b[3] = np.nan
        with pytest.raises(mg.MGError) as e:
            mg.mg_solve(ctx, 1, b, np.zeros((p.n, 1)), 1e-8, 3)
        assert e.value.code == mg.MG_ERR_NUMERIC
        mg.mg_set_zero_guess(ctx, True)                  # rho_0 = 1 shortcut keeps a NaN |b| a NaN
        with pytest.raises(mg.MGError) as e:
            mg.mg_solve(ctx, 1, b, np.zeros((p.n, 1)), 1e-8, 3)
        assert e.value.code == mg.MG_ERR_NUMERIC
        mg.mg_set_zero_guess(ctx, False)
        # the binding checks extents the C side cannot see
        with pytest.raises(ValueError):
            mg.mg_solve(ctx, 1, np.ones((p.n - 1, 1)), np.zeros((p.n - 1, 1)), 1e-8, 3)
        with pytest.raises(ValueError):
            mg.mg_solve(ctx, 3, np.ones((p.n, 2)), np.zeros((p.n, 2)), 1e-8, 3)
        with pytest.raises(ValueError):
            mg.mg_solve(ctx, 1, np.ones((p.n, 1)), np.zeros((p.n, 1)), 1e-8, 3, np.zeros(3))
        with pytest.raises(ValueError):
            mg.mg_apply_mass(ctx, 1, np.ones((p.n, 2)), np.zeros((p.n, 2)))
        with pytest.raises(ValueError):
            mg.mg_set_matrix_cotan(ctx, p.levels[0][0][:-1], 1.0, 1e-3)
        with pytest.raises(mg.MGError) as e:
            mg.mg_set_matrix(ctx, p.n - 1, 1, np.zeros(p.n, np.int32), np.zeros(1, np.int32), np.ones(1))
        assert e.value.code == mg.MG_ERR_SHAPE
    finally:
        mg.mg_destroy(ctx)


# --------------------------------------------------------------------------- full sizes


@pytest.mark.slow
@pytest.mark.parametrize("cid", [2, 3, 4])
def test_full_size_parity(ora, cid):
    """BASELINE.json configs 2, 3 and 4 at full size (the launch configuration
    bench.py times), full-vector comparison: every level's pattern, colouring
    and values, and the solve at the oracle's own cycle count."""
    p = meshgen.make_config(cid)
    A, M, mgo = oracle_problem(ora, p)
    S = gpu_solver(p)
    S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
    for l in range(len(p.sizes)):
        check_level_parity(S, mgo, l)
    Bo = oracle_rhs(ora, p, M)
    Xo, ho, rco, tauo = oracle_solve_tau(mgo, A.to_scipy(), Bo, rel_tol=p.rel_tol, max_cycles=p.max_cycles)
    assert rco == 0
    Xg = np.zeros_like(Bo)
    rc, cyc, hg = S.solve(_gpu_rhs(S, p, p.n), Xg, rel_tol=0.0, max_cycles=ho.shape[0] - 1)
    check_x(Xg, Xo)
    check_history(hg, ho, tauo)


def test_launch_modes_agree(ora):
    """Scheduling variants (mg_set_execution) must not change the arithmetic:
    PDL on/off, the pipelined (TMA bulk) vs plain tile kernels and the
    device-side cycle loop give bitwise-identical iterates.  The one-CTA triangular
    coarsest solve vs the explicit-inverse GEMV (both Alg. 2's direct solve,
    reading A12) agree with the oracle to the X tolerance."""
    from paper_2104_13755_b200 import mg
    for cid, kw in ((4, {"subdiv": 6}), (3, {"grid": (160, 128)})):
        p = meshgen.make_config(cid, **kw)
        A, M, mgo = oracle_problem(ora, p)
        Bo = oracle_rhs(ora, p, M)
        Xo, ho, _ = mgo.solve(Bo, rel_tol=0.0, max_cycles=5)
        variants = {
            "default": 0,
            "nopdl": mg.MG_EXEC_NO_PDL,
            "nopipe": mg.MG_EXEC_NO_PIPE,
            "nopdl_nopipe": mg.MG_EXEC_NO_PDL | mg.MG_EXEC_NO_PIPE,
            "deviceloop": mg.MG_EXEC_DEVICE_LOOP,
            "trsv": mg.MG_EXEC_COARSE_TRSV,
        }
        out = {}
        for name, flags in variants.items():
            S = gpu_solver(p)
            mg.mg_set_execution(S.ctx, flags)
            S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
            X = np.zeros_like(Bo)
            S.solve(Bo, X, rel_tol=0.0, max_cycles=5)
            check_x(X, Xo)
            out[name] = X
            # symmetric V-cycle (reversed post colours) through the same kernels
            S.set_smoother(0, 0.8, True)
            Xs = np.zeros_like(Bo)
            S.solve(Bo, Xs, rel_tol=0.0, max_cycles=3)
            out[name + "_sym"] = Xs
            S.close()
        for name in variants:
            if name == "trsv":
                continue
            assert np.array_equal(out["default"], out[name]), name
            assert np.array_equal(out["default_sym"], out[name + "_sym"]), name


@pytest.mark.parametrize("cid,kw", [(4, {"subdiv": 5}), (3, {"grid": (96, 80)})])
def test_fast_alpha_sweep_matches_slow_path(ora, cid, kw):
    """SURVEY row f1 (App. D): P^T Q P and P^T M P precomputed once,
    A_h(alpha) = alpha Q_h + (1 - alpha) M_h by scaled addition.  Every level
    must equal the oracle's SLOW path (Galerkin of the assembled
    A = alpha L + (1 - alpha) M, App. D eq. 1) to 1e-12, the solve of
    (alpha L + (1 - alpha) M) x = (1 - alpha) M f must match, and the alpha
    loop must run zero triple products (profile counter)."""
    from paper_2104_13755_b200 import mg
    p = meshgen.make_config(cid, **kw)
    V, F = p.levels[0]
    S = gpu_solver(p)
    S.set_matrix_split_cotan(V)
    mg.mg_set_profiling(S.ctx, ["galerkin", "alpha"])
    mg.mg_get_profile(S.ctx)
    f = np.random.default_rng(7).standard_normal((p.n, 1))
    for alpha in (0.0, 0.1, 0.5, 0.9, 1e-4 / (1 + 1e-4)):
        S.set_alpha(alpha)
        A, M = ora.assemble(V, F, 1.0 - alpha, alpha)
        mgo = ora.MG(p.sizes, p.P, A)
        for l in range(len(p.sizes)):
            check_level_parity(S, mgo, l)
        B = np.ascontiguousarray((1.0 - alpha) * M[:, None] * f)
        Xo, ho, _, tauo = oracle_solve_tau(mgo, A.to_scipy(), B, rel_tol=0.0, max_cycles=4)
        Xg = np.zeros_like(B)
        rc, cyc, hg = S.solve(B, Xg, rel_tol=0.0, max_cycles=4)
        check_x(Xg, Xo)
        check_history(hg, ho, tauo)
    prof = mg.mg_get_profile(S.ctx)
    assert "galerkin" not in prof, prof                       # no triple product in the alpha loop
    assert sum(n for _, n in prof["alpha"].values()) == 5 * len(p.sizes)


def test_split_csr_equals_split_cotan(ora):
    """mg_set_matrix_split with user CSR (Q = L, M = diag mass on the same
    pattern) gives the same operators as the GPU-assembled split path."""
    import scipy.sparse as sp
    from paper_2104_13755_b200 import mg
    p = meshgen.make_config(2, subdiv=4)
    V, F = p.levels[0]
    L, _ = ora.assemble(V, F, 0.0, 1.0)
    _, M = ora.assemble(V, F, 1.0, 0.0)
    Ls = L.to_scipy().tocsr()
    Ls.sort_indices()
    Mv = np.zeros_like(Ls.data)
    rows = np.repeat(np.arange(p.n), np.diff(Ls.indptr))
    Mv[Ls.indices == rows] = M                                # M on the diagonal slots of the same pattern
    Ms = sp.csr_matrix((Mv, Ls.indices.copy(), Ls.indptr.copy()), shape=Ls.shape)
    S1 = gpu_solver(p)
    S1.set_matrix_split(Ls.indptr.astype(np.int32), Ls.indices.astype(np.int32), Ls.data, Ms.data)
    S2 = gpu_solver(p)
    S2.set_matrix_split_cotan(V)
    for alpha in (0.25, 0.75):
        S1.set_alpha(alpha)
        S2.set_alpha(alpha)
        A, _ = ora.assemble(V, F, 1.0 - alpha, alpha)
        mgo = ora.MG(p.sizes, p.P, A)
        for l in range(len(p.sizes)):
            check_level_parity(S1, mgo, l)
            check_level_parity(S2, mgo, l)
    with pytest.raises(mg.MGError):
        gpu_solver(p).set_alpha(0.5)                          # MG_ERR_STATE: no split operators


@pytest.mark.parametrize("cid,kw", [(4, {"subdiv": 5}), (3, {"grid": (96, 80)}), (4, {"subdiv": 8})])
def test_smoother_variants_parity(ora, cid, kw):
    """Row f4: damped-Jacobi smoothing (App. E) and the symmetric
    (reversed post colours) V-cycle match the oracle's same variants (the
    655k-row case runs level 1 through the pipelined lanes-per-row tiles)."""
    p = meshgen.make_config(cid, **kw)
    A, M, _ = oracle_problem(ora, p)
    Bo = oracle_rhs(ora, p, M)
    for kind, omega, sym in ((1, 0.8, False), (1, 0.6, True), (0, 0.8, True)):
        mgo = ora.MG(p.sizes, p.P, A).set_smoother(kind, omega, sym)
        Xo, ho, _, tauo = oracle_solve_tau(mgo, A.to_scipy(), Bo, rel_tol=0.0, max_cycles=4)
        S = gpu_solver(p)
        S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
        S.set_smoother(kind, omega, sym)
        Xg = np.zeros_like(Bo)
        rc, cyc, hg = S.solve(Bo, Xg, rel_tol=0.0, max_cycles=4)
        check_x(Xg, Xo)
        check_history(hg, ho, tauo)
        S.close()


@pytest.mark.parametrize("cid,kw", [(4, {"subdiv": 5}), (3, {"grid": (96, 80)}), (2, {"subdiv": 5})])
def test_pcg_parity(ora, cid, kw):
    """Row f4: MG-preconditioned CG on the GPU against the oracle's
    PCG: same iterate after the same iterations, same recursive-residual
    history; its own stopping rule within +-1 iteration."""
    p = meshgen.make_config(cid, **kw)
    A, M, _ = oracle_problem(ora, p)
    Bo = oracle_rhs(ora, p, M)
    for kind in (0, 1):
        mgo = ora.MG(p.sizes, p.P, A).set_smoother(kind, 0.8)
        Xo, ho, rco = mgo.pcg(Bo, rel_tol=1e-10, max_iters=60)
        it_o = ho.shape[0] - 1
        S = gpu_solver(p)
        S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
        S.set_smoother(kind, 0.8)
        Xg = np.zeros_like(Bo)
        rc, it, hg = S.solve_pcg(Bo, Xg, rel_tol=0.0, max_iters=it_o)
        assert it == it_o
        check_x(Xg, Xo)
        check_history(hg, ho, tau_floor(A.to_scipy(), Xo, Bo))
        Xg2 = np.zeros_like(Bo)
        rc2, it2, _ = S.solve_pcg(Bo, Xg2, rel_tol=1e-10, max_iters=60)
        assert rc2 == 0 and abs(it2 - it_o) <= 1
        S.close()
    # a solved (zero) column among k = 3 stays solved: alpha = beta = 0 (reading A27)
    Bz = np.ascontiguousarray(np.concatenate([Bo[:, :1], np.zeros((p.n, 1)), Bo[:, :1] * 2.0], axis=1))
    mgo = ora.MG(p.sizes, p.P, A)
    Xo, ho, rco = mgo.pcg(Bz, rel_tol=0.0, max_iters=5)
    assert np.all(np.isfinite(Xo)) and np.all(Xo[:, 1] == 0.0)
    S = gpu_solver(p)
    S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
    Xg = np.zeros_like(Bz)
    rc, it, hg = S.solve_pcg(Bz, Xg, rel_tol=0.0, max_iters=5)
    assert rc == 0 and np.all(Xg[:, 1] == 0.0)
    check_x(Xg, Xo)
    S.close()
    from paper_2104_13755_b200 import mg
    S = gpu_solver(p, mu=(2, 1))
    S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
    with pytest.raises(mg.MGError):
        S.solve_pcg(Bo, np.zeros_like(Bo))                # mu_pre != mu_post: not a symmetric preconditioner


@pytest.mark.slow
def test_full_size_mcf_steps(ora):
    """BASELINE.json config 5 exactly as stated: 20 implicit MCF steps on the
    655,362-vertex sphere (GPU assembly -> Galerkin -> factor -> B = M X ->
    warm-started solve to 1e-8, X_{t+1} = X).  The GPU chain feeds its OWN
    positions into the next step's assembly, so drift over the 20 steps is
    what is tested: after every step X within 1e-9 per column of the oracle's
    chain at the oracle's cycle count, the residual history by the A20 rule
    (tau_k at x_k) with the literal rule logged; a second GPU chain with its
    own stopping rule stops within +-1 cycle of the oracle at every step."""
    p = meshgen.make_config(5)
    V, F = p.levels[0]
    steps = 20
    S = gpu_solver(p)
    S2 = gpu_solver(p)
    Xo = np.ascontiguousarray(V, np.float64).copy()
    Xg = Xo.copy()
    Xs = Xo.copy()
    for t in range(steps):
        A, M = ora.assemble(Xo, F, p.mass_coeff, p.lap_coeff)
        mgo = ora.MG(p.sizes, p.P, A)
        Bo = np.ascontiguousarray(M[:, None] * Xo)
        Xo, ho, rco, tauo = oracle_solve_tau(mgo, A.to_scipy(), Bo, X0=Xo, rel_tol=p.rel_tol,
                                              max_cycles=p.max_cycles)
        assert rco == 0
        cyc_o = ho.shape[0] - 1
        S.set_matrix_cotan(Xg, p.mass_coeff, p.lap_coeff)   # GPU positions: drift accumulates here
        B = np.empty_like(Xg)
        S.apply_mass(Xg, B)
        rc, cyc, hg = S.solve(B, Xg, rel_tol=0.0, max_cycles=cyc_o)
        assert cyc == cyc_o
        check_x(Xg, Xo)
        check_history(hg, ho, tauo, tag=f"C5 full size, step {t + 1} of {steps}")
        S2.set_matrix_cotan(Xs, p.mass_coeff, p.lap_coeff)
        B2 = np.empty_like(Xs)
        S2.apply_mass(Xs, B2)
        rc2, cyc2, _ = S2.solve(B2, Xs, rel_tol=p.rel_tol, max_cycles=p.max_cycles)
        assert rc2 == 0 and abs(cyc2 - cyc_o) <= 1, (t, cyc2, cyc_o)
    # own stopping rule: the chain stays on the oracle's to the solve tolerance
    assert np.abs(Xs - Xo).max() <= 1e-6 * np.abs(Xo).max()
    S.close()
    S2.close()


def _dirichlet_case(ora, p, known, k, seed):
    rng = np.random.default_rng(seed)
    A, M = ora.assemble(p.levels[0][0], p.levels[0][1], p.mass_coeff, p.lap_coeff)
    X0 = np.zeros((p.n, k))
    X0[known] = rng.standard_normal((len(known), k))
    B = np.ascontiguousarray(M[:, None] * rng.standard_normal((p.n, k)))
    return A, M, X0, B


@pytest.mark.parametrize("cid,kw,frac", [(2, {"subdiv": 5}, 0.1), (3, {"grid": (96, 80)}, 0.0), (1, {}, 0.3)])
def test_dirichlet_parity(ora, cid, kw, frac):
    """Row f2 (App. B): constrained solves through both matrix paths (user
    CSR and GPU cotan assembly) against the oracle's reduction: reduced
    patterns and colourings bit-exact, X and history within tolerance, known
    rows untouched.  Config 3 constrains both boundary loops (Dirichlet BC
    on the open cylinder)."""
    import torch
    p = meshgen.make_config(cid, **kw)
    rng = np.random.default_rng(31)
    if cid == 3:
        z = p.levels[0][0][:, 2]
        known = np.nonzero((z <= z.min() + 1e-12) | (z >= z.max() - 1e-12))[0]
    else:
        known = np.sort(rng.choice(p.n, int(frac * p.n), replace=False))
    A, M, X0, B = _dirichlet_case(ora, p, known, 2, 32)
    Xo, ho, rco, mgo = ora.dirichlet_solve(p.sizes, p.P, A, B, X0, known, rel_tol=0.0, max_cycles=5)
    rp, col, val = A.arrays()
    for path in ("csr", "cotan", "csr_device"):
        S = gpu_solver(p)
        S.set_dirichlet(known)
        if path == "cotan":
            S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
        elif path == "csr":
            S.set_matrix(rp.astype(np.int32), col, val)
        else:
            S.set_matrix(torch.from_numpy(rp.astype(np.int32)).cuda(), torch.from_numpy(col).cuda(),
                         torch.from_numpy(val).cuda())
        for l in range(mgo.n_levels):
            check_level_parity(S, mgo, l)
        if path == "csr_device":
            Xt = torch.from_numpy(X0.copy()).cuda()
            rc, cyc, hg = S.solve(torch.from_numpy(B).cuda(), Xt, rel_tol=0.0, max_cycles=5)
            Xg = Xt.cpu().numpy()
        else:
            Xg = X0.copy()
            rc, cyc, hg = S.solve(B, Xg, rel_tol=0.0, max_cycles=5)
        assert np.array_equal(Xg[known], X0[known])
        check_x(Xg, Xo)
        Su = A.to_scipy()
        u = np.setdiff1d(np.arange(p.n), known)
        bu = B[u] - Su[u][:, known] @ X0[known]
        check_history(hg, ho, tau_floor(Su[u][:, u], Xo[u], bu))
        if path == "cotan":
            Mg = np.empty((p.n, 2))
            S.apply_mass(np.ones((p.n, 2)), Mg)
            assert np.abs(Mg[:, 0] - M).max() <= 1e-12 * M.max()
        S.close()


def test_dirichlet_edge_cases(ora):
    from paper_2104_13755_b200 import mg
    p = meshgen.make_config(1, subdiv=3)                  # nested: 642 -> 162 -> 42
    A, M = ora.assemble(p.levels[0][0], p.levels[0][1], p.mass_coeff, p.lap_coeff)
    rp, col, val = A.arrays()
    rp = rp.astype(np.int32)
    rng = np.random.default_rng(33)
    # every child of coarse vertex 7 known: its column of P_{u:} vanishes
    c0, w0 = p.P[0]
    children = np.nonzero(((c0 == 7) & (w0 != 0.0)).any(axis=1))[0]
    A_, M_, X0, B = _dirichlet_case(ora, p, children, 1, 34)
    Xo, ho, _, mgo = ora.dirichlet_solve(p.sizes, p.P, A, B, X0, children, rel_tol=0.0, max_cycles=6)
    S = gpu_solver(p)
    S.set_dirichlet(children)
    S.set_matrix(rp, col, val)
    assert mg.mg_level_info(S.ctx, 1)[0] == p.sizes[1] - 1
    for l in range(mgo.n_levels):
        check_level_parity(S, mgo, l)
    Xg = X0.copy()
    S.solve(B, Xg, rel_tol=0.0, max_cycles=6)
    check_x(Xg, Xo)
    # all known: nothing to solve, X unchanged
    S.set_dirichlet(np.arange(p.n))
    S.set_matrix(rp, col, val)
    Xa = rng.standard_normal((p.n, 1))
    Xc = Xa.copy()
    rc, cyc, h = S.solve(B, Xc, rel_tol=1e-10, max_cycles=5)
    assert rc == 0 and cyc == 0 and np.array_equal(Xc, Xa)
    # no constraints again: identical to a fresh unconstrained context
    S.set_dirichlet([])
    S.set_matrix(rp, col, val)
    X1 = np.zeros_like(B)
    S.solve(B, X1, rel_tol=0.0, max_cycles=4)
    S2 = gpu_solver(p)
    S2.set_matrix(rp, col, val)
    X2 = np.zeros_like(B)
    S2.solve(B, X2, rel_tol=0.0, max_cycles=4)
    assert np.array_equal(X1, X2)
    with pytest.raises(mg.MGError):
        S.set_dirichlet([0, 0])                           # repeated index
    with pytest.raises(mg.MGError):
        S.set_dirichlet([p.n])                            # out of range


@pytest.mark.parametrize("cid,kw", [(2, {"subdiv": 5}), (3, {"grid": (96, 80)}), (1, {})])
def test_bilaplacian_parity(ora, cid, kw):
    """Row f3: GPU assembly of A = (1 - alpha) M + alpha L M^{-1} L on the
    2-ring (E_{Delta^2} smoothing) against the oracle (scipy product of its
    own L and M): 2-ring pattern / colourings bit-exact on every level,
    values, M and the smoothing solve within tolerance; also with Dirichlet
    constraints (row f2 on a 2-ring operator)."""
    p = meshgen.make_config(cid, **kw)
    V, F = p.levels[0]
    alpha = 1e-3
    A, M = ora.assemble_bilaplacian(V, F, 1 - alpha, alpha)
    f = np.random.default_rng(51).standard_normal((p.n, 2))
    B = np.ascontiguousarray((1 - alpha) * M[:, None] * f)
    mgo = ora.MG(p.sizes, p.P, A)
    Xo, ho, _, tauo = oracle_solve_tau(mgo, A.to_scipy(), B, rel_tol=0.0, max_cycles=5)
    S = gpu_solver(p)
    S.set_matrix_bilaplacian(V, 1 - alpha, alpha)
    from paper_2104_13755_b200 import mg
    assert np.abs(mg.mg_get_mass(S.ctx, p.n) - M).max() <= 1e-12 * M.max()
    for l in range(len(p.sizes)):
        check_level_parity(S, mgo, l)
    Xg = np.zeros_like(B)
    rc, cyc, hg = S.solve(B, Xg, rel_tol=0.0, max_cycles=5)
    check_x(Xg, Xo)
    check_history(hg, ho, tauo)
    known = np.sort(np.random.default_rng(52).choice(p.n, p.n // 8, replace=False))
    X0 = np.zeros_like(B)
    X0[known] = 1.0
    Xo2, ho2, _, mgo2 = ora.dirichlet_solve(p.sizes, p.P, A, B, X0, known, rel_tol=0.0, max_cycles=4)
    S.set_dirichlet(known)
    S.set_matrix_bilaplacian(V, 1 - alpha, alpha)
    for l in range(mgo2.n_levels):
        check_level_parity(S, mgo2, l)
    Xg2 = X0.copy()
    S.solve(B, Xg2, rel_tol=0.0, max_cycles=4)
    check_x(Xg2, Xo2)
    S.close()


@pytest.mark.parametrize("mu", [(1, 3), (0, 2), (3, 0)])
def test_relaxation_counts_parity(ora, mu):
    """mg_set_options(mu_pre, mu_post): asymmetric and one-sided
    relaxation match the oracle with the same counts."""
    p = meshgen.make_config(2, subdiv=5)
    A, M, mgo = oracle_problem(ora, p, mu)
    Bo = oracle_rhs(ora, p, M)
    Xo, ho, _, tauo = oracle_solve_tau(mgo, A.to_scipy(), Bo, rel_tol=0.0, max_cycles=4)
    S = gpu_solver(p, mu)
    S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
    Xg = np.zeros_like(Bo)
    S.solve(Bo, Xg, rel_tol=0.0, max_cycles=4)
    check_x(Xg, Xo)
    check_history(S.solve(Bo, np.zeros_like(Bo), rel_tol=0.0, max_cycles=4)[2], ho, tauo)


def test_k4_and_mass_dominated(ora):
    """k = 4 right-hand sides (the kernels' maximum) and A = M (lap_coeff 0:
    a diagonal fine operator, every colour class independent)."""
    p = meshgen.make_config(3, grid=(80, 64))
    V, F = p.levels[0]
    for lap in (1e-2, 0.0):
        A, M = ora.assemble(V, F, 1.0, lap)
        mgo = ora.MG(p.sizes, p.P, A)
        B = np.random.default_rng(61).standard_normal((p.n, 4))
        Xo, ho, _, tauo = oracle_solve_tau(mgo, A.to_scipy(), B, rel_tol=0.0, max_cycles=3)
        S = gpu_solver(p)
        S.set_matrix_cotan(V, 1.0, lap)
        Xg = np.zeros_like(B)
        rc, cyc, hg = S.solve(B, Xg, rel_tol=0.0, max_cycles=3)
        check_x(Xg, Xo)
        check_history(hg, ho, tauo)
        S.close()


def test_new_api_errors():
    from paper_2104_13755_b200 import mg
    p = meshgen.make_config(1)
    S = gpu_solver(p)
    with pytest.raises(mg.MGError) as e:
        S.set_alpha(0.5)                                  # no split operators yet
    assert e.value.code == mg.MG_ERR_STATE
    with pytest.raises(mg.MGError) as e:
        S.set_smoother(2)                                 # unknown kind
    assert e.value.code == mg.MG_ERR_INVALID_ARG
    with pytest.raises(mg.MGError) as e:
        S.set_smoother(1, 1.5)                            # Jacobi damping outside (0, 1]
    assert e.value.code == mg.MG_ERR_INVALID_ARG
    S.set_matrix_split_cotan(p.levels[0][0])
    with pytest.raises(mg.MGError) as e:
        S.set_alpha(float("nan"))
    assert e.value.code == mg.MG_ERR_INVALID_ARG
    S.set_dirichlet([1, 2, 3])
    with pytest.raises(mg.MGError) as e:
        S.set_matrix_split_cotan(p.levels[0][0])          # split operators + constraints
    assert e.value.code == mg.MG_ERR_STATE
    with pytest.raises(mg.MGError) as e:
        S.solve(np.zeros((p.n, 1)), np.zeros((p.n, 1)))   # constraints reset the matrix
    assert e.value.code == mg.MG_ERR_STATE
    S.close()


def test_zero_guess(ora):
    """mg_set_zero_guess: X is output only — garbage on input gives the same
    iterate (bitwise) as an explicit zero guess, for host and device X, for
    mg_solve and mg_solve_pcg; ignored under Dirichlet constraints."""
    import torch
    p = meshgen.make_config(4, subdiv=5)
    A, M, mgo = oracle_problem(ora, p)
    Bo = oracle_rhs(ora, p, M)
    Xo, ho, _, tauo = oracle_solve_tau(mgo, A.to_scipy(), Bo, rel_tol=0.0, max_cycles=3)
    S = gpu_solver(p)
    S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
    X0 = np.zeros_like(Bo)
    S.solve(Bo, X0, rel_tol=0.0, max_cycles=3)
    check_x(X0, Xo)
    S.set_zero_guess(True)
    Xg = np.full_like(Bo, 1e30)
    _, _, hz = S.solve(Bo, Xg, rel_tol=0.0, max_cycles=3)
    assert np.array_equal(Xg, X0)
    assert np.all(hz[0] == 1.0)                        # r0 = b exactly: rho_0 = 1 without a residual pass
    check_history(hz, ho, tauo)
    Xd = torch.full(Bo.shape, float("nan"), dtype=torch.float64, device="cuda")
    S.solve(torch.from_numpy(Bo).cuda(), Xd, rel_tol=0.0, max_cycles=3)
    assert np.array_equal(Xd.cpu().numpy(), X0)
    P1 = np.full_like(Bo, -7.0)
    S.solve_pcg(Bo, P1, rel_tol=0.0, max_iters=3)
    S.set_zero_guess(False)
    P0 = np.zeros_like(Bo)
    S.solve_pcg(Bo, P0, rel_tol=0.0, max_iters=3)
    assert np.array_equal(P1, P0)
    S.close()


def test_device_loop_matches_host_loop(ora):
    """The device-side cycle loop (conditional graph node, one launch per
    solve) applies mg_solve's stopping rule exactly like the host loop: same
    cycle count, bitwise-identical history and iterate, for a tolerance stop,
    a cycle-budget stop and a zero budget."""
    p = meshgen.make_config(4, subdiv=5)
    A, M, mgo = oracle_problem(ora, p)
    Bo = oracle_rhs(ora, p, M)
    res = {}
    from paper_2104_13755_b200 import mg
    for mode in ("1", "0"):
        S = gpu_solver(p, execution=mg.MG_EXEC_DEVICE_LOOP if mode == "1" else 0)
        S.set_matrix_cotan(p.levels[0][0], p.mass_coeff, p.lap_coeff)
        out = []
        for tol, mc in ((1e-8, 50), (1e-30, 4), (1e-8, 0)):
            X = np.zeros_like(Bo)
            rc, cyc, h = S.solve(Bo, X, rel_tol=tol, max_cycles=mc)
            out.append((rc, cyc, h.copy(), X.copy()))
        res[mode] = out
        S.close()
    for a, b in zip(res["1"], res["0"]):
        assert a[0] == b[0] and a[1] == b[1]
        assert np.array_equal(a[2], b[2])
        assert np.array_equal(a[3], b[3])
    assert res["1"][1][1] == 4 and res["1"][2][1] == 0
