"""CPU-only checks of the C-ABI library: it loads, exports every symbol
include/mg.h declares, fails loudly without a GPU, and its host pattern-setup
steps (Alg. 3 colouring, symbolic P^T A P) are bit-exact with the oracle."""
import os
import re

import numpy as np
import pytest

import meshgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mglib():
    from paper_2104_13755_b200 import build
    build.build()
    from paper_2104_13755_b200 import mg
    return mg


def test_header_symbols_exported(mglib):
    src = open(os.path.join(ROOT, "include", "mg.h")).read()
    names = set(re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+(mg_\w+)\s*\(", src, re.M))
    assert len(names) >= 19
    L = mglib.lib()
    for n in sorted(names):
        assert hasattr(L, n), n
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", mglib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mg_\w+)", out))
    assert names <= exported


def test_binary_targets_sm100a(mglib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mglib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_create_fails_loudly_without_gpu(mglib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mglib.MGError):
        mglib.mg_create(0)


def _levels_patterns(ora, p):
    V, F = p.levels[0]
    A, _ = ora.assemble(V, F, p.mass_coeff, p.lap_coeff)
    out = [A]
    for l, (c, w) in enumerate(p.P):
        out.append(ora.galerkin(ora.prolongation(p.sizes[l + 1], c, w), out[-1]))
    return out


@pytest.mark.parametrize("cid,kw", [(1, {}), (1, {"four_grids": True}), (2, {"subdiv": 6}), (3, {"grid": (128, 128)}),
                                    (4, {"subdiv": 5}), (5, {"subdiv": 5})])
def test_host_colouring_and_symbolic_bit_exact(ora, mglib, cid, kw):
    p = meshgen.make_config(cid, **kw)
    mats = _levels_patterns(ora, p)
    for l, A in enumerate(mats):
        rp, col, _ = A.arrays()
        c_lib, k_lib = mglib.mg_util_greedy_colouring(rp.astype(np.int32), col)
        c_ora, k_ora = ora.greedy_colouring(A)
        assert k_lib == k_ora and np.array_equal(c_lib, c_ora), f"level {l}"
        if l + 1 < len(mats):
            Pc, Pw = p.P[l]
            crp, ccol = mglib.mg_util_galerkin_pattern(rp.astype(np.int32), col, p.sizes[l + 1], Pc, Pw)
            orp, ocol, _ = mats[l + 1].arrays()
            assert np.array_equal(crp, orp) and np.array_equal(ccol, ocol), f"level {l + 1}"


def test_host_colouring_random_graphs_bit_exact(ora, mglib):
    import scipy.sparse as sp
    rng = np.random.default_rng(11)
    for t in range(300):
        n = int(rng.integers(1, 60))
        m = int(rng.integers(0, 4 * n + 1))
        e = rng.integers(0, n, size=(m, 2))
        rows = np.concatenate([np.arange(n), e[:, 0], e[:, 1]])
        cols = np.concatenate([np.arange(n), e[:, 1], e[:, 0]])
        S = sp.csr_matrix((np.ones(rows.size), (rows, cols)), shape=(n, n))
        S.sum_duplicates()
        S.sort_indices()
        c_lib, k_lib = mglib.mg_util_greedy_colouring(S.indptr.astype(np.int32), S.indices.astype(np.int32))
        c_ora, k_ora = ora.greedy_colouring(ora.Csr.from_scipy(S))
        assert k_lib == k_ora and np.array_equal(c_lib, c_ora)


def test_symbolic_zero_weights_carry_no_structure(mglib):
    """Reading A9: a P entry with w == 0.0 is padding (no coarse structure)."""
    rp = np.array([0, 2, 4], np.int32)
    col = np.array([0, 1, 0, 1], np.int32)
    Pc = np.array([[0, 1, 1], [1, 0, 0]], np.int32)
    Pw = np.array([[1.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    crp, ccol = mglib.mg_util_galerkin_pattern(rp, col, 2, Pc, Pw)
    assert crp.tolist() == [0, 2, 4] and ccol.tolist() == [0, 1, 0, 1]
    Pw2 = np.array([[1.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    rp1 = np.array([0, 1, 2], np.int32)
    col1 = np.array([0, 1], np.int32)
    crp, ccol = mglib.mg_util_galerkin_pattern(rp1, col1, 2, Pc, Pw2)
    assert crp.tolist() == [0, 1, 2] and ccol.tolist() == [0, 1]


def test_profile_classes_match_library():
    """The binding's kernel-class list must match the library's enum (the
    profile arrays are sized from it)."""
    import re
    from paper_2104_13755_b200 import mg
    src = open(os.path.join(ROOT, "paper_2104_13755_b200", "csrc", "mg_internal.h")).read()
    n = int(re.search(r"constexpr int kProfClasses = (\d+);", src).group(1))
    enum = re.findall(r"PC_\w+ = (\d+)", src)
    assert len(mg.PROF_CLASSES) == n == len(enum) == max(map(int, enum)) + 1


def _brute_opposites(F, i, j):
    """Vertices o with a face {i, j, o} (brute force over the face list)."""
    out = []
    for f in F:
        s = set(int(v) for v in f)
        if i in s and j in s:
            out.extend(s - {i, j})
    return sorted(out)


def _fan(n_ring, closed):
    F = [(0, 1 + k, 1 + (k + 1) % n_ring) for k in range(n_ring)]
    n = n_ring + 1
    if closed:
        F += [(n, 1 + (k + 1) % n_ring, 1 + k) for k in range(n_ring)]
        n += 1
    return n, np.asarray(F, np.int32)


@pytest.mark.parametrize("mesh", ["ico2", "cyl", "fan9", "disk7", "fan14"])
def test_one_ring_pattern_and_opposite_slots(ora, mglib, mesh):
    """Host pattern setup of the cotan assembly: the 1-ring CSR pattern equals
    the oracle's assembled pattern, and the packed row-local slots decode to
    exactly the vertices opposite each stored edge (brute force over the face
    list); diagonal entries and missing opposites (boundary edges) decode to
    'none'."""
    if mesh == "ico2":
        V, F = meshgen.icosphere(2)
        n = V.shape[0]
    elif mesh == "cyl":
        p = meshgen.make_config(3, grid=(12, 9))
        V, F = p.levels[0]
        n = V.shape[0]
    else:
        n, F = _fan(int(mesh[3:] if mesh.startswith("fan") else mesh[4:]), mesh.startswith("fan"))
        V = None
    rp, col, sl = mglib.mg_util_one_ring(n, F)
    if V is not None:
        A, _ = ora.assemble(np.ascontiguousarray(V, np.float64), np.asarray(F, np.int32), 1.0, 1.0)
        orp, ocol, _ = A.arrays()
        assert np.array_equal(rp, orp) and np.array_equal(col, ocol)
    for i in range(n):
        row = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(row) > 0) and i in row
        for e in range(rp[i], rp[i + 1]):
            j = int(col[e])
            got = sorted(int(row[s]) for s in (int(sl[e]) & 15, int(sl[e]) >> 4) if s != 15)
            want = [] if j == i else _brute_opposites(F, i, j)
            assert got == want, (i, j)


def test_one_ring_errors(mglib):
    n, F = _fan(20, True)                      # apex rows of 21 entries: no packed form
    rp, col, _ = mglib.mg_util_one_ring(n, F, slots=False)
    assert rp[1] - rp[0] == 21
    with pytest.raises(mglib.MGError):
        mglib.mg_util_one_ring(n, F)
    with pytest.raises(mglib.MGError):
        mglib.mg_util_one_ring(n + 1, F)       # a vertex in no face
    with pytest.raises(mglib.MGError):
        mglib.mg_util_one_ring(3, np.array([[0, 1, 5]], np.int32))   # index out of range
