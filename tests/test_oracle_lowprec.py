"""Pins for the oracle's stage 1 (Alg. 1 step 1):
FP32 LDL^T with symmetric max-|diag| pivoting and threshold postponing,
rules [R2]-[R10] of DESIGN.md."""
import numpy as np
import pytest

import hf_inputs as hi
import oracle
from tests.exact_ldlt import left_looking_ldlt


def _scaled(n, seed, kind="sym"):
    rng = np.random.default_rng(seed)
    if kind == "sym":
        A = rng.standard_normal((n, n))
        Kb = A + A.T
    elif kind == "int":          # small integers: many exact ties mid-factorization
        A = rng.integers(-3, 4, (n, n)).astype(float)
        Kb = A + A.T + np.diag(rng.integers(1, 4, n))
    else:
        raise ValueError(kind)
    K, _ = oracle.scale(Kb)
    return K


@pytest.mark.parametrize("n,seed,kind", [(5, 0, "sym"), (8, 1, "sym"), (12, 2, "sym"),
                                         (9, 3, "int"), (12, 4, "int"), (10, 5, "sym")])
def test_bitwise_equal_to_exact_left_looking_emulation(n, seed, kind):
    """Right-looking with swaps (oracle) == left-looking without swaps in exact
    rational arithmetic with explicit binary32 rounding (test), bit for bit:
    pivot order, D and L.  Pins argmax/tie rule, stop rule, the role-symmetric
    update and its order (R3, R4, R7, R8, R10)."""
    K = _scaled(n, seed, kind)
    tau = 1e-2
    piv, D, Lcols = left_looking_ldlt(K, tau)
    F = oracle.factor_lowprec(K, tau)
    assert F.Ntau == len(piv)
    assert list(F.perm[: F.N]) == piv
    assert np.array_equal(F.D, np.array(D, dtype=np.float32))
    pos = {p: i for i, p in enumerate(piv)}
    for k, lc in enumerate(Lcols):
        for I, val in lc.items():
            if I in pos:
                assert F.Lfac[pos[I], k] == np.float32(val), (k, I)


def test_diagonal_matrix_sorted_with_smallest_index_ties():
    d = np.array([0.5, -2.0, 0.5, 3.0, -0.5, 1e-1, 2.0])
    K = np.diag(d)   # already "scaled" enough for stage 1 (only ratios matter)
    F = oracle.factor_lowprec(K, 1e-3)
    expect = sorted(range(7), key=lambda i: (-abs(d[i]), i))
    assert list(F.perm) == expect
    assert np.array_equal(F.D, d[expect].astype(np.float32))
    assert np.array_equal(F.Lfac, np.eye(7, dtype=np.float32))


def test_spec_postpone_example():
    # diag(1, 0.9, 1e-9), tau = 0.05 -> third index postponed
    F = oracle.factor_lowprec(np.diag([1.0, 0.9, 1e-9]), 0.05)
    assert F.N == 2 and list(F.lam2) == [2] and list(F.lam1) == [0, 1]


def test_ratio_exactly_tau_is_not_postponed():
    # |d1/d0| = 0.5 == tau: strict "<" keeps it
    F = oracle.factor_lowprec(np.diag([1.0, 0.5, 0.25]), 0.5)
    assert F.N == 3


def test_zero_first_pivot_postpones_all():
    F = oracle.factor_lowprec(np.array([[0.0, 1.0], [1.0, 0.0]]), 1e-2)
    assert F.N == 0 and list(F.lam2) == [0, 1]


def test_identity_and_bad_tau():
    F = oracle.factor_lowprec(np.eye(6), 1e-2)
    assert F.N == 6 and list(F.perm) == list(range(6))
    for bad in (0.0, 1.0, -1.0):
        with pytest.raises(ValueError):
            oracle.factor_lowprec(np.eye(3), bad)


def test_floor_and_enlargement_move_last_pivots():
    K = _scaled(30, 11)
    F0 = oracle.factor_lowprec(K, 1e-2)
    assert F0.N == F0.Ntau == 30
    F1 = oracle.factor_lowprec(K, 1e-2, n_min=3)           # [R5]
    assert F1.N == 27 and list(F1.lam1) == list(F0.perm[:27])
    assert list(F1.lam2) == sorted(F0.perm[27:])
    F2 = oracle.factor_lowprec(K, 1e-2, n_min=3, n_extra=2)  # [R9] P:82
    assert F2.N == 25 and np.array_equal(F2.Lfac, F0.Lfac[:25, :25])
    F3 = oracle.factor_lowprec(K, 1e-2, n_extra=4)          # nothing postponed: no enlargement
    assert F3.N == 30


def _lfull(F):
    return F.Lfac.astype(np.float64), F.D.astype(np.float64)


@pytest.mark.parametrize("name,seed", [("C0", 0), ("C0", 1), ("N32", 0), ("S24", 0), ("P512", 0)])
def test_reconstruction_and_ratio_guarantee(name, seed):
    spec = hi.CONFIGS[name]
    K, _ = oracle.scale(hi.make_kbar(name, seed).numpy())
    F = oracle.factor_lowprec(K, spec.tau, n_min=spec.n_min)
    Lf, D = _lfull(F)
    K11 = K[np.ix_(F.lam1, F.lam1)]
    err = np.abs(Lf @ np.diag(D) @ Lf.T - K11).max()
    # SPEC invariant: within 50 N eps32 ||K11|| entrywise
    assert err <= 50 * F.N * np.finfo(np.float32).eps * np.abs(K11).max()
    # ratio guarantee: accepted consecutive pivots satisfy |d_k| >= tau |d_{k-1}|
    d = np.abs(F.D.astype(np.float64))
    assert np.all(d[1:] >= spec.tau * d[:-1])
    assert np.all(np.abs(F.Lfac[np.triu_indices(F.N, 1)]) == 0)


@pytest.mark.parametrize("seed", range(3))
def test_pivot_is_fp64_schur_argmax_on_separated_input(seed):
    """Each FP32 pivot is, to FP32 accuracy, the max |diagonal| of the exact
    (FP64) Schur complement at its step, computed independently."""
    rng = np.random.default_rng(100 + seed)
    n = 40
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = rng.uniform(1.0, 4.0, n) * rng.choice([-1, 1], n)
    K, _ = oracle.scale(Q @ np.diag(lam) @ Q.T)
    K = np.tril(K) + np.tril(K, -1).T
    F = oracle.factor_lowprec(K, 1e-3)
    assert F.N == n
    S = K.copy()
    idx = list(range(n))
    for k in range(n):
        dg = np.abs(np.diag(S))
        p = idx.index(F.perm[k])
        assert dg[p] >= dg.max() * (1 - 1e-4)
        assert abs(S[p, p] - F.D[k]) <= 1e-4 * dg.max()
        c = S[:, p].copy()
        S = S - np.outer(c, c) / S[p, p]
        keep = [i for i in range(len(idx)) if i != p]
        S = S[np.ix_(keep, keep)]
        idx = [idx[i] for i in keep]


def test_planted_count_fp64_and_fp32_small():
    """|Lambda_2| equals the planted number of near-singular directions where
    the precision resolves the gap (north_star)."""
    for seed in range(4):
        K, _ = oracle.scale(hi.make_kbar("P64", seed).numpy())
        assert oracle.factor_lowprec(K, 1e-2, prec="f64").Ntau == 62
        assert oracle.factor_lowprec(K, 1e-2, prec="f32").Ntau == 62
    for seed in range(3):
        K, _ = oracle.scale(hi.make_kbar("C0", seed).numpy())
        assert oracle.factor_lowprec(K, 1e-2, prec="f64").Ntau == 252


def test_neumann_postpones_one_per_inclusion_and_one_bulk():
    spec = hi.CONFIGS["N32"]
    K, _ = oracle.scale(hi.make_kbar("N32", 0).numpy())
    F = oracle.factor_lowprec(K, 1e-2)
    boxes = hi.configs._inclusions(spec, 0)
    n, s = spec.grid, spec.incl_size

    def which(i):
        y, x = divmod(int(i), n)
        for b, (x0, y0) in enumerate(boxes):
            if x0 <= x < x0 + s and y0 <= y < y0 + s:
                return b
        return -1

    owners = sorted(which(i) for i in F.lam2)
    assert owners == [-1, 0, 1, 2]


def test_determinism():
    K, _ = oracle.scale(hi.make_kbar("P512", 1).numpy())
    a = oracle.factor_lowprec(K, 1e-2)
    b = oracle.factor_lowprec(K, 1e-2)
    assert np.array_equal(a.perm, b.perm) and np.array_equal(a.D, b.D)
    assert np.array_equal(a.Lfac, b.Lfac)


def test_prefix_run_equals_full_run_columns():
    """factor_lowprec_prefix (the bounded run used for the C4 prefix parity test)
    returns the same pivots, D and factor columns as the full run, for every
    row: map the prefix run's positions to the full run's pivot order."""
    Kb = hi.make_kbar("C0", 3)
    K, _ = oracle.scale(Kb.numpy())
    full = oracle.factor_lowprec(K, 1e-2, n_min=4)
    k = 40
    pre = oracle.factor_lowprec_prefix(K, 1e-2, k, n_min=4)
    assert np.array_equal(pre.pivots, full.perm[:k])
    assert np.array_equal(pre.D, full.D[:k])
    rank = np.full(K.shape[0], -1)
    rank[full.perm[:full.N]] = np.arange(full.N)
    rows = rank[pre.pos_orig]
    ok = rows >= 0
    assert np.array_equal(pre.Lcols[ok], full.Lfac[rows[ok], :k])
    assert sorted(pre.pos_orig.tolist()) == list(range(K.shape[0]))
