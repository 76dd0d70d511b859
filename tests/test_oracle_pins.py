"""Pins for the CPU oracle (-m "not gpu").

Each test ties an oracle function to something other than itself: a
brute-force loop, a closed form, a worked example fixed by the paper's
definitions (tests/golden/spec_examples.json), or an invariant the paper
states.  Chosen so that a dropped term, a wrong sign/index or a transposed
operand in oracle/cpals.py fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rnd(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def brute_mttkrp(T, A, n):
    """Σ over all index tuples of T(i) Π_{m≠n} A^(m)(i_m, r) (P:168-175 elementwise)."""
    R = A[0].shape[1]
    M = np.zeros((T.shape[n], R))
    for idx in itertools.product(*[range(s) for s in T.shape]):
        for r in range(R):
            p = T[idx]
            for m, i in enumerate(idx):
                if m != n:
                    p *= A[m][i, r]
            M[idx[n], r] += p
    return M


# --------------------------- worked examples --------------------------------

def test_golden_khatri_rao():
    g = GOLD["khatri_rao"]
    out = O.khatri_rao([np.array(g["A"], float), np.array(g["B"], float)])
    assert np.array_equal(out, np.array(g["expect"], float))


def test_golden_multi_ttv():
    M = np.zeros((2, 2, 2))
    for a, b, r in itertools.product(range(2), repeat=3):
        M[a, b, r] = (a + 1) + (b + 1) + (r + 1)
    v = np.array([[1.0, 1.0], [2.0, 2.0]])          # v(b, r) = b (1-based)
    out = O.mttv(M, v, 1)
    assert np.array_equal(out, np.array(GOLD["multi_ttv"]["expect"], float))


def test_golden_mttkrp_all_ones_and_gram_hadamard():
    T = np.ones((2, 2, 2))
    A = [np.ones((2, 1))] * 3
    assert np.array_equal(O.mttkrp(T, A, 0), np.array(GOLD["mttkrp_all_ones"]["expect"], float))
    for c in GOLD["gram"]["cases"]:
        assert np.array_equal(O.gram(np.array(c["A"], float)), np.array(c["expect"], float))
    h = GOLD["hadamard"]
    G = O.gamma([np.array(h["A"], float), np.eye(2) * 0 + 7, np.array(h["B"], float)], 1)
    assert np.array_equal(G, np.array(h["expect"], float))


def test_golden_generalized_unfolding_defines_pair_operator():
    """The paper's unfolding T_(1,3)(j,l,k+(m-1)s_2) times A^(4) ⊙ A^(2) is
    Eq. 4's M^(1,3); the oracle's pair operator (a=0,b=2) must equal it elementwise."""
    s = GOLD["generalized_unfolding"]["shape"]
    T = rnd(s, 1)
    A = [rnd((n, 3), 10 + i) for i, n in enumerate(s)]
    U = np.zeros((s[0], s[2], s[1] * s[3]))
    for j, k, l, m in itertools.product(*[range(n) for n in s]):
        U[j, l, k + m * s[1]] = T[j, k, l, m]       # 0-based form of k+(m-1)s_2
    # Kolda KRP A^(4) ⊙ A^(2): row (i4 * s2 + i2), second operand fastest
    P = np.stack([np.kron(A[3][:, r], A[1][:, r]) for r in range(3)], axis=1)
    ref = np.einsum("jlc,cr->jlr", U, P)
    st = O.pp_init(T, A)
    assert np.abs(st.ops[(0, 2)] - ref).max() <= 1e-12 * np.abs(ref).max()


def test_golden_splitmix64():
    g = GOLD["splitmix64"]
    with np.errstate(over="ignore"):
        out = [int(synth._splitmix64(np.uint64(g["seed"]) + np.uint64(k) * synth.GOLDEN)) for k in range(5)]
    assert out == [int(x) for x in g["expect"]]


# --------------------------- MTTKRP definition -----------------------------

@pytest.mark.parametrize("shape,R", [((5, 4, 6), 3), ((3, 4, 2, 3), 2), ((3, 2, 3, 2, 3), 2), ((2, 3, 4), 1)])
def test_mttkrp_bruteforce(shape, R):
    T = rnd(shape, 2)
    A = [rnd((s, R), 20 + i) for i, s in enumerate(shape)]
    for n in range(len(shape)):
        ref = brute_mttkrp(T, A, n)
        assert np.abs(O.mttkrp(T, A, n) - ref).max() <= 1e-12 * np.abs(ref).max()


def test_mttkrp_blocked_krp_equals_unblocked():
    T = rnd((7, 6, 5), 3)
    A = [rnd((s, 4), 30 + i) for i, s in enumerate(T.shape)]
    for n in range(3):
        a, b = O.mttkrp(T, A, n), O.mttkrp(T, A, n, block_rows=2)
        assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


@pytest.mark.parametrize("N,s", [(3, 4), (4, 3), (5, 2)])
def test_mttkrp_closed_forms(N, s):
    T = np.ones((s,) * N)
    A = [np.ones((s, 1))] * N
    for n in range(N):
        assert np.all(O.mttkrp(T, A, n) == s ** (N - 1))
    # one-hot factors select a fiber: M^(n)(:,0) = T(0,..,:,..,0)
    T = rnd((s,) * N, 4)
    E = [np.eye(s)[:, :1]] * N
    for n in range(N):
        idx = [0] * N
        idx[n] = slice(None)
        assert np.array_equal(O.mttkrp(T, E, n)[:, 0], T[tuple(idx)])


def test_gamma_is_gram_of_krp():
    """Γ^(n) = P^(n)T P^(n) (Eq. 1 and the normal equations)."""
    A = [rnd((s, 4), 40 + i) for i, s in enumerate((3, 5, 4, 2))]
    S = [O.gram(a) for a in A]
    for n in range(4):
        P = O.khatri_rao([A[m] for m in range(4) if m != n])
        assert np.abs(O.gamma(S, n) - P.T @ P).max() <= 1e-12 * np.abs(P.T @ P).max()


def test_gram_exactly_symmetric():
    S = O.gram(rnd((50, 7), 5))
    assert np.array_equal(S, S.T)


def test_solve_cases():
    M = rnd((9, 4), 6)
    assert np.allclose(O.solve(np.eye(4), M), M, rtol=0, atol=1e-15)
    At = rnd((9, 4), 7)
    B = rnd((20, 4), 8)
    G = B.T @ B
    X = O.solve(G, At @ G)
    assert np.linalg.norm(X - At) <= 1e-10 * np.linalg.norm(At)


# --------------------------- ALS / fitness -----------------------------------

def _cfg_small(seed=7, noise=1e-6, N=3, s=12, R=3):
    return synth.custom(N, s, R, noise_var=noise, seed=seed)


def test_fitness_eq3_equals_eq2():
    cfg = _cfg_small(noise=1e-4)
    T = O.make_tensor(cfg)
    A = synth.init_factors(cfg)
    for _ in range(4):
        out = O.als_sweep(T, A)
        A = out["A"]
        r2 = O.residual_eq2(T, A)
        assert abs(out["r"] - r2) <= 1e-9
    # after an exact solve <M^(N), A^(N)> = <Γ^(N), S^(N)> (derived from the normal equations)
    assert abs(np.sum(out["M"][-1] * A[-1]) - np.sum(out["G"][-1] * out["S"][-1])) <= 1e-9 * np.sum(out["G"][-1] * out["S"][-1])


def test_als_residual_monotone():
    """Each ALS subproblem is solved exactly, so r never increases."""
    cfg = synth.custom(3, 10, 4, noise_var=1e-2, seed=11)
    T = O.make_tensor(cfg)
    A = synth.init_factors(cfg)
    rs = []
    for _ in range(30):
        out = O.als_sweep(T, A)
        A = out["A"]
        rs.append(out["r"])
    assert all(b <= a + 1e-12 for a, b in zip(rs, rs[1:]))


def test_exact_low_rank_recovery():
    """σ = 0, R = true rank: fitness -> 1 (north_star pin)."""
    cfg = synth.custom(3, 8, 2, noise_var=0.0, seed=3)
    T = O.make_tensor(cfg)
    A = synth.init_factors(cfg)
    for _ in range(300):
        out = O.als_sweep(T, A)
        A = out["A"]
    assert out["f"] > 1 - 1e-6


def test_noisy_recovery_floor():
    """Converged r ≈ ||E||/||T|| sqrt(1 - R(Σ s_n - N + 1)/Π s_n): residual projection
    onto the CP manifold of dimension R(Σ s_n - N + 1) (SURVEY §8(c) pins)."""
    cfg = synth.custom(3, 24, 3, noise_var=1e-4, seed=5)
    T = O.make_tensor(cfg)
    E = T - O.kruskal(synth.true_factors(cfg))
    A = synth.init_factors(cfg)
    for _ in range(150):
        A = O.als_sweep(T, A)["A"]
    r = O.residual_eq2(T, A)
    dof = cfg.R * (3 * cfg.s - 3 + 1)
    pred = math.sqrt(O.norm2(E) / O.norm2(T)) * math.sqrt(1 - dof / cfg.s ** 3)
    assert abs(r - pred) <= 0.02 * pred


# --------------------------- dimension trees ---------------------------------

@pytest.mark.parametrize("N,s", [(3, 5), (4, 4), (5, 3), (6, 2)])
def test_msdt_and_dt_equal_direct(N, s):
    """MSDT and DT are exact: equal to the direct MTTKRP under arbitrary
    factor updates between MTTKRPs; TTM counts N per N-1 sweeps vs 2 per sweep."""
    T = rnd((s,) * N, 9)
    rng = np.random.default_rng(1)
    for Model in (O.MSDTModel, O.DTModel):
        A = [rnd((s, 3), 50 + i) for i in range(N)]
        m = Model(T)
        n_sweeps = 2 * (N - 1)
        for t in range(N * n_sweeps):
            n = t % N
            ref = O.mttkrp(T, A, n)
            got = m.next_mttkrp(A)
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
            A[n] = A[n] + rng.standard_normal(A[n].shape)
        expect = N * n_sweeps // (N - 1) if Model is O.MSDTModel else 2 * n_sweeps
        assert m.n_ttm == expect


def test_block_contract_brute_force():
    """block_contract (upper-level fusion) against nested loops over the definition
    Σ_{i_c, c in C} T[i] Π_c A^(c)(i_c, r), for a middle block, a trailing block and a block that wraps
    around from mode N to mode 1; a one-mode block equals the first-level TTM."""
    T = rnd((3, 2, 4, 3), 17)
    A = [rnd((s, 2), 30 + i) for i, s in enumerate(T.shape)]
    for C in ([1, 2], [2, 3], [3, 0], [3, 0, 1], [0, 1, 2]):
        got = O.block_contract(T, A, C)
        kept = [m for m in range(4) if m not in C]
        ref = np.zeros([T.shape[m] for m in kept] + [2])
        for idx in itertools.product(*[range(s) for s in T.shape]):
            for r in range(2):
                w = T[idx]
                for c in C:
                    w *= A[c][idx[c], r]
                ref[tuple(idx[m] for m in kept) + (r,)] += w
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max(), C
    for j in range(4):
        assert np.allclose(O.block_contract(T, A, [j]), O.ttm(T, A[j], j), rtol=1e-14, atol=0)


@pytest.mark.parametrize("N,s,l", [(4, 4, 2), (5, 3, 2), (5, 3, 3), (6, 2, 2), (6, 2, 3), (6, 2, 4)])
def test_msdt_fused_levels_equal_direct(N, s, l):
    """MSDT with the upper l levels combined is still exact: every MTTKRP equals the
    direct one under arbitrary factor updates; N roots per N-l sweeps (the paper's cost
    2N/(N-l) s^N R per sweep: one pass over T per root); each root contracts the l modes that
    follow its served block cyclically, and its largest node keeps N-l modes."""
    T = rnd((s,) * N, 9)
    rng = np.random.default_rng(2)
    A = [rnd((s, 3), 60 + i) for i in range(N)]
    m = O.MSDTModel(T, levels=l)
    n_sweeps = N - l
    for t in range(N * n_sweeps):
        n = t % N
        ref = O.mttkrp(T, A, n)
        got = m.next_mttkrp(A)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (t, n)
        A[n] = A[n] + rng.standard_normal(A[n].shape)
    assert m.n_ttm == N
    for C, served in m.trace:
        assert len(C) == l and len(served) == N - l
        assert sorted(set(C) | set(served)) == list(range(N))
        assert (served[-1] + 1) % N == C[0]
    with pytest.raises(ValueError):
        O.MSDTModel(T, levels=N - 1)


def test_msdt_fig2_schedule_N4():
    """Fig. 2: roots T×4, T×3, T×2, T×1 serving (1,2,3), (4,1,2), (3,4,1), (2,3,4)."""
    T = rnd((2, 2, 2, 2), 1)
    A = [rnd((2, 2), i) for i in range(4)]
    m = O.MSDTModel(T)
    for _ in range(12):
        m.next_mttkrp(A)
    got = [(j + 1, [x + 1 for x in L]) for j, L in m.trace]
    assert got == [(4, [1, 2, 3]), (3, [4, 1, 2]), (2, [3, 4, 1]), (1, [2, 3, 4])]
    assert O.msdt_roots(4, 3) == [3, 2, 1, 0]


# --------------------------- pairwise perturbation ---------------------------

def _pp_setup(N=3, s=6, R=3, seed=0):
    T = rnd((s,) * N, seed)
    A = [rnd((s, R), 100 + i) for i in range(N)]
    return T, A


@pytest.mark.parametrize("N", [3, 4])
def test_pp_zero_perturbation_is_exact(N):
    """dA = 0 -> M~^(n) = M^(n) exactly (Eq. 5 with U = V = 0); the first PP sweep
    after init then equals an exact ALS sweep."""
    T, A = _pp_setup(N=N, s=5)
    st = O.pp_init(T, A)
    for n in range(N):
        assert np.abs(st.Mp[n] - O.mttkrp(T, A, n)).max() <= 1e-12 * np.abs(st.Mp[n]).max()
    out = O.pp_approx_sweep(st, A, O.norm2(T))
    ex = O.als_sweep(T, A)
    # mode 1 sees dA = 0; mode 2 sees only one perturbed factor (exact by multilinearity)
    assert np.linalg.norm(out["M"][0] - ex["M"][0]) <= 1e-12 * np.linalg.norm(ex["M"][0])
    assert np.linalg.norm(out["M"][1] - ex["M"][1]) <= 1e-11 * np.linalg.norm(ex["M"][1])


@pytest.mark.parametrize("N", [3, 4, 5])
def test_pp_single_perturbed_factor_is_exact(N):
    """Only one factor perturbed -> Eq. 6's first-order term is exact (multilinearity)."""
    T, A = _pp_setup(N=N, s=4)
    st = O.pp_init(T, A)
    i = N - 1
    A2 = [a.copy() for a in A]
    A2[i] = A2[i] + 0.3 * rnd(A2[i].shape, 77)
    n = 0
    Mt = st.Mp[n] + np.einsum("xyk,yk->xk", st.ops[(n, i)], A2[i] - A[i])
    ref = O.mttkrp(T, A2, n)
    assert np.abs(Mt - ref).max() <= 1e-12 * np.abs(ref).max()


def _kruskal_exactness_err(N=3, R=3, s=6, delta=0.2):
    """Max over modes of ||M~^(n) - M^(n)|| / ||M^(n)|| for one oracle.pp_approx_sweep with
    T = [[A]] and A_p = A + δG, M^(n) the exact MTTKRP at the factors current when mode n is formed."""
    A = [rnd((s, R), 200 + i) for i in range(N)]
    T = O.kruskal(A)
    Ap = [a + delta * rnd(a.shape, 300 + i) for i, a in enumerate(A)]
    st = O.pp_init(T, Ap)
    out = O.pp_approx_sweep(st, A, O.norm2(T))
    err = 0.0
    for n in range(N):
        cur = out["A"][:n] + A[n:]
        ref = O.mttkrp(T, cur, n)
        err = max(err, np.linalg.norm(out["M"][n] - ref) / np.linalg.norm(ref))
    return err, out, A


def test_pp_order3_kruskal_tensor_is_exact():
    """N=3 and T = [[A]]: the expansion of Eqs. 5-8 is exact for any A_p (second order is the
    highest order in the other two factors), and [[A]] is a fixed point of the exact update, so
    every mode of a whole oracle.pp_approx_sweep reproduces the exact MTTKRP and keeps A.  Pins
    Eq. 7's form, Eq. 8's orientation (a transposed dS fails at ~1e-3) and the presence of V."""
    err, out, A = _kruskal_exactness_err()
    assert err <= 1e-11, err
    for a, b in zip(out["A"], A):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    assert np.linalg.norm(out["V"][0]) > 1e-3 * np.linalg.norm(out["M"][0])   # V is not negligible here
    assert abs(out["rad"]) <= 1e-12 and abs(out["f"] - 1.0) <= 1e-6


def _decay_ratios(N):
    """T ≈ low rank, A_p = true factors, A = A_p + δG: ||M~^(1) - M^(1)|| from oracle.pp_approx_sweep
    (its first mode sees every other factor perturbed) for δ = 0.1, 0.05, 0.025."""
    s, R = 6, 2
    At = [rnd((s, R), 400 + i) for i in range(N)]
    T = O.kruskal(At) + 1e-3 * rnd((s,) * N, 5)
    st = O.pp_init(T, At)
    G = [rnd((s, R), 500 + i) for i in range(N)]
    errs = []
    for d in (0.1, 0.05, 0.025):
        A = [a + d * g for a, g in zip(At, G)]
        out = O.pp_approx_sweep(st, A, O.norm2(T))
        errs.append(np.linalg.norm(out["M"][0] - O.mttkrp(T, A, 0)))
    return errs[0] / errs[1], errs[1] / errs[2]


@pytest.mark.parametrize("N", [3, 4])
def test_pp_error_decay_third_order(N):
    """Halving δ cuts ||M~ - M|| by ≈ 8x: the neglected terms are third order (SPEC S:390 requires
    ≥ 3.5x); a wrong or missing second-order term leaves a second-order error (≈ 4x)."""
    r1, r2 = _decay_ratios(N)
    assert r1 >= 3.5 and r2 >= 3.5
    assert 6.0 <= r2 <= 10.0, (r1, r2)


def test_pp_pins_detect_oracle_mutations(monkeypatch):
    """The two PP pins above fail when the oracle's Eq. 7/8 is wrong: a transposed dS^(i)
    (dA^T A instead of A^T dA) or a dropped V term (W = 0).  The mutations are patched into the
    oracle module itself, so the pins are shown to guard oracle.pp_approx_sweep, not a copy."""
    good_err, _, _ = _kruskal_exactness_err()
    assert good_err <= 1e-11
    mutations = {
        "dS transposed": ("dS_of", lambda a, d: d.T @ a),
        "V = 0": ("pp_second_order", lambda A, dA, S, n: np.zeros_like(S[0])),
    }
    import oracle.cpals as OC
    for name, (attr, fn) in mutations.items():
        with monkeypatch.context() as mp:
            mp.setattr(OC, attr, fn)
            err, _, _ = _kruskal_exactness_err()
            r3 = _decay_ratios(3)
            r4 = _decay_ratios(4)
        assert err > 1e-4, (name, err)
        assert not (6.0 <= r3[1] <= 10.0 and 6.0 <= r4[1] <= 10.0), (name, r3, r4)


def test_pp_controller_eps_zero_is_plain_als():
    """ε -> 0 never activates PP (Alg. 2 line 5), so the trace equals exact ALS."""
    cfg = _cfg_small()
    T = O.make_tensor(cfg)
    A0 = synth.init_factors(cfg)
    _, tr = O.pp_controller_run(T, A0, eps=1e-300, max_sweeps=6)
    A = A0
    fs = []
    for _ in range(6):
        out = O.als_sweep(T, A)
        A = out["A"]
        fs.append(out["f"])
    assert [k for k, _ in tr] == ["regular"] * len(tr)
    assert np.allclose([f for _, f in tr], fs[:len(tr)], rtol=0, atol=1e-14)


def test_pp_controller_enters_and_converges():
    cfg = synth.custom(3, 16, 3, noise_var=1e-6, seed=8)
    T = O.make_tensor(cfg)
    _, tr = O.pp_controller_run(T, synth.init_factors(cfg), eps=0.1, max_sweeps=300)
    kinds = [k for k, _ in tr]
    assert "pp_approx" in kinds
    assert tr[-1][1] > 0.99


# --------------------------- generator ---------------------------------------

def test_collinear_generator():
    A = synth.collinear_factors((64,) * 2, 32, 0.5, 1004)
    for a in A:
        n = np.linalg.norm(a, axis=0)
        assert np.allclose(n, 8.0, rtol=0, atol=1e-12)
        C = (a.T @ a) / np.outer(n, n)
        off = C[~np.eye(32, dtype=bool)]
        assert np.abs(off - 0.5).max() <= 1e-10
    # cond(Γ) at the true C4 factors: Γ = (s^4)·(C^4 11^T + (1-C^4) I) has cond (1+31 C^4)/(1-C^4) = 47/15
    S = [O.gram(a) for a in synth.collinear_factors((64,) * 5, 32, 0.5, 1004)]
    assert abs(np.linalg.cond(O.gamma(S, 0)) - 47 / 15) <= 1e-8


def test_hash_generator_statistics():
    idx = np.arange(200000, dtype=np.uint64)
    u = synth.hash_uniform(5, idx)
    assert 0 <= u.min() and u.max() < 1 and abs(u.mean() - 0.5) < 5e-3
    z = synth.hash_normal(5, idx)
    assert abs(z.mean()) < 1e-2 and abs(z.var() - 1) < 2e-2


def test_tensor_slab_and_slice_consistency():
    cfg = synth.custom(3, 8, 2, noise_var=1e-2, seed=9)
    T = O.make_tensor(cfg)
    parts = [O.make_tensor(cfg, p, 4) for p in range(4)]
    assert np.array_equal(np.concatenate(parts, axis=-1), T)
    assert np.array_equal(O.make_tensor_slice(cfg, 1, 3), T[:, 3, :])
    # noise only: T - [[A_true]] has the requested variance scale
    E = T - O.kruskal(synth.true_factors(cfg))
    assert 0.05 < E.std() < 0.2
    A = synth.init_factors(cfg)
    rows = [0, 5]
    assert np.abs(O.mttkrp_rows(cfg, A, 2, rows) - O.mttkrp(T, A, 2)[rows]).max() <= 1e-12 * np.abs(T).max() * 100


# --------------------------- parallel (1-D grid) simulation -------------------

@pytest.mark.parametrize("P", [2, 4])
def test_parallel_sim_equals_sequential(P):
    """Alg. 3 / Alg. 4 on a 1-D grid equal the sequential sweep up to reduction order."""
    T = rnd((6, 5, 8), 12)
    A = [rnd((s, 3), 600 + i) for i, s in enumerate(T.shape)]
    T6 = rnd((8, 8, 8), 13)
    A6 = [rnd((8, 3), 700 + i) for i in range(3)]
    seq = O.als_sweep(T6, A6)
    par = O.par_als_sweep_sim(T6, A6, P)
    for a, b in zip(seq["A"], par["A"]):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(a)
    assert abs(seq["f"] - par["f"]) <= 1e-10
    st = O.pp_init(T6, A6)
    A2 = [a + 0.05 * rnd(a.shape, 800 + i) for i, a in enumerate(A6)]
    s1 = O.pp_approx_sweep(st, A2, O.norm2(T6))
    s2 = O.par_pp_approx_sweep_sim(T6, st, A2, P, O.norm2(T6))
    for a, b in zip(s1["M"], s2["M"]):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(a)
    del T, A


@pytest.mark.parametrize("N", [3, 4, 5])
def test_pp_rows_equal_full_operators(N):
    """pp_init_rows / pp_approx_rows (row-restricted Eq. 4-8 for full-size checks) equal the rows
    of the full oracle.pp_init / pp_approx_sweep operators and M~ (mode by mode of one sweep)."""
    cfg = synth.custom(N, 5 if N > 3 else 7, 3, noise_var=1e-2, seed=20 + N)
    T = O.make_tensor(cfg)
    Ap = [rnd((cfg.s, 3), 900 + i) for i in range(N)]
    st = O.pp_init(T, Ap)
    A = [a + 0.1 * rnd(a.shape, 950 + i) for i, a in enumerate(Ap)]
    out = O.pp_approx_sweep(st, A, O.norm2(T))
    rows = [1, 3]
    cache = {}
    for n in range(N):
        sr = O.pp_init_rows(cfg, Ap, n, rows, cache)
        for (a, b), op in sr.ops.items():
            full = st.ops[(a, b)]
            ref = full[rows] if a == n else full[:, rows]
            assert np.abs(op - ref).max() <= 1e-12 * np.abs(full).max()
        assert np.abs(sr.Mp[n] - st.Mp[n][rows]).max() <= 1e-12 * np.abs(st.Mp[n]).max()
        cur = out["A"][:n] + A[n:]
        got = O.pp_approx_rows(sr, cur, n, rows)
        assert np.abs(got - out["M"][n][rows]).max() <= 1e-12 * np.abs(out["M"][n]).max()


@pytest.mark.parametrize("grid", [(2, 2, 2), (1, 1, 4), (1, 1, 2), (2, 1, 3), (4, 2, 1)])
def test_grid_sim_equals_sequential(grid):
    """Alg. 3 / Alg. 4 on an N-D processor grid equal the sequential sweep
    up to reduction order; (1, 1, P) is the 1-D grid of par_als_sweep_sim."""
    T = rnd((8, 6, 12), 14)
    A = [rnd((s, 3), 710 + i) for i, s in enumerate(T.shape)]
    seq = O.als_sweep(T, A)
    par = O.par_als_sweep_grid_sim(T, A, grid)
    for a, b in zip(seq["A"], par["A"]):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(a)
    assert abs(seq["f"] - par["f"]) <= 1e-10
    if grid[0] == grid[1] == 1 and all(d % grid[2] == 0 for d in T.shape):
        p1 = O.par_als_sweep_sim(T, A, grid[2])
        assert abs(p1["f"] - par["f"]) <= 1e-12
    st = O.pp_init(T, A)
    A2 = [a + 0.05 * rnd(a.shape, 810 + i) for i, a in enumerate(A)]
    s1 = O.pp_approx_sweep(st, A2, O.norm2(T))
    s2 = O.par_pp_approx_sweep_grid_sim(T, st, A2, grid, O.norm2(T))
    for a, b in zip(s1["M"], s2["M"]):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(a)


def test_grid_sim_order4():
    T = rnd((4, 6, 4, 6), 15)
    A = [rnd((s, 2), 720 + i) for i, s in enumerate(T.shape)]
    seq = O.als_sweep(T, A)
    par = O.par_als_sweep_grid_sim(T, A, (2, 3, 1, 2))
    assert abs(seq["f"] - par["f"]) <= 1e-10
    for a, b in zip(seq["A"], par["A"]):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(a)
