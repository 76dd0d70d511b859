"""Randomised shapes through the whole C ABI (-m gpu): orders 3-6, non-equidimensional mode sizes
(2..37, so K tails and ragged 128-row tiles occur), ranks 1..40 (at most half the rank any Γ can
have, so the normal equations stay SPD), both TTM
engines and both reduce paths of the 1-D grid.  Per case: two MSDT sweeps, one DT sweep (each
state-synchronised with the oracle's exact sweep, fitness and every M^(n) at 1e-10), pp_init and
two approximated sweeps (state-synchronised, the oracle's Eqs. 4-8), each MTTKRP against the oracle.
Seeded, so a failure reproduces."""
import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def cpd():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2010_12056_b200 as pkg
    from paper_2010_12056_b200 import build
    build.build()
    pkg.load_library()
    return pkg


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def case(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(3, 7))
    budget = 60000  # elements, so the oracle stays fast
    dims = []
    for n in range(N):
        hi = max(2, int(round((budget / max(1, np.prod(dims) if dims else 1)) ** (1.0 / (N - n)))))
        dims.append(int(rng.integers(2, max(2, min(37, hi)) + 1)))
    rmax = min(int(np.prod(dims)) // max(dims) // 2, 40)   # rank of Γ^(n) <= prod of the other sizes
    R = int(rng.integers(1, max(1, rmax) + 1))
    return N, tuple(dims), R, int(rng.integers(0, 2))


@pytest.mark.parametrize("seed", range(16))
def test_random_shape_schedule(cpd, seed):
    N, dims, R, impl = case(seed)
    cfg = synth.custom(N, 0, R, noise_var=1e-3, seed=300 + seed, dims=dims)
    To = O.make_tensor(cfg)
    if O.norm2(To) == 0.0:
        pytest.skip("zero tensor")
    nt2 = O.norm2(To)
    T = torch.from_numpy(np.ascontiguousarray(To)).cuda()
    A = synth.init_factors(cfg)
    m = cpd.cp_als_init(T, cfg.shape, R, A, ttm_impl=impl)
    try:
        for sweep in (m.msdt_sweep, m.msdt_sweep, m.dt_sweep):
            f = sweep()
            A1 = [m.get_factor(n) for n in range(N)]
            for n in range(N):
                cur = A1[:n] + A[n:]
                ref = O.mttkrp(To, cur, n)
                assert rel(m.get_last_mttkrp(n), ref) <= TOL, (sweep.__name__, n, dims, R)
            out = O.als_sweep(To, A, nt2)
            G = O.gamma([O.gram(a) for a in out["A"][:-1] + [A1[-1]]], N - 1)
            if np.linalg.cond(G) < 1e6:  # fitness parity where the solves are well conditioned (R19)
                assert abs(f - out["f"]) <= 1e-9 * max(1.0, abs(out["f"])), (sweep.__name__, f, out["f"], dims, R)
            A = A1
        m.pp_init()
        st = O.pp_init(To, A)
        for _ in range(2):
            m.pp_approx_sweep()
            A1 = [m.get_factor(n) for n in range(N)]
            for n in range(N):
                cur = A1[:n] + A[n:]
                # M~^(n) at the GPU's current factors, through the oracle's first/second-order terms
                dA = [c - p for c, p in zip(cur, st.Ap)]
                S = [O.gram(c) for c in cur]
                ref = O.pp_first_order(st, dA, n) + cur[n] @ O.pp_second_order(cur, dA, S, n)
                assert rel(m.get_last_mttkrp(n), ref) <= TOL, ("pp", n, dims, R)
            A = A1
    finally:
        m.close()


@pytest.mark.parametrize("seed", range(16, 32))
def test_random_shape_fused_levels(cpd, seed):
    """Upper-level fusion (msdt_levels) on random shapes: a random l in [2, N-2] (orders 4-6),
    N - l + 1 MSDT sweeps (a full cycle of roots and the start of the next), every M^(n) against the
    oracle's direct MTTKRP at the GPU's current factors."""
    N, dims, R, impl = case(seed)
    if N < 4:
        N, dims = 4, dims + (3,) * (4 - len(dims))
    cfg = synth.custom(N, 0, R, noise_var=1e-3, seed=500 + seed, dims=dims)
    To = O.make_tensor(cfg)
    if O.norm2(To) == 0.0:
        pytest.skip("zero tensor")
    l = int(np.random.default_rng(seed).integers(2, N - 1))
    T = torch.from_numpy(np.ascontiguousarray(To)).cuda()
    A = synth.init_factors(cfg)
    m = cpd.cp_als_init(T, cfg.shape, R, A, ttm_impl=impl, msdt_levels=l)
    try:
        for _ in range(N - l + 1):
            m.msdt_sweep()
            A1 = [m.get_factor(n) for n in range(N)]
            for n in range(N):
                ref = O.mttkrp(To, A1[:n] + A[n:], n)
                assert rel(m.get_last_mttkrp(n), ref) <= TOL, (n, dims, R, l)
            A = A1
    finally:
        m.close()
