"""Parity of the CUDA path (through the C ABI) with the CPU oracle (-m gpu).

Tolerance (north_star): 1e-10 relative, norm-wise per MTTKRP / factor (reading Q18)
and relative per-sweep fitness.  Inputs: the seeded synth recipe on both sides.
"""
import itertools

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


def dev_tensor(cpd, cfg, rank=0, world=1):
    lo, hi = synth.slab_range(cfg.shape[-1], rank, world)
    shp = list(cfg.shape[:-1]) + [hi - lo]
    T = torch.empty(shp, dtype=torch.float64, device="cuda")
    if cfg.kind == "uniform":
        cpd.cpd_gen_tensor(T, cfg.shape, lo, hi, 1, None, 0.0, cfg.seed_noise)
    else:
        cpd.cpd_gen_tensor(T, cfg.shape, lo, hi, 0, synth.true_factors(cfg), np.sqrt(cfg.noise_var),
                           cfg.seed_noise)
    return T


# ------------------------------- generator -----------------------------------------

@pytest.mark.parametrize("cfg", [synth.config(1), synth.custom(4, 9, 3, seed=2), synth.custom(5, 5, 3, seed=3),
                                 synth.custom(4, 7, 0, kind="uniform", true_rank=0, noise_var=0.0, seed=4),
                                 synth.custom(5, 6, 4, noise_var=1e-3, collinearity=0.5, seed=6)])
def test_generator_matches_oracle(cpd, cfg):
    if cfg.kind == "uniform":
        cfg = synth.Config(**{**cfg.__dict__, "R": 3})
    T = dev_tensor(cpd, cfg).cpu().numpy()
    To = O.make_tensor(cfg)
    assert rel(T, To) <= 1e-14


def test_generator_slabs(cpd):
    cfg = synth.custom(3, 8, 3, noise_var=1e-2, seed=8)
    full = dev_tensor(cpd, cfg).cpu().numpy()
    parts = [dev_tensor(cpd, cfg, p, 4).cpu().numpy() for p in range(4)]
    assert np.array_equal(np.concatenate(parts, axis=-1), full)


# ------------------------------- single kernels --------------------------------------

@pytest.mark.parametrize("shape,R", [((37, 29, 41), 8), ((16, 130, 12), 64), ((33, 20, 17), 13), ((9, 10, 11, 12), 100),
                                     ((11, 7, 13), 200), ((6, 5, 3), 1), ((200, 3, 130), 33), ((5, 300, 4), 17)])
def test_ttm_all_positions(cpd, shape, R):
    rng = np.random.default_rng(sum(shape) + R)
    Tn = rng.standard_normal(shape)
    T = torch.from_numpy(Tn).cuda()
    for j in range(len(shape)):
        A = rng.standard_normal((shape[j], R))
        pre = int(np.prod(shape[:j])) if j else 1
        post = int(np.prod(shape[j + 1:])) if j < len(shape) - 1 else 1
        out = torch.empty((pre * post, R), dtype=torch.float64, device="cuda")
        cpd.cpd_ttm(T, pre, shape[j], post, torch.from_numpy(A).cuda(), R, out)
        ref = O.ttm(Tn, A, j).reshape(pre * post, R)
        assert rel(out.cpu().numpy(), ref) <= 1e-13, (j, rel(out.cpu().numpy(), ref))


@pytest.mark.parametrize("shape,R", [((41, 48, 64), 64), ((41, 48, 50), 100), ((40, 32, 48), 200), ((33, 64, 80), 32),
                                     ((35, 36, 96), 24), ((37, 40, 112), 18), ((9, 16, 10, 32), 100), ((130, 34, 16), 16),
                                     ((3, 70, 128), 128), ((257, 64), 72), ((20, 34, 200), 64), ((6, 40, 72), 100),
                                     ((5, 33, 100), 32), ((3, 4, 36, 66), 200)])
def test_ttm_dmma_tma_staged_shapes(cpd, shape, R):
    """FP64 DMMA engine, TMA-staged tiles (Eq. 4 with one contracted mode): shapes that take the
    swizzled-box path -- even K (last mode), post % 16 == 0 (other modes), even R >= 16 -- with ragged row tiles,
    K tails inside a 16-wide box, tiles that straddle two p, odd fragment counts (R = 24, 100, 200: the unpaired
    last column fragment), R not a multiple of 8 (zero-filled columns), two N tiles (R = 200), post % 16 != 0 (rows padded per p to 16: post = 200, 72, 100, 66)."""
    rng = np.random.default_rng(sum(shape) * 7 + R)
    Tn = rng.standard_normal(shape)
    T = torch.from_numpy(Tn).cuda()
    for j in range(len(shape)):
        A = rng.standard_normal((shape[j], R))
        pre = int(np.prod(shape[:j])) if j else 1
        post = int(np.prod(shape[j + 1:])) if j < len(shape) - 1 else 1
        out = torch.full((pre * post, R), float("nan"), dtype=torch.float64, device="cuda")
        cpd.cpd_ttm(T, pre, shape[j], post, torch.from_numpy(A).cuda(), R, out)
        ref = O.ttm(Tn, A, j).reshape(pre * post, R)
        assert rel(out.cpu().numpy(), ref) <= 1e-13, (j, rel(out.cpu().numpy(), ref))


@pytest.mark.parametrize("shape,R", [((37, 29, 41), 8), ((16, 130), 64), ((33, 20, 17), 13), ((9, 10, 11, 5), 100),
                                     ((3, 1000, 2), 7), ((4, 5), 200)])
def test_mttv_all_axes(cpd, shape, R):
    rng = np.random.default_rng(len(shape) * 7 + R)
    Xn = rng.standard_normal(tuple(shape) + (R,))
    X = torch.from_numpy(Xn).cuda()
    for a in range(len(shape)):
        v = rng.standard_normal((shape[a], R))
        pre = int(np.prod(shape[:a])) if a else 1
        post = int(np.prod(shape[a + 1:])) if a < len(shape) - 1 else 1
        ref = O.mttv(Xn, v, a).reshape(pre, post * R)
        out = torch.zeros((pre, post * R), dtype=torch.float64, device="cuda")
        cpd.cpd_mttv(X, pre, shape[a], post, R, torch.from_numpy(v).cuda(), out, 0)
        assert rel(out.cpu().numpy(), ref) <= 1e-13
        # beta = 1 accumulates
        cpd.cpd_mttv(X, pre, shape[a], post, R, torch.from_numpy(v).cuda(), out, 1)
        assert rel(out.cpu().numpy(), 2 * ref) <= 1e-13


# ------------------------------- sweeps ------------------------------------------------

def _model(cpd, cfg, T, A0=None, **kw):
    return cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg) if A0 is None else A0, **kw)


@pytest.mark.parametrize("ttm_impl", [0, 1])
def test_c1_full_trajectory(cpd, ttm_impl):
    """C1: 10 msdt_sweep, then pp_init + 5 forced pp_approx_sweep (reading Q14); every
    M^(n) and every fitness compared with the oracle (full-trajectory parity); with the
    DMMA and with the INT8 tensor-core TTM."""
    cfg = synth.config(1)
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    nt2 = O.norm2(To)
    m = _model(cpd, cfg, T, ttm_impl=ttm_impl)
    A = synth.init_factors(cfg)
    for sweep in range(10):
        f = m.msdt_sweep()
        out = O.als_sweep(To, A, nt2)
        for n in range(3):
            assert rel(m.get_last_mttkrp(n), out["M"][n]) <= TOL, (sweep, n)
        assert abs(f - out["f"]) <= TOL * abs(out["f"])
        A = out["A"]
    for n in range(3):
        assert rel(m.get_factor(n), A[n]) <= TOL
    m.pp_init()
    st = O.pp_init(To, A)
    for a, b in itertools.combinations(range(3), 2):
        assert rel(m.debug_pp_operator(a, b), st.ops[(a, b)]) <= TOL
    for k in range(5):
        f, valid = m.pp_approx_sweep()
        out = O.pp_approx_sweep(st, A, nt2, eps=0.1)
        for n in range(3):
            assert rel(m.get_last_mttkrp(n), out["M"][n]) <= TOL, (k, n)
        assert abs(f - out["f"]) <= TOL * abs(out["f"])
        assert valid == out["still_valid"]
        A = out["A"]
    m.close()


@pytest.mark.parametrize("early", [1, 2, 3])
def test_c1_early_pp_exercises_second_order(cpd, early):
    """C1-early: pp_init after 1-3 sweeps, 3 forced PP sweeps (||V||/||M|| ~ 1e-2, so a
    wrong Eq. 7/8 fails); state-synchronised: the oracle starts from the GPU factors."""
    cfg = synth.config(1)
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    nt2 = O.norm2(To)
    m = _model(cpd, cfg, T)
    for _ in range(early):
        m.msdt_sweep()
    A = [m.get_factor(n) for n in range(3)]
    m.pp_init()
    st = O.pp_init(To, A)
    vmax = 0.0
    for k in range(3):
        Ag = [m.get_factor(n) for n in range(3)]
        f, _ = m.pp_approx_sweep()
        out = O.pp_approx_sweep(st, Ag, nt2)
        for n in range(3):
            assert rel(m.get_last_mttkrp(n), out["M"][n]) <= TOL, (k, n)
            vmax = max(vmax, np.linalg.norm(out["V"][n]) / np.linalg.norm(out["M"][n]))
        assert abs(f - out["f"]) <= TOL * abs(out["f"])
    assert vmax > 1e-4  # the second-order term is really exercised
    m.close()


@pytest.mark.parametrize("ttm_impl", [0, 1])
@pytest.mark.parametrize("N,s,R", [(4, 12, 5), (5, 6, 3), (3, 40, 24), (6, 4, 2), (4, 72, 6), (7, 3, 2), (8, 3, 3),
                                   (3, 56, 64)])
def test_msdt_and_dt_sweeps_order_N(cpd, N, s, R, ttm_impl):
    cfg = synth.custom(N, s, R, noise_var=1e-4, seed=N * 10 + s)
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    nt2 = O.norm2(To)
    for kind in ("msdt", "dt"):
        m = _model(cpd, cfg, T, ttm_impl=ttm_impl)
        A = synth.init_factors(cfg)
        for sweep in range(2 * (N - 1)):
            f = m.msdt_sweep() if kind == "msdt" else m.dt_sweep()
            out = O.als_sweep(To, A, nt2)
            for n in range(N):
                assert rel(m.get_last_mttkrp(n), out["M"][n]) <= TOL, (kind, sweep, n)
            assert abs(f - out["f"]) <= TOL * abs(out["f"])
            A = [m.get_factor(n) for n in range(N)]  # state-synchronised
        c = m.counters()
        roots = c["roots"]
        if kind == "msdt":
            assert roots == N * 2
        else:
            assert roots == 2 * 2 * (N - 1)
        m.close()


@pytest.mark.parametrize("ttm_impl", [0, 1])
@pytest.mark.parametrize("dims,R,l", [((6, 7, 5, 9), 5, 2), ((5, 4, 6, 3, 7), 4, 2), ((5, 4, 6, 3, 7), 4, 3),
                                      ((3, 4, 2, 3, 5, 4), 3, 2), ((3, 4, 2, 3, 5, 4), 3, 4), ((4, 4, 130, 130), 3, 2),
                                      ((130, 3, 2, 3, 130), 3, 2), ((2, 130, 130, 2, 64), 3, 2), ((20, 12, 16, 32), 50, 2)])
def test_msdt_fused_levels(cpd, dims, R, l, ttm_impl):
    """Upper-level fusion (opts.msdt_levels = l): every root contracts a cyclic block of l
    modes in one pass over T with the Khatri-Rao product of their factors.  N - l state-synchronised
    MSDT sweeps (one full cycle: N roots) against the oracle's ALS sweep (explicit unfolding and KRP),
    every M^(n) and the fitness at 1e-10.  The shapes exercise middle, trailing and wrapping blocks,
    padded innermost modes (w = 5, 7, 9, 130), K chunks on the digit planes (a trailing block of
    130 x 144 padded K rows, a middle block of K = 16900, a wrapping block of 130 slabs of 160 K rows)
    and 56-column N tiles (R = 50)."""
    cfg = synth.custom(len(dims), 0, R, noise_var=1e-4, seed=sum(dims) % 89 + l, dims=dims)
    N = cfg.N
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    nt2 = O.norm2(To)
    m = _model(cpd, cfg, T, ttm_impl=ttm_impl, msdt_levels=l)
    A = synth.init_factors(cfg)
    for sweep in range(N - l):
        f = m.msdt_sweep()
        out = O.als_sweep(To, A, nt2)
        for n in range(N):
            assert rel(m.get_last_mttkrp(n), out["M"][n]) <= TOL, (sweep, n, rel(m.get_last_mttkrp(n), out["M"][n]))
        assert abs(f - out["f"]) <= TOL * abs(out["f"])
        A = [m.get_factor(n) for n in range(N)]
    assert m.counters()["roots"] == N
    m.close()


@pytest.mark.parametrize("N,s,R", [(5, 8, 4), (6, 6, 3)])
def test_msdt_fused_levels_memory(cpd, N, s, R):
    """The trade-off of P:700-702: with the upper l levels combined the largest tree node holds
    s^(N-l) R elements, so cpd_get_memory's high-water mark falls with l (l <= N/2: beyond that the
    block's Khatri-Rao product, s^l R, is the larger buffer), for N/(N-l) passes over T per sweep (the
    roots ledger: N roots in N - l sweeps); the fitness equals the l = 1 run's at 1e-10."""
    cfg = synth.custom(N, s, R, noise_var=1e-4, seed=N + s)
    T = dev_tensor(cpd, cfg)
    peaks = []
    for l in range(1, N // 2 + 1):
        m = _model(cpd, cfg, T, msdt_levels=l)
        fl = [m.msdt_sweep() for _ in range(N - l)]
        peaks.append(m.get_memory()["peak"])
        assert m.counters()["roots"] == N
        m.close()
        m1 = _model(cpd, cfg, T)
        f1 = [m1.msdt_sweep() for _ in range(N - l)]
        assert abs(fl[-1] - f1[-1]) <= TOL * abs(f1[-1])
        m1.close()
    assert all(b < a for a, b in zip(peaks, peaks[1:])), peaks


@pytest.mark.parametrize("N,s,R", [(4, 10, 4), (5, 6, 3), (6, 4, 2), (8, 3, 2), (3, 48, 64), (4, 20, 128)])
def test_pp_order_N_state_synchronised(cpd, N, s, R):
    cfg = synth.custom(N, s, R, noise_var=1e-3, seed=N + 40)
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    nt2 = O.norm2(To)
    m = _model(cpd, cfg, T)
    for _ in range(2):
        m.msdt_sweep()
    A = [m.get_factor(n) for n in range(N)]
    m.pp_init()
    st = O.pp_init(To, A)
    for a, b in itertools.combinations(range(N), 2):
        assert rel(m.debug_pp_operator(a, b), st.ops[(a, b)]) <= TOL, (a, b)
    for k in range(3):
        Ag = [m.get_factor(n) for n in range(N)]
        f, _ = m.pp_approx_sweep()
        out = O.pp_approx_sweep(st, Ag, nt2)
        for n in range(N):
            assert rel(m.get_last_mttkrp(n), out["M"][n]) <= TOL, (k, n)
        assert abs(f - out["f"]) <= TOL * abs(out["f"])
    # back to a regular sweep after PP restarts the MSDT cycle and stays exact
    Ag = [m.get_factor(n) for n in range(N)]
    f = m.msdt_sweep()
    out = O.als_sweep(To, Ag, nt2)
    assert abs(f - out["f"]) <= TOL * abs(out["f"])
    m.close()


def test_pp_zero_perturbation_equals_exact(cpd):
    """First mode of the first PP sweep sees dA = 0: M~^(1) = M^(1) at A_p exactly (Eq. 5)."""
    cfg = synth.custom(3, 20, 4, noise_var=1e-4, seed=77)
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    m = _model(cpd, cfg, T)
    m.msdt_sweep()
    A = [m.get_factor(n) for n in range(3)]
    m.pp_init()
    m.pp_approx_sweep()
    assert rel(m.get_last_mttkrp(0), O.mttkrp(To, A, 0)) <= TOL
    m.close()


def test_pp_root_reuse_changes_only_rounding(cpd):
    cfg = synth.custom(4, 10, 4, noise_var=1e-3, seed=91)
    T = dev_tensor(cpd, cfg)
    res = []
    for reuse in (True, False):
        m = _model(cpd, cfg, T, reuse_root_in_pp_init=reuse)
        m.msdt_sweep()
        m.pp_init()
        c = m.counters()
        f, _ = m.pp_approx_sweep()
        res.append((f, c["roots"]))
        m.close()
    assert abs(res[0][0] - res[1][0]) <= TOL
    assert res[0][1] == res[1][1] - 1   # one first-level TTM saved (P:384 footnote)


def test_errors(cpd):
    cfg = synth.custom(3, 8, 3, seed=5)
    T = dev_tensor(cpd, cfg)
    m = _model(cpd, cfg, T)
    with pytest.raises(cpd.CPDError) as e:
        m.pp_approx_sweep()
    assert e.value.status == 2
    with pytest.raises(cpd.CPDError) as e:
        m.get_factor(7, out=np.empty((8, 3)))
    assert e.value.status == 1
    m.close()
    with pytest.raises(cpd.CPDError) as e:
        cpd.cp_als_init(T, cfg.shape, cpd.CPD_MAX_RANK + 1, synth.init_factors(cfg))
    assert e.value.status == 1
    # rank-deficient factors -> Γ not SPD
    A0 = synth.init_factors(cfg)
    A0 = [a.copy() for a in A0]
    A0[1][:, 1] = 0.0
    A0[2][:, 1] = 0.0
    m = _model(cpd, cfg, T, A0=A0)
    with pytest.raises(cpd.CPDError) as e:
        m.msdt_sweep()
    assert e.value.status == 3
    m.close()


def test_set_factors_restarts_cycle(cpd):
    cfg = synth.custom(3, 16, 4, noise_var=1e-4, seed=12)
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    m = _model(cpd, cfg, T)
    m.msdt_sweep()
    A = [a + 0.01 for a in synth.init_factors(cfg)]
    m.set_factors(A)
    f = m.msdt_sweep()
    out = O.als_sweep(To, A)
    assert abs(f - out["f"]) <= TOL * abs(out["f"])
    m.close()


# ------------------------------- full-size sampled checks --------------------------------

@pytest.mark.parametrize("ttm_impl", [0, 1])
@pytest.mark.parametrize("c", [2, 3, 4, 5])
def test_full_size_sampled_rows(cpd, c, ttm_impl):
    """BASELINE configs at full size: one msdt_sweep and one dt_sweep; sampled rows of every M^(n)
    against the oracle's slice-by-slice explicit-KRP rows with the GPU's input factors."""
    cfg = synth.config(c)
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info()
    # T (8 B/element) + the int8 engine's digit planes (7 B/element) + two live tree nodes of
    # root size (8 B x numel/s x R) + workspaces; every ctx returns its memory at close
    need = 8 * cfg.numel + (7 * cfg.numel if ttm_impl == 1 else 0) + 2 * 8 * cfg.numel // cfg.s * cfg.R + 4e9
    assert need < total, "config does not fit one B200"
    if free < need:
        pytest.skip(f"not enough free device memory ({free / 1e9:.1f} GB < {need / 1e9:.1f} GB)")
    T = dev_tensor(cpd, cfg)
    m = _model(cpd, cfg, T, ttm_impl=ttm_impl)
    A0 = synth.init_factors(cfg)
    rng = np.random.default_rng(c)
    # one MSDT sweep, then one standard-DT sweep (Fig. 1a) from the MSDT sweep's factors
    for sweep in (m.msdt_sweep, m.dt_sweep):
        sweep()
        A1 = [m.get_factor(n) for n in range(cfg.N)]
        for n in range(cfg.N):
            Ause = A1[:n] + A0[n:]   # modes < n already updated in this sweep
            rows = rng.choice(cfg.s, 2 if c == 5 else 3, replace=False)
            ref = O.mttkrp_rows(cfg, Ause, n, rows)
            got = m.get_last_mttkrp(n)[rows]
            assert rel(got, ref) <= TOL, (sweep.__name__, n, rel(got, ref))
        A0 = A1
    m.close()
    del T
    torch.cuda.empty_cache()


@pytest.mark.parametrize("c", [3, 4])
def test_full_size_fused_levels_sampled_rows(cpd, c):
    """Upper-level fusion at full size, in the launch configuration `bench.py --msdt-levels 2` times (C3:
    block roots of K = 200 x 208 padded rows in 3 K chunks; C4: K = 4096, a wrapping block): one full MSDT
    cycle (N roots in N - 2 sweeps), sampled rows of every M^(n) against the oracle's explicit-KRP rows with
    the GPU's input factors."""
    cfg = synth.config(c)
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info()
    need = 15 * cfg.numel + 4e9   # T + digit planes + (small) block roots and workspaces
    if free < need:
        pytest.skip(f"not enough free device memory ({free / 1e9:.1f} GB < {need / 1e9:.1f} GB)")
    T = dev_tensor(cpd, cfg)
    m = _model(cpd, cfg, T, msdt_levels=2)
    A0 = synth.init_factors(cfg)
    rng = np.random.default_rng(c + 10)
    for _ in range(cfg.N - 2):
        m.msdt_sweep()
        A1 = [m.get_factor(n) for n in range(cfg.N)]
        for n in range(cfg.N):
            rows = rng.choice(cfg.s, 3, replace=False)
            ref = O.mttkrp_rows(cfg, A1[:n] + A0[n:], n, rows)
            got = m.get_last_mttkrp(n)[rows]
            assert rel(got, ref) <= TOL, (n, rel(got, ref))
        A0 = A1
    assert m.counters()["roots"] == cfg.N
    m.close()
    del T
    torch.cuda.empty_cache()


# ------------------------------- INT8 tensor-core TTM -----------------------------------

@pytest.mark.parametrize("digits", [True, False])
@pytest.mark.parametrize("shape,R", [((37, 29, 41), 8), ((16, 130, 12), 64), ((33, 20, 17), 13), ((9, 10, 11, 12), 100),
                                     ((11, 7, 13), 200), ((6, 5, 3), 1), ((200, 3, 130), 33), ((5, 300, 4), 17),
                                     ((64, 64, 64), 64), ((40, 33, 257), 32), ((3, 256, 128), 48), ((130, 48, 256), 64),
                                     ((64, 64, 64), 32), ((12, 48, 32), 16), ((6, 8, 64, 64), 24),
                                     ((9, 30, 200), 64), ((5, 7, 6, 100), 40), ((3, 130, 72), 20),
                                     ((4, 8, 200), 20), ((3, 16, 24), 12), ((2, 16, 8, 200), 100),
                                     ((7, 9, 5, 24), 50), ((20, 6, 16), 80), ((8, 16, 56), 56), ((4, 9, 208), 200)])
def test_ttm_i8_all_positions(cpd, shape, R, digits):
    """cpd_ttm_i8 (int8 digit slicing on tcgen05) against the oracle's T x_j A at every
    contraction position: ragged M tiles, K tails (odd K, K % 32 != 0), 1-4 N tiles, N tiles
    padded to 16 columns and to 8 (Rp = 40, 56: the zero rows after the last plane)."""
    rng = np.random.default_rng(sum(shape) + R + 1)
    Tn = rng.standard_normal(shape)
    T = torch.from_numpy(Tn).cuda()
    for j in range(len(shape)):
        A = rng.standard_normal((shape[j], R))
        pre = int(np.prod(shape[:j])) if j else 1
        post = int(np.prod(shape[j + 1:])) if j < len(shape) - 1 else 1
        out = torch.empty((pre * post, R), dtype=torch.float64, device="cuda")
        cpd.cpd_ttm_i8(T, pre, shape[j], post, torch.from_numpy(A).cuda(), R, out, use_digits=digits)
        ref = O.ttm(Tn, A, j).reshape(pre * post, R)
        assert rel(out.cpu().numpy(), ref) <= 1e-13, (j, rel(out.cpu().numpy(), ref))


def test_ttm_i8_wide_dynamic_range(cpd):
    """Entries spread over 12 orders of magnitude and column scales over 6: the error is
    relative to max|T| (one tensor exponent), so the norm-wise bound still holds."""
    rng = np.random.default_rng(7)
    shape = (48, 40, 36)
    Tn = rng.standard_normal(shape) * 10.0 ** rng.uniform(-12, 0, shape)
    T = torch.from_numpy(Tn).cuda()
    for j in range(3):
        A = rng.standard_normal((shape[j], 24)) * 10.0 ** rng.uniform(-3, 3, (1, 24))
        pre = int(np.prod(shape[:j])) if j else 1
        post = int(np.prod(shape[j + 1:])) if j < 2 else 1
        out = torch.empty((pre * post, 24), dtype=torch.float64, device="cuda")
        cpd.cpd_ttm_i8(T, pre, shape[j], post, torch.from_numpy(A).cuda(), 24, out)
        ref = O.ttm(Tn, A, j).reshape(pre * post, 24)
        got = out.cpu().numpy()
        for c in range(24):  # per column (columns have different scales)
            assert rel(got[:, c], ref[:, c]) <= 1e-12, (j, c, rel(got[:, c], ref[:, c]))


def test_ttm_engine_auto_selection(cpd):
    """CPD_TTM_AUTO: the int8 digit engine when max|T| <= 256 rms(T) (its error bound is then
    FP64-class), the DMMA engine for a tensor with a wide dynamic range; both match the oracle."""
    cfg = synth.custom(3, 48, 4, noise_var=1e-4, seed=77)
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    m = _model(cpd, cfg, T)
    assert m.ttm_engine() == "int8-digits"
    m.close()
    m = _model(cpd, cfg, T, ttm_impl=0)
    assert m.ttm_engine() == "dmma"
    m.close()
    # one huge entry: max|T| / rms(T) -> sqrt(48^3) = 333 > 256 -> DMMA
    Tw = T.clone()
    Tw.view(-1)[5] = 1e6
    Tow = Tw.cpu().numpy()
    m = _model(cpd, cfg, Tw)
    assert m.ttm_engine() == "dmma"
    f = m.msdt_sweep()
    out = O.als_sweep(Tow, synth.init_factors(cfg))
    assert abs(f - out["f"]) <= TOL * abs(out["f"])
    m.close()
    m = _model(cpd, cfg, Tw, ttm_impl=1)  # forced int8 still runs (norm-wise bound relative to max|T|)
    assert m.ttm_engine() == "int8-digits"
    m.close()


@pytest.mark.parametrize("ttm_impl", [0, 2])
def test_set_tensor_new_contents(cpd, ttm_impl):
    """cpd_set_tensor: new contents in the same buffer -> ||T||^2, exponent and digit planes
    recomputed, caches dropped; the next sweeps match the oracle on the new tensor."""
    c1 = synth.custom(3, 40, 5, noise_var=1e-4, seed=91)
    c2 = synth.custom(3, 40, 5, noise_var=1e-4, seed=92)
    T = dev_tensor(cpd, c1)
    m = _model(cpd, c1, T, ttm_impl=ttm_impl)
    m.msdt_sweep()
    m.msdt_sweep()
    T.copy_(dev_tensor(cpd, c2))
    m.set_tensor()
    A = synth.init_factors(c2)
    m.set_factors(A)
    To2 = O.make_tensor(c2)
    nt2 = O.norm2(To2)
    for _ in range(3):
        f = m.msdt_sweep()
        out = O.als_sweep(To2, A, nt2)
        assert abs(f - out["f"]) <= TOL * abs(out["f"])
        A = out["A"]
    m.close()


def test_caller_stream_ordering(cpd):
    """opts.stream semantics (cpd.h): the library runs on its own streams, ordered after the work
    already enqueued on the caller's stream.  The new tensor contents are written on a caller
    stream behind a ~1 ms spin and cpd_set_tensor is called with no host synchronisation: the
    sweeps must see the new contents (the oracle on the new tensor)."""
    c1 = synth.custom(3, 48, 6, noise_var=1e-4, seed=93)
    c2 = synth.custom(3, 48, 6, noise_var=1e-4, seed=94)
    s = torch.cuda.Stream()
    T = dev_tensor(cpd, c1)
    T2 = dev_tensor(cpd, c2)
    torch.cuda.synchronize()
    m = _model(cpd, c1, T, stream=s.cuda_stream)
    m.msdt_sweep()
    with torch.cuda.stream(s):
        torch.cuda._sleep(2_000_000)  # the copy lands long after the host returns
        T.copy_(T2)
    m.set_tensor()                    # no host sync: must be ordered after the copy on `s`
    A = synth.init_factors(c2)
    m.set_factors(A)
    To2 = O.make_tensor(c2)
    nt2 = O.norm2(To2)
    for _ in range(2):
        f = m.msdt_sweep()
        out = O.als_sweep(To2, A, nt2)
        assert abs(f - out["f"]) <= TOL * abs(out["f"])
        A = out["A"]
    m.close()


@pytest.mark.parametrize("dims,R", [((4520, 280, 280), 64), ((128, 128, 3, 7200), 32), ((1024, 1344, 33, 9), 32)])
def test_dataset_shaped_sampled_rows(cpd, dims, R):
    """Non-equidimensional tensors shaped like the paper's datasets (4520x280x280,
    128x128x3x7200, 1024x1344x33x9; synthetic values only): one msdt_sweep and one
    dt_sweep, sampled rows of every M^(n) against the oracle's explicit-KRP rows, fitness finite.
    Exercises extents of 3 and 9 (K tails, KC boxes with one partial K step), inner modes that
    are not multiples of 128 (D_MCP tiling) and factor images for every position."""
    cfg = synth.custom(len(dims), 0, R, noise_var=1e-4, seed=sum(dims) % 97, dims=dims)
    free, total = torch.cuda.mem_get_info()
    if free < 2.5 * 8 * cfg.numel + 8e9:
        pytest.skip("not enough device memory")
    T = dev_tensor(cpd, cfg)
    m = _model(cpd, cfg, T)
    rng = np.random.default_rng(len(dims))
    for sweep in (m.msdt_sweep, m.dt_sweep):
        A0 = [m.get_factor(n) for n in range(cfg.N)]
        f = sweep()
        assert np.isfinite(f) and 0.0 < f <= 1.0
        A1 = [m.get_factor(n) for n in range(cfg.N)]
        for n in range(cfg.N):
            if cfg.numel // dims[n] > 2e7:
                continue  # the oracle's slice for this mode is too large; every root is still
                          # exercised through the other modes' MTTKRPs
            Ause = A1[:n] + A0[n:]   # modes < n already updated in this sweep
            rows = rng.choice(dims[n], 2, replace=False)
            ref = O.mttkrp_rows(cfg, Ause, n, rows)
            got = m.get_last_mttkrp(n)[rows]
            assert rel(got, ref) <= TOL, (n, rel(got, ref))
    m.close()
    del T
    torch.cuda.empty_cache()


@pytest.mark.parametrize("ttm_impl", [0, 1])
@pytest.mark.parametrize("dims,R", [((310, 260, 24), 300), ((40, 36, 530), 520), ((44, 40, 1040), 1024)])
def test_large_rank_sweeps(cpd, dims, R, ttm_impl):
    """R beyond one CTA's shared memory, up to CPD_MAX_RANK = 1024: Γ^-1 by the grid-wide blocked
    Gauss-Jordan, x = M Γ^-1 as a DMMA GEMM, the int8 TTM with 5-9 N tiles; two MSDT sweeps,
    one DT sweep, pp_init and one approximated sweep, each state-synchronised with the oracle."""
    cfg = synth.custom(3, 0, R, noise_var=1e-4, seed=R % 89, dims=dims)
    To = O.make_tensor(cfg)
    nt2 = O.norm2(To)
    T = dev_tensor(cpd, cfg)
    m = _model(cpd, cfg, T, ttm_impl=ttm_impl)
    A = synth.init_factors(cfg)
    for sweep in (m.msdt_sweep, m.msdt_sweep, m.dt_sweep):
        f = sweep()
        out = O.als_sweep(To, A, nt2)
        assert abs(f - out["f"]) <= TOL * abs(out["f"]), (f, out["f"])
        A1 = [m.get_factor(n) for n in range(3)]
        for n in range(3):
            # the MTTKRP itself at 1e-10, against the oracle at the GPU's own input factors
            cur = A1[:n] + A[n:]
            ref = O.mttkrp(To, cur, n)
            Mg = m.get_last_mttkrp(n)
            assert rel(Mg, ref) <= TOL, (n, rel(Mg, ref))
            # the factor: the oracle's Cholesky solve of the GPU's own M^(n); the forward error of
            # an SPD solve is ~cond(Γ) u (DESIGN R19), and Γ here (random initial factors, s_n < R
            # for some modes) has cond up to ~1e6
            G = O.gamma([O.gram(a) for a in cur], n)
            tol = max(TOL, 256 * np.finfo(float).eps * np.linalg.cond(G))
            xr = O.solve(G, Mg)
            assert rel(A1[n], xr) <= tol, (n, rel(A1[n], xr), tol)
        A = A1   # state-synchronised
    m.pp_init()
    st = O.pp_init(To, A)
    f, _ = m.pp_approx_sweep()
    out = O.pp_approx_sweep(st, A, nt2)
    assert abs(f - out["f"]) <= TOL * abs(out["f"]), (f, out["f"])
    m.close()


@pytest.mark.parametrize("seed,kind", [(1, "kruskal"), (7, "kruskal"), (3, "uniform")])
def test_last_sweep_status_flags_inconsistent_eq3(cpd, seed, kind):
    """cpd_last_sweep_status: an approximated sweep forced from a random state (far outside the ε
    regime) leaves M~ and A inconsistent -- the Eq. 3 radicand is negative beyond rounding and the
    fitness is the clamped 1; the flag and the radicand/||T||^2 match the oracle's, and regular
    sweeps never raise the flag."""
    cfg = synth.custom(3, 6, 4, kind=kind, noise_var=1e-2, seed=seed)
    To = O.make_tensor(cfg)
    A0 = synth.init_factors(cfg)
    T = dev_tensor(cpd, cfg)
    m = _model(cpd, cfg, T)
    m.pp_init()
    f, _ = m.pp_approx_sweep()
    stt = m.last_sweep_status()
    out = O.pp_approx_sweep(O.pp_init(To, A0), A0, O.norm2(To))
    S = out["S"]
    G = S[0] * S[1]
    rad = (O.norm2(To) + float(np.sum(G * S[2])) - 2.0 * float(np.sum(out["M"][2] * out["A"][2]))) / O.norm2(To)
    assert stt["radicand_negative"] == (rad < -1e-8)
    assert abs(stt["radicand_rel"] - rad) <= 1e-9 * max(1.0, abs(rad))
    if rad < -1e-8:
        assert f == 1.0
    m.set_factors(A0)
    m.msdt_sweep()
    assert not m.last_sweep_status()["radicand_negative"]
    m.close()


@pytest.mark.parametrize("c,rows_per_mode", [(2, 3), (3, 3), (4, 2), (5, 2)])
def test_full_size_pp_state_synchronised(cpd, c, rows_per_mode):
    """C2-C5 at full size: MSDT sweeps, pp_init, then 3 forced approximated sweeps (Alg. 2
    lines 11-16, Eqs. 5-8), each state-synchronised: before every sweep the oracle takes
    the GPU's factors.  Sampled rows of every M~^(n) against the oracle's row-restricted Eq. 5
    (pp_init_rows / pp_approx_rows: operator rows from T's slices with explicit partial KRPs),
    factor rows against the oracle's solve of those rows (cond(Γ)-scaled tolerance, R19), and
    still_valid against the oracle's ε test on the GPU's factors.  A sweep whose Eq. 3 radicand is
    flagged negative (R18) is checked the same way (M~ and factors, not the clamped f)."""
    cfg = synth.config(c)
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info()
    # T + digit planes + the pair operators and one transient root (N = 3: three root-sized pairs)
    need = 15 * cfg.numel + 4 * 8 * cfg.numel // cfg.s * cfg.R + 4e9
    if free < need:
        pytest.skip(f"not enough free device memory ({free / 1e9:.1f} GB)")
    eps = 0.2 if c == 4 else 0.1
    T = dev_tensor(cpd, cfg)
    m = _model(cpd, cfg, T, pp_eps=eps)
    for _ in range(3):
        m.msdt_sweep()
    Ap = [m.get_factor(n) for n in range(cfg.N)]
    m.pp_init()
    rng = np.random.default_rng(100 + c)
    rows = [np.sort(rng.choice(cfg.s, rows_per_mode, replace=False)) for _ in range(cfg.N)]
    cache = {}
    st_rows = [O.pp_init_rows(cfg, Ap, n, rows[n], cache) for n in range(cfg.N)]
    A = Ap
    for sweep in range(3):
        f, valid = m.pp_approx_sweep()
        flagged = m.last_sweep_status()["radicand_negative"]
        A1 = [m.get_factor(n) for n in range(cfg.N)]
        for n in range(cfg.N):
            cur = A1[:n] + A[n:]
            ref = O.pp_approx_rows(st_rows[n], cur, n, rows[n])
            got = m.get_last_mttkrp(n)[rows[n]]
            assert rel(got, ref) <= TOL, (sweep, n, rel(got, ref))
            G = O.gamma([O.gram(a) for a in cur], n)
            tol = max(TOL, 256 * np.finfo(float).eps * np.linalg.cond(G))
            xr = O.solve(G, got)   # the oracle's solve of the GPU's M~ rows (R19)
            assert rel(A1[n][rows[n]], xr) <= tol, (sweep, n, rel(A1[n][rows[n]], xr), tol)
        dA = [a - p for a, p in zip(A1, Ap)]
        ratios = [np.linalg.norm(d) / np.linalg.norm(a) for d, a in zip(dA, A1)]
        if all(abs(r - eps) > 1e-9 * eps for r in ratios):   # not at the ε boundary (Q17)
            assert valid == O.pp_condition(dA, A1, eps)
        if flagged:
            assert f == 1.0
        A = A1
    m.close()
    del T
    torch.cuda.empty_cache()


@pytest.mark.parametrize("N,s,R", [(3, 48, 6), (4, 12, 4), (5, 8, 3)])
def test_pp_back_to_back_speculation(cpd, N, s, R):
    """Approximated sweeps called back to back with no other call in between, so every speculative
    filler-stream launch (the next sweep's mode-1 streams and its mode-0 M~, started during and at
    the end of a sweep) is consumed: the fitness trace and the final factors against the oracle's
    pp_approx_sweep chain (Eqs. 5-8) from the same state.  Also covers the first sweep after
    pp_init, whose dA = 0 terms are taken as M_p directly."""
    cfg = synth.custom(N, s, R, noise_var=1e-4, seed=60 + N)
    T = dev_tensor(cpd, cfg)
    To = O.make_tensor(cfg)
    nt2 = O.norm2(To)
    m = _model(cpd, cfg, T)
    A = synth.init_factors(cfg)
    for _ in range(4):
        m.msdt_sweep()
        A = O.als_sweep(To, A, nt2)["A"]
    A = [m.get_factor(n) for n in range(N)]
    m.pp_init()
    st = O.pp_init(To, A)
    fs = [m.pp_approx_sweep()[0] for _ in range(4)]
    for k in range(4):
        out = O.pp_approx_sweep(st, A, nt2)
        A = out["A"]
        assert abs(fs[k] - out["f"]) <= TOL * abs(out["f"]), (k, fs[k], out["f"])
    for n in range(N):
        assert rel(m.get_factor(n), A[n]) <= 1e-9, (n, rel(m.get_factor(n), A[n]))
    m.close()


def test_c2_full_trajectory(cpd):
    """C2 (1024^3, R = 64) full-trajectory parity (SURVEY §8(d) run schedule): 4 msdt_sweep on the GPU
    from the seeded initial factors against 4 exact oracle ALS sweeps (explicit unfolding + explicit
    KRP + Cholesky) from the same factors on the host copy of the tensor (synth recipe, generated in
    parallel blocks by bench.host_tensor; ~1e-16 from oracle.make_tensor): fitness at 1e-10 and
    factors at 1e-9 every sweep (no state synchronisation)."""
    import bench
    cfg = synth.config(2)
    torch.cuda.empty_cache()
    if torch.cuda.mem_get_info()[0] < 8 * cfg.numel * 2.2:
        pytest.skip("not enough device memory")
    T = dev_tensor(cpd, cfg)
    A0 = synth.init_factors(cfg)
    m = _model(cpd, cfg, T)
    f_gpu, A_gpu = [], []
    for _ in range(4):
        f_gpu.append(m.msdt_sweep())
        A_gpu.append([m.get_factor(n) for n in range(cfg.N)])
    m.close()
    del T
    torch.cuda.empty_cache()
    To = bench.host_tensor(cfg)
    nt2 = O.norm2(To)
    A = A0
    for k in range(4):
        out = O.als_sweep(To, A, nt2)
        A = out["A"]
        assert abs(f_gpu[k] - out["f"]) <= TOL * abs(out["f"]), (k, f_gpu[k], out["f"])
        for n in range(cfg.N):
            assert rel(A_gpu[k][n], A[n]) <= 1e-9, (k, n, rel(A_gpu[k][n], A[n]))
