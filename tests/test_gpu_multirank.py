"""The 1-D-grid multi-rank path (Alg. 3 / Alg. 4: slab-local contractions, reduce-scatter
of the partial MTTKRP, all-gather of factor rows, all-reduce of the last mode's Gram, dS and
scalars) run on ONE GPU with P ranks of an in-process cpd_local_group, each rank driven by
its own host thread, compared with P = 1 and with the oracle (-m gpu)."""
import threading

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


def slab(cpd, cfg, rank, world):
    lo, hi = synth.slab_range(cfg.s, rank, world)
    T = torch.empty([cfg.s] * (cfg.N - 1) + [hi - lo], dtype=torch.float64, device="cuda")
    cpd.cpd_gen_tensor(T, cfg.shape, lo, hi, 0, synth.true_factors(cfg), np.sqrt(cfg.noise_var), cfg.seed_noise)
    torch.cuda.synchronize()
    return T


def schedule(m, N):
    """3 MSDT sweeps, PP init + 2 PP sweeps, 1 MSDT sweep, 1 DT sweep; record everything."""
    rec = {"f": [], "M": [], "A": []}
    for _ in range(3):
        rec["f"].append(m.msdt_sweep())
        rec["M"].append([m.get_last_mttkrp(n) for n in range(N)])
    rec["A"].append([m.get_factor(n) for n in range(N)])
    m.pp_init()
    for _ in range(2):
        rec["f"].append(m.pp_approx_sweep()[0])
        rec["M"].append([m.get_last_mttkrp(n) for n in range(N)])
    rec["f"].append(m.msdt_sweep())
    rec["f"].append(m.dt_sweep())
    rec["A"].append([m.get_factor(n) for n in range(N)])
    return rec


def block(cpd, cfg, rank, grid):
    """Rank `rank`'s block of the N-D processor grid (row-major rank order, last mode fastest)."""
    coord, rem = [0] * cfg.N, rank
    for n in reversed(range(cfg.N)):
        coord[n], rem = rem % grid[n], rem // grid[n]
    lo = [c * (s // g) for c, s, g in zip(coord, cfg.shape, grid)]
    hi = [l + s // g for l, s, g in zip(lo, cfg.shape, grid)]
    T = torch.empty([h - l for l, h in zip(lo, hi)], dtype=torch.float64, device="cuda")
    cpd.cpd_gen_tensor_block(T, cfg.shape, lo, hi, 0, synth.true_factors(cfg), np.sqrt(cfg.noise_var),
                             cfg.seed_noise)
    torch.cuda.synchronize()
    return T


def run_group(cpd, cfg, P, grid=None, fused_rs=False, msdt_levels=1):
    group = cpd.cpd_local_group_create(P)
    Ts = [slab(cpd, cfg, r, P) if grid is None else block(cpd, cfg, r, grid) for r in range(P)]
    out, errs = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            m = cpd.cp_als_init(Ts[r], cfg.shape, cfg.R, synth.init_factors(cfg), rank=r, world=P,
                                local_group=group, stream=torch.cuda.Stream(), grid=grid, fused_rs=fused_rs,
                                msdt_levels=msdt_levels)
            out[r] = schedule(m, cfg.N)
            m.close()
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    cpd.cpd_local_group_destroy(group)
    assert not errs, errs
    assert all(not t.is_alive() for t in th)
    return out


@pytest.mark.parametrize("cfg,P", [(synth.config(1), 2), (synth.config(1), 4), (synth.custom(4, 8, 3, noise_var=1e-3, seed=31), 2),
                                   (synth.custom(3, 16, 5, noise_var=1e-4, seed=32), 8)])
def test_local_group_equals_single_rank_and_oracle(cpd, cfg, P):
    ref = run_group(cpd, cfg, 1)[0]
    got = run_group(cpd, cfg, P)
    for r in range(P):  # every rank returns the same gathered results
        for a, b in zip(got[r]["f"], ref["f"]):
            assert abs(a - b) <= TOL * abs(b)
        for Ms, Mr in zip(got[r]["M"], ref["M"]):
            for a, b in zip(Ms, Mr):
                assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(b)
        for As, Ar in zip(got[r]["A"], ref["A"]):
            for a, b in zip(As, Ar):
                assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(b)
    # and the first three sweeps against the oracle directly
    T = O.make_tensor(cfg)
    A = synth.init_factors(cfg)
    for k in range(3):
        o = O.als_sweep(T, A)
        A = o["A"]
        assert abs(got[0]["f"][k] - o["f"]) <= TOL * abs(o["f"])


def test_local_group_rejects_bad_world(cpd):
    g = cpd.cpd_local_group_create(2)
    cfg = synth.custom(3, 8, 2, seed=33)
    T = slab(cpd, cfg, 0, 4)
    with pytest.raises(cpd.CPDError) as e:
        cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), rank=0, world=4, local_group=g)
    assert e.value.status == 1
    cpd.cpd_local_group_destroy(g)


@pytest.mark.parametrize("cfg,grid", [(synth.custom(3, 16, 5, noise_var=1e-4, seed=34), (2, 2, 2)),
                                      (synth.custom(3, 24, 4, noise_var=1e-4, seed=35), (2, 1, 3)),
                                      (synth.custom(4, 8, 3, noise_var=1e-3, seed=36), (2, 2, 1, 2)),
                                      (synth.custom(3, 16, 6, noise_var=1e-4, seed=37), (1, 4, 2))])
def test_nd_grid_equals_single_rank_and_oracle(cpd, cfg, grid):
    """Alg. 3 / Alg. 4 on an N-D processor grid: every rank holds
    a cubical block, M^(n) reduce-scattered in Proc-Slice(x_n), A^(n) all-gathered there, Grams
    all-reduced; same schedule as above, P ranks of a local group on one GPU, against P = 1 and the
    oracle's grid simulation (oracle.par_als_sweep_grid_sim)."""
    P = int(np.prod(grid))
    ref = run_group(cpd, cfg, 1)[0]
    got = run_group(cpd, cfg, P, grid=grid)
    for r in range(P):
        for a, b in zip(got[r]["f"], ref["f"]):
            assert abs(a - b) <= TOL * abs(b)
        for Ms, Mr in zip(got[r]["M"], ref["M"]):
            for a, b in zip(Ms, Mr):
                assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(b)
        for As, Ar in zip(got[r]["A"], ref["A"]):
            for a, b in zip(As, Ar):
                assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(b)
    T = O.make_tensor(cfg)
    A = synth.init_factors(cfg)
    for k in range(3):
        o = O.par_als_sweep_grid_sim(T, A, grid)
        A = o["A"]
        assert abs(got[0]["f"][k] - o["f"]) <= TOL * abs(o["f"])


@pytest.mark.parametrize("cfg,grid", [(synth.config(1), None), (synth.custom(3, 16, 5, noise_var=1e-4, seed=34), (2, 2, 2)),
                                      (synth.custom(4, 8, 3, noise_var=1e-3, seed=36), (2, 2, 1, 2))])
def test_fused_reduce_scatter_epilogue(cpd, cfg, grid):
    """opts.fused_rs (Alg. 3 line 14, Alg. 4 line 9): the mTTV / PP-stream launch that
    completes each rank's partial M^(n) stores the owners' rows straight into their receive slots,
    then a stream-ordered barrier and a fixed-order slot sum replace the reduce-scatter collective.
    Same schedule (MSDT, PP, DT sweeps) against the collective path and P = 1."""
    P = 4 if grid is None else int(np.prod(grid))
    ref = run_group(cpd, cfg, 1)[0]
    plain = run_group(cpd, cfg, P, grid=grid)
    fused = run_group(cpd, cfg, P, grid=grid, fused_rs=True)
    for r in range(P):
        for a, b, c in zip(fused[r]["f"], plain[r]["f"], ref["f"]):
            assert abs(a - c) <= TOL * abs(c) and abs(a - b) <= TOL * abs(b)
        for Ms, Mr in zip(fused[r]["M"], ref["M"]):
            for a, b in zip(Ms, Mr):
                assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(b)
        for As, Ar in zip(fused[r]["A"], ref["A"]):
            for a, b in zip(As, Ar):
                assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(b)


def test_grid_validation(cpd):
    """cpd_opts.grid errors (include/cpd.h): prod(grid) != world, s_n % I_n != 0, or a block not
    divisible over its slice -> CPD_ERR_INVALID_ARG at cp_als_init (every rank; checked on rank 0 of
    a local group of 4, where the call fails before any collective)."""
    g = cpd.cpd_local_group_create(4)
    cfg = synth.custom(3, 8, 2, seed=38)
    T = torch.empty(4, 4, 4, dtype=torch.float64, device="cuda")
    for grid in [(2, 2, 2), (3, 1, 1), (2, 1, 1)]:
        with pytest.raises(cpd.CPDError) as e:
            cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), rank=0, world=4, local_group=g, grid=grid)
        assert e.value.status == 1
    cfg6 = synth.custom(3, 6, 2, seed=39)   # 6 % 4 != 0 for a 1x1x4 grid
    with pytest.raises(cpd.CPDError) as e:
        cpd.cp_als_init(T, cfg6.shape, cfg6.R, synth.init_factors(cfg6), rank=0, world=4, local_group=g,
                        grid=(1, 1, 4))
    assert e.value.status == 1
    cpd.cpd_local_group_destroy(g)


@pytest.mark.parametrize("cfg,grid,fused_rs", [(synth.custom(4, 8, 3, noise_var=1e-3, seed=38), None, False),
                                               (synth.custom(4, 8, 3, noise_var=1e-3, seed=38), (2, 2, 1, 2), False),
                                               (synth.custom(5, 4, 3, noise_var=1e-3, seed=39), (1, 2, 1, 1, 2), True)])
def test_fused_levels_partitioned(cpd, cfg, grid, fused_rs):
    """Upper-level fusion (msdt_levels = 2) on the partitioned path: every rank contracts its
    own block of T with the Khatri-Rao product of its factor blocks (the block contraction is local,
    Table 1), the leaves are reduce-scattered as in Alg. 3; the whole schedule equals P = 1 with l = 1."""
    P = 2 if grid is None else int(np.prod(grid))
    ref = run_group(cpd, cfg, 1)[0]
    got = run_group(cpd, cfg, P, grid=grid, fused_rs=fused_rs, msdt_levels=2)
    for r in range(P):
        for a, b in zip(got[r]["f"], ref["f"]):
            assert abs(a - b) <= TOL * abs(b)
        for Ms, Mr in zip(got[r]["M"], ref["M"]):
            for a, b in zip(Ms, Mr):
                assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(b)
        for As, Ar in zip(got[r]["A"], ref["A"]):
            for a, b in zip(As, Ar):
                assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(b)
