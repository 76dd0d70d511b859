"""Alg. 2 controller (paper_2010_12056_b200.driver) on the GPU against the oracle's
controller (oracle.pp_controller_run), same seeded inputs (-m gpu).

Both sides take the ε branch (Alg. 2 lines 5/10) and the Δ stop test
(reading Q21) from their own fitness/norms; the cases were chosen (with the
oracle only) so that no branch is within 10 % of its threshold (reading Q17), so the
phase sequences must be identical and the fitness of every sweep within 1e-10.
"""
import io

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


def _dev_tensor(cpd, cfg):
    T = torch.empty(cfg.shape, dtype=torch.float64, device="cuda")
    cpd.cpd_gen_tensor(T, cfg.shape, 0, cfg.s, 0, synth.true_factors(cfg), np.sqrt(cfg.noise_var), cfg.seed_noise)
    return T


# (N, s, R, noise variance, seed, ε, Δ, max_pp_run): the first case re-enters PP
# (RRRRRIppppRIp), the second is order 4 (RRRRRIppp)
CASES = [(3, 64, 8, 1e-6, 1001, 0.2, 1e-9, 4), (4, 12, 4, 1e-3, 17, 0.2, 1e-8, 3)]


@pytest.mark.parametrize("stop_test", ["regular", "any"])
@pytest.mark.parametrize("case", CASES)
def test_alg2_controller_matches_oracle(cpd, case, stop_test):
    from paper_2010_12056_b200 import driver
    N, s, R, nv, seed, eps, delta, mpr = case
    cfg = synth.custom(N, s, R, noise_var=nv, seed=seed)
    To = O.make_tensor(cfg)
    A0 = synth.init_factors(cfg)
    _, tr_o = O.pp_controller_run(To, A0, eps, delta=delta, max_sweeps=80, max_pp_run=mpr, stop_test=stop_test)
    T = _dev_tensor(cpd, cfg)
    m = cpd.cp_als_init(T, cfg.shape, cfg.R, A0, pp_eps=eps)
    buf = io.StringIO()
    rows = driver.pp_cp_als(m, delta=delta, max_sweeps=80, max_pp_run=mpr, trace=buf, stop_test=stop_test)
    m.close()
    kinds_o = [k for k, _ in tr_o]
    kinds_g = [r[1] for r in rows]
    assert kinds_g == kinds_o
    assert "pp_approx" in kinds_g
    for (k, fo), r in zip(tr_o, rows):
        if fo is not None:
            assert abs(r[3] - fo) <= TOL * abs(fo), (k, r[3], fo)
    counts = driver.phase_counts(rows)
    assert counts["pp_init"] == kinds_o.count("pp_init")
    csv = buf.getvalue().splitlines()
    assert csv[0] == "sweep,phase,residual,fitness,wall_seconds" and len(csv) == len(rows) + 1
