"""Alg. 2 controller host logic (-m "not gpu"): `driver.pp_cp_als` (the product's
controller above the C ABI) driven by a stand-in model whose sweeps are the oracle's,
against `oracle.pp_controller_run` on the same inputs.  Checks the max_sweeps count
(regular + approximated sweeps, no PP initialisations: P:931 against Table 3's columns
P:836-849) and the handling of a sweep with a negative Eq. 3 radicand (reading R18)."""
import numpy as np
import pytest

import oracle as O
import oracle.cpals as OC
import synth
from paper_2010_12056_b200 import driver


class OracleModel:
    """The CPDecomposition interface the controller uses, backed by the oracle."""

    def __init__(self, T, A0, eps):
        self.T, self.A, self.eps = T, [a.copy() for a in A0], eps
        self.nt2 = O.norm2(T)
        self.dA = [a.copy() for a in A0]     # Alg. 2 line 2
        self.st = None
        self.rad = 0.0

    def pp_condition(self):
        return O.pp_condition(self.dA, self.A, self.eps)

    def msdt_sweep(self):
        out = O.als_sweep(self.T, self.A, self.nt2)
        self.A, self.dA, self.rad = out["A"], out["dA"], out["rad"]
        return out["f"]

    def pp_init(self):
        self.st = O.pp_init(self.T, self.A)
        self.dA = [np.zeros_like(a) for a in self.A]

    def pp_approx_sweep(self):
        out = OC.pp_approx_sweep(self.st, self.A, self.nt2, self.eps)
        self.A, self.dA, self.rad = out["A"], out["dA"], out["rad"]
        return out["f"], bool(out["still_valid"])

    def last_sweep_status(self):
        return {"radicand_negative": self.rad < -O.RADICAND_TOL, "radicand_rel": self.rad}


def _case():
    cfg = synth.custom(3, 16, 3, noise_var=1e-6, seed=8)
    return O.make_tensor(cfg), synth.init_factors(cfg)


@pytest.mark.parametrize("stop_test", ["any", "regular"])
@pytest.mark.parametrize("max_sweeps", [7, 300])
def test_driver_matches_oracle_controller(max_sweeps, stop_test):
    T, A0 = _case()
    _, tr = O.pp_controller_run(T, A0, 0.1, max_sweeps=max_sweeps, stop_test=stop_test)
    rows = driver.pp_cp_als(OracleModel(T, A0, 0.1), max_sweeps=max_sweeps, stop_test=stop_test)
    assert [k for k, _ in tr] == [r[1] for r in rows]
    for (k, f), r in zip(tr, rows):
        assert (f is None and r[3] is None) or abs(f - r[3]) <= 1e-13
    assert "pp_approx" in [k for k, _ in tr]
    n_sweeps = sum(1 for k, _ in tr if k != "pp_init")
    if max_sweeps == 7:
        assert n_sweeps == 7 and "pp_init" in [k for k, _ in tr]     # pp_init rows do not count
    assert rows[-1][0] == n_sweeps


def test_flagged_radicand_ends_pp_run(monkeypatch):
    """A PP sweep with Eq. 3 radicand < -1e-8 ||T||^2: fitness None, the PP run ends, a regular
    sweep follows, and the Δ test never uses the clamped value (both controllers)."""
    T, A0 = _case()
    real = OC.pp_approx_sweep
    calls = {"n": 0}

    def flag_second(st, A, nt2, eps=None):
        out = real(st, A, nt2, eps)
        calls["n"] += 1
        if calls["n"] == 2:
            out = dict(out, rad=-1e-3, f=1.0)     # as a clamped f = 1 would be reported
        return out

    monkeypatch.setattr(OC, "pp_approx_sweep", flag_second)
    _, tr = O.pp_controller_run(T, A0, 0.1, max_sweeps=40)
    calls["n"] = 0
    rows = driver.pp_cp_als(OracleModel(T, A0, 0.1), max_sweeps=40)
    kinds = [k for k, _ in tr]
    assert kinds == [r[1] for r in rows]
    i = [j for j, k in enumerate(kinds) if k == "pp_approx"][1]
    assert tr[i][1] is None and rows[i][3] is None
    assert kinds[i + 1] == "regular"
    assert all(f is None or f < 1.0 for _, f in tr)
