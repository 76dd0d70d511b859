"""Alg. 2 (PP-CP-ALS) regime controller: the driver loop above the C ABI.

SURVEY §8(b): the library exports single sweeps (msdt_sweep / pp_init /
pp_approx_sweep) and only *reports* the PP condition; the regime logic of Alg. 2
 lives here, on the host, calling nothing but those entry points.

Readings:
  * dA <- A initially (Alg. 2 line 2), so the first sweep is always regular;
  * enter PP iff ∀i ‖dA⁽ⁱ⁾‖_F < ε‖A⁽ⁱ⁾‖_F with dA the last regular sweep's update
    (Alg. 2 line 5; strict '<', Q17) -- `cpd_pp_condition`;
  * inside the PP regime run approximated sweeps while `still_valid` (line 11),
    with no cap unless max_pp_run is given, then one regular sweep (line 18,
    P:361; the paper "calls the MSDT subroutine for the regular ALS sweeps");
    re-entry re-initialises;
  * fitness after every sweep (reading Q21); the Δ stop test between neighbouring sweeps of
    any kind (the P:931 wording, reading R12, default) or, with stop_test="regular", between
    consecutive regular sweeps as Alg. 2 prints it; or after max_sweeps sweeps, counting
    regular and approximated sweeps but not PP initialisations (the 300-iteration cap of P:931
    against Table 3's separate Num-ALS / Num-PP-init / Num-PP-approx columns);
  * an approximated sweep whose Eq. 3 radicand is negative beyond rounding
    (`cpd_last_sweep_status`, reading R18) has no residual: its row carries fitness None, the
    PP run ends there and the Δ test skips it (the next regular sweep is compared with the
    last valid fitness).

Timing of each sweep is the host wall clock around the blocking ABI call (each call
returns only after its stream work completed); it is a trace, not a bench number.
"""
from __future__ import annotations

import time


def pp_cp_als(model, delta=1e-5, max_sweeps=300, max_pp_run=None, regular="msdt", trace=None,
              stop_test="any"):
    """Run Alg. 2 on an initialised `CPDecomposition` until the Δ test or max_sweeps.

    stop_test: "any" (default, reading Q21/R12) -- Δ between neighbouring sweeps of any kind (the
    P:931 wording); "regular" -- Alg. 2 as printed (lines 3-4, 19-21): the
    residual r is updated only after a regular sweep and the run ends when |r - r_old| <= Δ
    between consecutive regular sweeps (r = 1, r_old = 0 initially).  The paper is at odds with
    itself here; DESIGN.md §10a compares the two on the collinearity study.

    Returns a list of trace rows ``(sweep, phase, residual, fitness, wall_seconds)``
    where phase ∈ {"regular", "pp_init", "pp_approx"} (S:251 CSV columns); pp_init rows
    and flagged approximated sweeps carry no fitness.  `regular` selects the regular sweep
    ("msdt" per P:788, or "dt").
    If `trace` is a file-like object the rows are also written to it as CSV.
    """
    if stop_test not in ("regular", "any"):
        raise ValueError("stop_test must be 'regular' or 'any'")
    sweep_fn = model.msdt_sweep if regular == "msdt" else model.dt_sweep
    rows = []
    f_old = None
    f_reg_old = 0.0  # r = 1 before the first regular sweep (Alg. 2 line 3)
    n_sweeps = 0

    def log(phase, f, dt):
        row = (n_sweeps, phase, None if f is None else 1.0 - f, f, dt)
        rows.append(row)
        if trace is not None:
            trace.write(",".join("" if v is None else (repr(v) if isinstance(v, float) else str(v))
                                 for v in row) + "\n")

    if trace is not None:
        trace.write("sweep,phase,residual,fitness,wall_seconds\n")
    while n_sweeps < max_sweeps:
        stop = False
        if model.pp_condition():                       # Alg. 2 line 5
            t0 = time.perf_counter()
            model.pp_init()                            # lines 6-9
            log("pp_init", None, time.perf_counter() - t0)
            n_run = 0
            while True:                                # lines 10-17
                t0 = time.perf_counter()
                f, still_valid = model.pp_approx_sweep()
                n_sweeps += 1
                flagged = model.last_sweep_status()["radicand_negative"]
                log("pp_approx", None if flagged else f, time.perf_counter() - t0)
                n_run += 1
                if flagged:
                    break
                if stop_test == "any":
                    stop = f_old is not None and abs(f - f_old) <= delta
                f_old = f
                if stop or not still_valid or n_sweeps >= max_sweeps or \
                        (max_pp_run is not None and n_run >= max_pp_run):
                    break
            if stop or n_sweeps >= max_sweeps:
                break
        t0 = time.perf_counter()
        f = sweep_fn()                                 # line 18: a regular sweep
        n_sweeps += 1
        log("regular", f, time.perf_counter() - t0)
        if stop_test == "any":
            if f_old is not None and abs(f - f_old) <= delta:
                break
        elif abs(f - f_reg_old) <= delta:              # lines 19-21 (and line 4)
            break
        f_old = f
        f_reg_old = f
    return rows


def phase_counts(rows):
    """Sweep counts per phase (the paper's Table 3/4 columns)."""
    out = {"regular": 0, "pp_init": 0, "pp_approx": 0}
    for r in rows:
        out[r[1]] += 1
    return out
