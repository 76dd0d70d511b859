"""CPU oracle for the MSDT / pairwise-perturbation CP-ALS hot path (arXiv 2010.12056).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2010_12056_b200``) never imports it and
shares no code with it; the only common module is ``synth`` (seeded inputs,
no method arithmetic).

Plain NumPy/SciPy in float64.  Every function cites the PAPER.md passage it
follows (``P:<line>``).  Exact reorganisations (DT, MSDT) are checked against
the *plain definition* (explicit unfolding x explicit Khatri-Rao product);
pairwise perturbation follows Eqs. 5-8 / Alg. 2 step by step.

Pins (tests/test_oracle_pins.py, ``-m "not gpu"``) tie every function here to
something other than itself: brute-force loops, closed forms, SPEC/paper
worked examples (tests/golden), invariants of the method.
"Oracle and pins" for the table; no function is "parity unpinned" except the
multi-sweep PP trajectory on structureless data.
"""
from .cpals import *  # noqa: F401,F403
