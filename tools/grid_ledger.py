"""Per-rank work ledger of the 1-D vs the N-D processor grid (Table 1) on ONE
GPU through the local group: P ranks (one host thread each), the same global tensor split either
1 x .. x 1 x P or on `grid`; per rank the PP-approximated sweep's operator-stream bytes (main +
filler streams), the MSDT sweep's TTM flops / stream bytes from the library's ledger, and the aux-memory
high-water marks (cpd_get_memory) of the MSDT sweeps and of pp_init (Table 1's aux-memory column).
usage: python tools/grid_ledger.py s R g1,g2,g3 [ttm_impl]   (order 3; e.g. 1024 200 2,2,2)"""
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_12056_b200 as cpd  # noqa: E402
import synth  # noqa: E402

s, R = int(sys.argv[1]), int(sys.argv[2])
grid = tuple(int(x) for x in sys.argv[3].split(","))
impl = int(sys.argv[4]) if len(sys.argv) > 4 else 0
P = int(np.prod(grid))
cfg = synth.custom(3, s, R, noise_var=1e-4, seed=5)


def block(rank, g):
    coord, rem = [0] * 3, rank
    for n in reversed(range(3)):
        coord[n], rem = rem % g[n], rem // g[n]
    lo = [c * (cfg.s // gg) for c, gg in zip(coord, g)]
    hi = [l + cfg.s // gg for l, gg in zip(lo, g)]
    T = torch.empty([h - l for l, h in zip(lo, hi)], dtype=torch.float64, device="cuda")
    cpd.cpd_gen_tensor_block(T, cfg.shape, lo, hi, 0, synth.true_factors(cfg), np.sqrt(cfg.noise_var),
                             cfg.seed_noise)
    return T


def run(g):
    group = cpd.cpd_local_group_create(P)
    out = [None] * P

    def worker(r):
        torch.cuda.set_device(0)
        T = block(r, g)
        torch.cuda.synchronize()
        m = cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), rank=r, world=P, local_group=group,
                            grid=g, ttm_impl=impl, stream=torch.cuda.Stream())
        for _ in range(2):
            m.msdt_sweep()
        m.reset_counters()
        m.msdt_sweep()
        m.msdt_sweep()
        c = m.counters()
        mem_msdt = m.get_memory()["peak"]
        m.reset_counters()
        m.pp_init()
        mem_pp = m.get_memory()["peak"]
        m.pp_approx_sweep()
        m.reset_counters()
        m.pp_approx_sweep()
        cp, fl = m.counters(), m.filler_counters()
        # aux memory: high-water marks of the library's intermediates (Table 1's aux-memory column)
        out[r] = {"msdt_ttm_gflop_per_sweep": c["ttm_flops"] / 2e9, "msdt_stream_gb_per_sweep": c["stream_bytes"] / 2e9,
                  "pp_operator_gb_per_sweep": (cp["stream_bytes"] + fl["bytes"]) / 1e9, "block": list(T.shape),
                  "msdt_aux_gb": mem_msdt / 1e9, "pp_init_aux_gb": mem_pp / 1e9}
        m.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    [t.start() for t in th]
    [t.join() for t in th]
    cpd.cpd_local_group_destroy(group)
    return out


res = {"s": s, "R": R, "P": P, "one_d": run((1, 1, P))[0], "grid": list(grid), "nd": run(grid)[0]}
print(json.dumps(res))
