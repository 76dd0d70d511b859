"""World-size-2 CPU test of the 1-D-grid parallel algorithm (Alg. 3 / Alg. 4) with real
torch.distributed collectives (gloo), against the sequential oracle sweep.

This covers the host-side logic of the multi-GPU path that the single-GPU runs of this
round cannot execute: slab ownership (synth.slab_range), reduce-scatter of the partial
MTTKRP for modes < N, solve on own rows, all-gather of the factor, all-reduce of the last
mode's Gram / dS and of the fitness scalars, and the NCCL-id broadcast the binding does.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reduce_scatter_rows(M, rank, world):
    """Reduce-scatter by rows (gloo: all_reduce + own block)."""
    t = torch.from_numpy(np.ascontiguousarray(M))
    dist.all_reduce(t)
    b = M.shape[0] // world
    return t.numpy()[rank * b:(rank + 1) * b].copy()


def _all_gather_rows(own, world):
    parts = [torch.empty_like(torch.from_numpy(own)) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(own)))
    return np.concatenate([p.numpy() for p in parts])


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(np.array(x, dtype=np.float64)))
    dist.all_reduce(t)
    return t.numpy()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # NCCL-id style broadcast of 128 opaque bytes (what bench.py / the binding do)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))

        cfg = synth.custom(3, 8, 3, noise_var=1e-3, seed=21)
        lo, hi = synth.slab_range(cfg.s, rank, world)
        Tl = O.make_tensor(cfg, rank, world)                  # this rank's slab only
        A = synth.init_factors(cfg)
        A = [a.copy() for a in A]
        Aloc_last = A[-1][lo:hi].copy()
        nt2 = float(_allreduce([O.norm2(Tl)])[0])
        S = [O.gram(a) for a in A[:-1]] + [_allreduce(O.gram(Aloc_last))]
        N = cfg.N
        for sweep in range(3):
            for n in range(N):
                G = O.gamma(S, n)
                Al = A[:-1] + [Aloc_last]
                Mloc = O.mttkrp(Tl, Al, n)                      # Local-MTTKRP (Alg. 3 line 13)
                if n < N - 1:
                    Mown = _reduce_scatter_rows(Mloc, rank, world)  # line 14
                    own = O.solve(G, Mown)                       # line 15
                    A[n] = _all_gather_rows(own, world)          # line 18
                    S[n] = O.gram(A[n])                          # replicated, no all-reduce
                else:
                    Aloc_last = O.solve(G, Mloc)                 # local rows are exact
                    S[n] = _allreduce(O.gram(Aloc_last))         # line 17
                    ma = float(_allreduce([np.sum(Mloc * Aloc_last)])[0])
                    gs = float(np.sum(G * S[n]))
            r = np.sqrt(max(nt2 + gs - 2 * ma, 0.0)) / np.sqrt(nt2)
            if rank == 0:
                q.put(("f", sweep, 1 - r))
        Afull_last = _all_gather_rows(Aloc_last, world)
        if rank == 0:
            q.put(("A", [A[0], A[1], Afull_last]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_parallel_als_equals_sequential():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    got = {}
    while not q.empty():
        item = q.get()
        if item[0] == "f":
            got[("f", item[1])] = item[2]
        else:
            got["A"] = item[1]
    cfg = synth.custom(3, 8, 3, noise_var=1e-3, seed=21)
    T = O.make_tensor(cfg)
    A = synth.init_factors(cfg)
    for sweep in range(3):
        out = O.als_sweep(T, A)
        A = out["A"]
        assert abs(got[("f", sweep)] - out["f"]) <= 1e-10
    for a, b in zip(got["A"], A):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)


# ------------------------- N-D processor grid, world 4 ------------------------------

def _grid_worker(rank, world, port, q, grid):
    """Alg. 3 on the grid `grid` with real collectives: block-local MTTKRP, reduce-scatter
    within Proc-Slice(x_n) (the ranks sharing x_n; gloo: all_reduce on the slice group + own rows),
    solve own rows, Gram of own rows all-reduced over all ranks, all-gather of the block in the slice
    -- the same exchange pattern libcpd's exchange_mode / update_mode uses."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.custom(3, 8, 3, noise_var=1e-3, seed=22)
        N = cfg.N
        procs = O.grid_procs(grid)
        x = procs[rank]
        # every rank creates every group (collective), keeps its own slice
        slices = {}
        for n in range(N):
            for c in range(grid[n]):
                g = dist.new_group([r for r, y in enumerate(procs) if y[n] == c])
                if x[n] == c:
                    slices[n] = (g, [r for r, y in enumerate(procs) if y[n] == c])
        blk = [synth.slab_range(s, k, g) for s, k, g in zip(cfg.shape, x, grid)]
        Tl = O.make_tensor_block(cfg, blk)
        A0 = synth.init_factors(cfg)
        Ab = [a[lo:hi].copy() for a, (lo, hi) in zip(A0, blk)]        # block rows of every factor
        nt2 = float(_allreduce([O.norm2(Tl)])[0])
        S = [O.gram(a) for a in A0]
        for sweep in range(3):
            for n in range(N):
                G = O.gamma(S, n)
                Mloc = O.mttkrp(Tl, Ab, n)                              # line 13
                g, members = slices[n]
                P = len(members)
                t = torch.from_numpy(np.ascontiguousarray(Mloc))
                dist.all_reduce(t, group=g)                               # line 14 (sum over the slice)
                b = Mloc.shape[0] // P
                me = members.index(rank)
                Mown = t.numpy()[me * b:(me + 1) * b]
                own = O.solve(G, Mown)                                    # line 15
                S[n] = _allreduce(O.gram(own))                            # lines 16-17 (all ranks)
                parts = [torch.empty_like(torch.from_numpy(own)) for _ in range(P)]
                dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(own)), group=g)  # line 18
                Ab[n] = np.concatenate([p.numpy() for p in parts])
                if n == N - 1:
                    ma = float(_allreduce([np.sum(Mown * own)])[0])
                    gs = float(np.sum(G * S[n]))
            r = np.sqrt(max(nt2 + gs - 2 * ma, 0.0)) / np.sqrt(nt2)
            if rank == 0:
                q.put(("f", sweep, 1 - r))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid", [(2, 2, 1), (1, 2, 2)])
def test_gloo_world4_grid_als_equals_sequential(grid):
    world = 4
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_grid_worker, args=(r, world, port, q, grid)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    got = {}
    while not q.empty():
        item = q.get()
        got[item[1]] = item[2]
    cfg = synth.custom(3, 8, 3, noise_var=1e-3, seed=22)
    T = O.make_tensor(cfg)
    A = synth.init_factors(cfg)
    for sweep in range(3):
        out = O.als_sweep(T, A)
        A = out["A"]
        assert abs(got[sweep] - out["f"]) <= 1e-10
