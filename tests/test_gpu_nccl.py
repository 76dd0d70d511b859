"""The NCCL backend of the 1-D grid (Alg. 3 P:419-456 / Alg. 4) on real GPUs:
world = 2 ranks, one process per GPU under torch.distributed.run, libcpd's own NCCL
communicator (reduce-scatter of the partial MTTKRP, all-gather of factor rows, all-reduce of
the last mode's Gram / dS / scalars).  The gathered fitness trace, MTTKRPs and factors must
equal a single-GPU run (P = 1) and the oracle within 1e-10 (-m gpu; skipped with < 2 GPUs)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-10
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(tmp_path, world, N, s, R, seed, mode="collective"):
    out = str(tmp_path / f"w{world}_N{N}_{mode}.npz")
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "nccl_worker.py"),
           out, str(N), str(s), str(R), str(seed), mode]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    if world > 1:   # NCCL's communicator-init lines name the rank count
        assert f"nranks {world}" in r.stdout + r.stderr
    return np.load(out)


@pytest.mark.parametrize("mode", ["collective", "fused"])
@pytest.mark.parametrize("N,s,R,seed", [(3, 64, 8, 41), (4, 16, 6, 42)])
def test_nccl_two_ranks_equal_single_rank_and_oracle(tmp_path, N, s, R, seed, mode):
    """mode "fused": opts.fused_rs -- the epilogue stores the partial MTTKRP rows into the owner's
    NCCL symmetric window (ncclMemAlloc + ncclCommWindowRegister, ncclGetPeerPointer) over NVLink."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2010_12056_b200 import build
    build.build()
    one = _run(tmp_path, 1, N, s, R, seed)
    two = _run(tmp_path, 2, N, s, R, seed, mode)
    assert np.all(np.abs(two["f"] - one["f"]) <= TOL * np.abs(one["f"]))
    assert np.linalg.norm(two["Mflat"] - one["Mflat"]) <= TOL * np.linalg.norm(one["Mflat"])
    assert np.linalg.norm(two["Aflat"] - one["Aflat"]) <= TOL * np.linalg.norm(one["Aflat"])
    cfg = synth.custom(N, s, R, noise_var=1e-4, seed=seed)
    T = O.make_tensor(cfg)
    A = synth.init_factors(cfg)
    for k in range(3):
        o = O.als_sweep(T, A)
        A = o["A"]
        assert abs(two["f"][k] - o["f"]) <= TOL * abs(o["f"])
