"""One rank of the real-NCCL multi-GPU run (launched by tests/test_gpu_nccl.py under
torch.distributed.run): the 1-D grid of Alg. 3 / Alg. 4 through libcpd with world > 1 over
NCCL (ncclReduceScatter / ncclAllGather / grouped ncclAllReduce), the schedule of
test_gpu_multirank.schedule; rank 0 writes the gathered results to an .npz file."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2010_12056_b200 as cpd  # noqa: E402


def main():
    out_path, N, s, R, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    fused = len(sys.argv) > 6 and sys.argv[6] == "fused"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [cpd.cpd_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = synth.custom(N, s, R, noise_var=1e-4, seed=seed)
    lo, hi = synth.slab_range(cfg.s, rank, world)
    T = torch.empty([cfg.s] * (N - 1) + [hi - lo], dtype=torch.float64, device="cuda")
    cpd.cpd_gen_tensor(T, cfg.shape, lo, hi, 0, synth.true_factors(cfg), np.sqrt(cfg.noise_var), cfg.seed_noise)
    torch.cuda.synchronize()
    m = cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), device=local, rank=rank, world=world,
                        nccl_id=obj[0], stream=torch.cuda.Stream(), fused_rs=fused)
    f, M, A = [], [], []
    for _ in range(3):
        f.append(m.msdt_sweep())
        M.append([m.get_last_mttkrp(n) for n in range(N)])
    A.append([m.get_factor(n) for n in range(N)])
    m.pp_init()
    for _ in range(2):
        f.append(m.pp_approx_sweep()[0])
        M.append([m.get_last_mttkrp(n) for n in range(N)])
    f.append(m.msdt_sweep())
    f.append(m.dt_sweep())
    A.append([m.get_factor(n) for n in range(N)])
    m.close()
    if rank == 0:
        np.savez(out_path, f=np.array(f), M=np.array([np.stack(x) for x in M]) if N == 3 else np.zeros(1),
                 Mflat=np.concatenate([x.ravel() for ms in M for x in ms]),
                 Aflat=np.concatenate([x.ravel() for a in A for x in a]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
