#!/usr/bin/env python
"""Benchmark of the MSDT / PP CP-ALS hot path on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A STEP is one pass over every row of SURVEY §8(a) on the BASELINE workload
(default configs[1] = C2: 1024^3 FP64, exact rank 64 + N(0,1e-4) noise, R = 64):
    (N-1) msdt_sweep   = one full MSDT cycle (N roots for N-1 sweeps, §III)
    pp_init            = PP operators (Alg. 2 lines 6-9)
    (N-1) pp_approx_sweep (Alg. 2 lines 11-16, forced)
    1 dt_sweep         = the standard dimension-tree baseline (Fig. 1a)
`value` = device time per MSDT sweep (ms, the metric's first item); the PP-approx,
PP-init and DT per-sweep times are reported beside it.  For N > 1 the tensor is
split along its last mode (strong scaling, Alg. 3 / Alg. 4 on a 1-D grid); times
are the max over ranks.  T (8.6 GB for C2) is far larger than L2, so no flush is
needed between timed iterations.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "CP-ALS per-sweep time (MSDT, PP-approx) and TTM FP64-TC % / TTV HBM GB/s at 1-8 GPU"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {"hbm_gbs": 6650.0, "_source": "fallback (B200_PROFILING.md)"}


def fp64_peak():
    """Measured DMMA peak (profiles/r01_peaks_fp64.json, one JSON object); a missing or
    unparsable file is an error, not a silent fallback."""
    p = os.path.join(ROOT, "profiles", "r01_peaks_fp64.json")
    d = json.load(open(p))
    v = max(v for k, v in d.items() if k.startswith("dmma"))
    return float(v), "measured DMMA mma.sync.m8n8k4/m16n8k8 f64 (profiles/r01_peaks_fp64.json)"


def ncu_traffic(name):
    """dram bytes per launch from a committed `ncu --set full` summary, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(name)
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.out = ""

    def summary(self, t0=None, t1=None):
        """Samples whose timestamp falls inside [t0, t1] (wall clock of the timed region)."""
        import datetime
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if ts is not None and t0 is not None and not (t0 - 0.06 <= ts <= t1 + 0.06):
                continue
            f = f[1:]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def self_launch(n):
    """`python bench.py --gpus N` outside torchrun: re-run this command under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1; NCCL prints its
    communicator-init lines (nranks) to stderr."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_slab(cpd, torch, cfg, rank, world, stream):
    lo, hi = synth.slab_range(cfg.s, rank, world)
    T = torch.empty([cfg.s] * (cfg.N - 1) + [hi - lo], dtype=torch.float64, device="cuda")
    if cfg.kind == "uniform":
        cpd.cpd_gen_tensor(T, cfg.shape, lo, hi, 1, None, 0.0, cfg.seed_noise, stream)
    else:
        cpd.cpd_gen_tensor(T, cfg.shape, lo, hi, 0, synth.true_factors(cfg), math.sqrt(cfg.noise_var),
                           cfg.seed_noise, stream)
    return T


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def host_tensor(cfg, rows=None):
    """T on the host for the oracle timing legs, from the synth recipe: the Kruskal part of the
    true factors as (explicit KRP of modes 1..N-1) x A^(N)^T plus the counter-hash noise (or the
    U(0,1) entries), generated in parallel blocks of the leading mode.  `rows` restricts mode 1."""
    import oracle as O
    from concurrent.futures import ThreadPoolExecutor
    shape = list(cfg.shape)
    lo0, hi0 = (0, shape[0]) if rows is None else rows
    out = np.empty([hi0 - lo0] + shape[1:])
    At = synth.true_factors(cfg)
    inner = int(np.prod(shape[1:]))

    def block(i0):
        i1 = min(i0 + 8, hi0)
        idx = (np.arange(i0 * inner, i1 * inner, dtype=np.uint64))
        v = synth.element_noise(cfg, idx).reshape([i1 - i0] + shape[1:])
        if At is not None:
            krp = O.khatri_rao([At[0][i0:i1]] + At[1:-1])
            v += (krp @ At[-1].T).reshape(v.shape)
        out[i0 - lo0:i1 - lo0] = v

    with ThreadPoolExecutor(max_workers=cpu_cores()) as ex:
        list(ex.map(block, range(lo0, hi0, 8)))
    return out


def oracle_full_sweeps(cfg, n_sweeps):
    """The oracle's als_sweep (explicit unfolding + explicit KRP + Cholesky + Eq. 3) on the FULL
    tensor of `cfg`, n_sweeps times from the seeded initial factors; per-sweep seconds."""
    import oracle as O
    from threadpoolctl import threadpool_limits
    cores = cpu_cores()
    T = host_tensor(cfg)
    A = synth.init_factors(cfg)
    nt2 = O.norm2(T)
    ts = []
    with threadpool_limits(limits=cores):
        for _ in range(n_sweeps):
            t0 = time.perf_counter()
            out = O.als_sweep(T, A, nt2)
            ts.append(time.perf_counter() - t0)
            A = out["A"]
    return ts, cores


def cpu_baseline(cfg, n_sweeps):
    ts, cores = oracle_full_sweeps(cfg, n_sweeps)
    return {"value": 1e3 * statistics.mean(ts), "unit": "ms/sweep (MSDT)", "cores": cores, "kind": "oracle",
            "sample": f"{n_sweeps} full oracle als_sweep on the whole {cfg.name} tensor "
                      f"({'x'.join(map(str, cfg.shape))}, R={cfg.R}; explicit unfolding + explicit KRP + "
                      f"Cholesky + Eq. 3), mean per sweep; per-sweep s: {[round(t, 2) for t in ts]}"}


def workload_config(cfg, world):
    """The `config` object of both arms (identical, static; run state goes elsewhere)."""
    return {"workload": cfg.name, "N": cfg.N, "s": cfg.s, "R": cfg.R,
            "tensor": f"exact rank {cfg.true_rank} + N(0,{cfg.noise_var}) noise" if cfg.kind == "kruskal"
            else "i.i.d. U(0,1)", "parallelism": f"1-D split of mode N over {world} GPU(s)",
            "step": f"{cfg.N - 1} msdt_sweep + pp_init + {cfg.N - 1} pp_approx_sweep + 1 dt_sweep",
            "l2": "inputs larger than L2 (no flush)"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands (the tier's reference arm), rank 0 only.
    A step is one mode update of the oracle's als_sweep on the FULL tensor (explicit unfolding,
    explicit KRP, Cholesky solve, Gram), cycling through the modes, so N consecutive steps are one
    full sweep; `value` = mean step time x N = ms per full sweep, measured over whole sweeps."""
    if rank != 0:
        return
    import oracle as O
    from threadpoolctl import threadpool_limits
    cfg = synth.config(args.config)
    N = cfg.N
    cores = cpu_cores()
    T = host_tensor(cfg)
    A = synth.init_factors(cfg)
    nt2 = O.norm2(T)
    S = [O.gram(a) for a in A]
    ts = []
    with threadpool_limits(limits=cores):
        for it in range(args.warmup + args.steps):
            n = it % N
            t0 = time.perf_counter()
            G = O.gamma(S, n)
            M = O.mttkrp(T, A, n)
            A[n] = O.solve(G, M)
            S[n] = O.gram(A[n])
            if n == N - 1:
                O.fitness_eq3(nt2, G, S[n], M, A[n])
            dt = time.perf_counter() - t0
            if it >= args.warmup:
                ts.append(dt)
    per_mode = {}
    for k, t in enumerate(ts):
        per_mode.setdefault((args.warmup + k) % N, []).append(t)
    per_sweep_ms = 1e3 * sum(statistics.mean(v) for v in per_mode.values()) * N / len(per_mode)
    step_ms = 1e3 * statistics.mean(ts)
    line = {
        "impl": "reference", "metric": METRIC, "value": per_sweep_ms, "unit": "ms/sweep (MSDT)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, world),
        "cpu_baseline": {"value": per_sweep_ms, "unit": "ms/sweep (MSDT)", "cores": cores, "kind": "oracle",
                         "sample": f"each step = one mode update of the oracle als_sweep (explicit unfolding + "
                                   f"explicit KRP + Cholesky + Gram) on the full {'x'.join(map(str, cfg.shape))} "
                                   f"tensor, modes cycling; value = mean step time per mode summed over the "
                                   f"{N} modes (ms per full sweep)"},
        "e2e": {"value": per_sweep_ms, "unit": "ms/sweep (MSDT)", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


TTM_IMPL = {"dmma": 0, "int8": 1, "auto": 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, help="BASELINE.json configs[c-1]")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--presweeps", type=int, default=60, help="max untimed MSDT sweeps before the steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dmma-compare", action="store_true", help="skip the FP64-DMMA engine comparison cycles")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sweeps", type=int, default=3, help="full oracle sweeps timed for cpu_baseline")
    ap.add_argument("--ttm-impl", default="auto", choices=["dmma", "int8", "auto"],
                    help="first-level TTM engine: FP64 DMMA, FP64 operands as int8 digits on tcgen05, or the "
                         "library's choice (int8 when its error bound is FP64-class)")
    ap.add_argument("--msdt-levels", type=int, default=1,
                    help="upper-level fusion (P:700-702): modes each MSDT root contracts at once (1 = MSDT)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    world, rank, local = dist_setup(args)
    if "WORLD_SIZE" in os.environ and args.gpus != world and rank == 0:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: measuring {world} rank(s)", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2010_12056_b200 as cpd

    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")        # communicator init lines (nranks) on stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    cfg = synth.config(args.config)
    N = cfg.N
    peaks = load_peaks()
    fp64, fp64_src = fp64_peak()

    nccl_id = None
    if world > 1:
        obj = [cpd.cpd_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    with torch.cuda.stream(stream):
        T = make_slab(cpd, torch, cfg, rank, world, stream)
    torch.cuda.synchronize()
    A0 = synth.init_factors(cfg)
    m = cpd.cp_als_init(T, cfg.shape, cfg.R, A0, device=local, rank=rank, world=world, nccl_id=nccl_id,
                        stream=stream, pp_eps=0.2 if args.config == 4 else 0.1, profile_phases=1,
                        ttm_impl=TTM_IMPL[args.ttm_impl], msdt_levels=args.msdt_levels)
    # untimed: converge until the PP entry condition holds (Alg. 2 line 5), so the forced
    # PP sweeps of each step run in their regime of validity
    pre = 0
    f = None
    while pre < args.presweeps:
        f = m.msdt_sweep()
        pre += 1
        if m.pp_condition():
            break
    pp_ok = m.pp_condition()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def one_step(rec):
        e0 = ev()
        for _ in range(N - 1):
            m.msdt_sweep()
        e1 = ev()
        m.pp_init()
        e2 = ev()
        for _ in range(N - 1):
            m.pp_approx_sweep()
        e3 = ev()
        m.dt_sweep()
        e4 = ev()
        rec.append((e0, e1, e2, e3, e4))

    junk = []
    clk = Clocks(local).__enter__()   # sampler starts before the warm-up so the timed region is covered
    for _ in range(args.warmup):
        one_step(junk)
    torch.cuda.synchronize()
    m.reset_counters()
    launches0 = m.counters()["kernel_launches"]
    recs = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if True:
        wall0 = time.time()
        t_start = ev()
        for _ in range(args.steps):
            one_step(recs)
        t_end = ev()
        torch.cuda.synchronize()
        wall1 = time.time()
    clk.__exit__(None, None, None)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    parts = np.array([[a.elapsed_time(b) for a, b in zip(r[:-1], r[1:])] for r in recs])  # steps x 4
    ph = m.phase_ms()
    ctr = m.counters()
    fill = m.filler_counters()
    aux_mem = m.get_memory()
    launches = int(ctr["kernel_launches"] - launches0)
    part_means = parts.mean(axis=0)
    vals = np.array([total_ms, part_means[0] / (N - 1), part_means[1], part_means[2] / (N - 1), part_means[3]])
    if world > 1:
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vals = t.cpu().numpy()
    total_ms, msdt_ms, ppinit_ms, ppapprox_ms, dt_ms = vals.tolist()

    # roofline of the dominant kernel (the first-level TTM on DMMA) and of the streams
    ttm_launch_flops = ctr["ttm_flops"] / max(ctr["ttm_launches"], 1)
    ttm_ms = ph["ttm"] / max(ctr["ttm_launches"], 1)
    ttm_tf = ttm_launch_flops / (ttm_ms * 1e-3) / 1e12 if ttm_ms > 0 else None
    st_launch_bytes = ctr["stream_bytes"] / max(ctr["stream_launches"], 1)
    st_ms = ph["mttv"] / max(ctr["stream_launches"], 1)
    st_gbs = st_launch_bytes / (st_ms * 1e-3) / 1e9 if st_ms > 0 else None
    # P:748 breakdown from two extra, untimed steps with every phase bracketed
    m.set_profile_level(2)
    m.reset_counters()
    for _ in range(2):
        one_step([])
    torch.cuda.synchronize()
    ph_all = m.phase_ms()
    m.set_profile_level(1)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cpd, torch, cfg, T, m, rank, world, local, nccl_id, stream)

    cpu = None

    engine = m.ttm_engine()
    if engine == "dmma":
        ttm_roof = dmma_roof(ttm_tf, fp64, fp64_src, ttm_launch_flops, ttm_ms, ctr)
        engines = None
    else:
        # int8-digit TTM: streams T's 7 digit planes (7 B/element) and writes the FP64 root; its
        # MMAs are 28 exact int8 digit-pair products per FP64 multiply-add.  Both
        # roofs are computed; the primary `bound` is the one the launch is closer to (the binding
        # roof), the other is kept beside it.
        t_el = ttm_launch_flops / (2 * cfg.R)
        # algorithmic bytes per launch from the library's ledger (cpd_get_ttm_bytes): T's digits once,
        # the FP64 output once, the factor's digit image -- first-level TTMs and block roots alike
        ttm_bytes = ctr["ttm_bytes"] / max(ctr["ttm_launches"], 1)
        ttm_gbs = ttm_bytes / (ttm_ms * 1e-3) / 1e9 if ttm_ms > 0 else None
        hbm = {"bound": "hbm", "achieved": ttm_gbs, "peak": peaks.get("hbm_gbs"),
               "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)", "unit": "GB/s",
               "frac": (ttm_gbs / peaks["hbm_gbs"]) if ttm_gbs and peaks.get("hbm_gbs") else None,
               "bytes_per_launch": ttm_bytes}
        # int8 peak = measured bf16 x the nominal int8/bf16 ratio 2 (sustained figure: the TTM runs
        # inside a long step)
        i8_ops = 28.0 * 2.0 * t_el * cfg.R
        i8_tops = i8_ops / (ttm_ms * 1e-3) / 1e12 if ttm_ms > 0 else None
        i8_peak = 2.0 * peaks["bf16_tflops_sustained"] if peaks.get("bf16_tflops_sustained") else None
        tensor = {"bound": "tensor", "achieved": i8_tops, "peak": i8_peak, "unit": "TOP/s",
                  "frac": (i8_tops / i8_peak) if i8_tops and i8_peak else None, "ops_per_launch": i8_ops,
                  "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops_sustained (nominal int8:bf16 = 2)"}
        prim, sec = (tensor, hbm) if (tensor["frac"] or 0) >= (hbm["frac"] or 0) else (hbm, tensor)
        ttm_roof = {"kernel": f"ttm_i8 ({engine}: first-level TTM, FP64 operands as exact int8 digit products, "
                              "tcgen05.mma kind::i8, TMEM accumulators)", **prim,
                    "traffic": ncu_traffic("ttm_i8d" if args.config == 2 else f"c{args.config}_ttm"),
                    "traffic_source": "dram bytes per launch, profiles/ncu_traffic.json (ncu --set full)",
                    "secondary": sec, "bytes_per_launch": ttm_bytes,
                    "fp64_equiv_tflops": ttm_tf, "fp64_equiv_over_dmma_peak": (ttm_tf / fp64) if ttm_tf else None,
                    "avg_launch_ms": ttm_ms, "launches": int(ctr["ttm_launches"])}
        if args.msdt_levels > 1:
            ttm_roof["note"] = ("msdt_levels > 1: the MSDT roots are block contractions (output s^(N-l) R); the "
                                "launch average mixes them with the first-level TTMs of pp_init and dt_sweep")
        engines = {engine: {"msdt_ms_per_sweep": msdt_ms, "ttm_ms": ttm_ms, "ttm_fp64_equiv_tflops": ttm_tf}}
        if not args.no_dmma_compare:
            engines["dmma"] = dmma_compare(cpd, torch, cfg, T, m, local, rank, world, nccl_id, stream, fp64, fp64_src)
    m.close()
    # the oracle on the host cores, after every GPU measurement (rank 0; other ranks wait)
    if rank == 0 and not args.no_cpu_baseline:
        if 8 * cfg.numel > 40e9:   # C5: the oracle's full sweep needs ~2x 69 GB of host memory
            cpu = {"value": None, "unit": "ms/sweep (MSDT)", "cores": cpu_cores(), "kind": "oracle",
                   "sample": "skipped: the full tensor exceeds the host budget of the timing leg"}
        else:
            cpu = cpu_baseline(cfg, args.cpu_sweeps)
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": msdt_ms, "unit": "ms/sweep (MSDT)", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, world),
            "state": {"presweeps": pre, "pp_condition_held": pp_ok, "fitness_before_steps": f,
                      "ttm_impl": args.ttm_impl, "msdt_levels": args.msdt_levels,
                      "aux_memory_bytes": aux_mem},
            "sweeps_ms": {"msdt": msdt_ms, "pp_approx": ppapprox_ms, "pp_init": ppinit_ms, "dt": dt_ms,
                          "dt_over_msdt": dt_ms / msdt_ms, "dt_over_pp_approx": dt_ms / ppapprox_ms},
            "phase_ms_per_step": {k: v / 2 for k, v in ph_all.items()},
            "roofline": ttm_roof, "ttm_engine": engine, "engines": engines,
            "roofline_stream": {"kernel": "mttv (mTTV levels + PP U-stream)", "bound": "hbm", "achieved": st_gbs,
                                "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                                "frac": (st_gbs / peaks["hbm_gbs"]) if st_gbs and peaks.get("hbm_gbs") else None,
                                "traffic": ncu_traffic("mttv" if args.config == 2 else f"c{args.config}_mttv"),
                                "bytes_per_launch": st_launch_bytes,
                                "avg_launch_ms": st_ms, "launches": int(ctr["stream_launches"]),
                                "scope": "main-stream launches (timed); the PP filler-stream launches overlap "
                                         "them and are ledgered separately (pp_filler_streams)"},
            "pp_filler_streams": {"bytes_per_step": fill["bytes"] / args.steps,
                                  "launches_per_step": fill["launches"] / args.steps},
            "roofline_pp_sweep": pp_sweep_roof(cfg, world, ppapprox_ms, peaks),
            "gpu_launches": launches, "clocks": clk.summary(wall0, wall1), "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pp_sweep_roof(cfg, world, pp_ms, peaks):
    """A PP-approximated sweep as a whole (Eqs. 5-6): every pair operator M_p^(a,b)
    ([s_a, s_b, R], the last mode's extent split over the ranks of the 1-D grid) is streamed twice
    per sweep (once for each of its two modes), 8 bytes per element, plus the dA reads and M~
    writes -- SURVEY §8(d)'s 8·N(N-1)·s²R leading term -- over the measured sweep time, against the
    HBM copy peak.  Main- and filler-stream launches overlap, so this is the honest per-sweep roof."""
    N, R = cfg.N, cfg.R
    ext = list(cfg.shape[:-1]) + [cfg.shape[-1] // world]
    b = 0.0
    for n in range(N):
        for i in range(N):
            if i != n:
                b += 8.0 * (ext[n] * ext[i] * R + ext[i] * R)
        b += 8.0 * 2 * ext[n] * R
    gbs = b / (pp_ms * 1e-3) / 1e9 if pp_ms > 0 else None
    return {"bound": "hbm", "bytes_per_sweep": b, "ms_per_sweep": pp_ms, "achieved": gbs, "peak": peaks.get("hbm_gbs"),
            "unit": "GB/s", "frac": (gbs / peaks["hbm_gbs"]) if gbs and peaks.get("hbm_gbs") else None}


def dmma_roof(ttm_tf, fp64, fp64_src, flops, ms, ctr):
    return {"kernel": "ttm_dmma_tma (first-level TTM, DMMA.8x8x4, TMA-staged swizzled tiles)", "bound": "tensor", "achieved": ttm_tf,
            "peak": fp64, "peak_source": fp64_src, "unit": "TFLOP/s", "frac": (ttm_tf / fp64) if ttm_tf else None,
            "traffic": ncu_traffic("ttm_dmma"), "flops_per_launch": flops, "avg_launch_ms": ms,
            "launches": int(ctr["ttm_launches"])}


def dmma_compare(cpd, torch, cfg, T, m, local, rank, world, nccl_id, stream, fp64, fp64_src):
    """The FP64 DMMA engine on the same tensor and factors (north_star's TTM FP64-TC %): two
    warm-up MSDT cycles, then three timed cycles (median); CUDA events on the caller's stream."""
    import torch.distributed as dist
    N = cfg.N
    A = [m.get_factor(n) for n in range(N)]
    md = cpd.cp_als_init(T, cfg.shape, cfg.R, A, device=local, rank=rank, world=world,
                         nccl_id=nccl_id if world == 1 else _new_id(cpd, dist, rank), stream=stream,
                         profile_phases=1, ttm_impl=TTM_IMPL["dmma"])
    for _ in range(2 * (N - 1)):
        md.msdt_sweep()
    torch.cuda.synchronize()
    md.reset_counters()
    # whole cycles, each bracketed by events; the median cycle (a second context shares the
    # device memory pool with the first, so a cycle may pay a one-off pool growth)
    cyc = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(N - 1):
            md.msdt_sweep()
        e1.record(stream)
        torch.cuda.synchronize()
        cyc.append(e0.elapsed_time(e1) / (N - 1))
    ms = float(np.median(cyc))
    ph, ctr = md.phase_ms(), md.counters()
    md.close()
    flops = ctr["ttm_flops"] / max(ctr["ttm_launches"], 1)
    tms = ph["ttm"] / max(ctr["ttm_launches"], 1)
    tf = flops / (tms * 1e-3) / 1e12 if tms > 0 else None
    return {"msdt_ms_per_sweep": ms, "ttm_ms": tms, "ttm_fp64_tflops": tf,
            "roofline": dmma_roof(tf, fp64, fp64_src, flops, tms, ctr)}


def run_e2e(args, cpd, torch, cfg, T, m, rank, world, local, nccl_id, stream):
    """Same metric through the public API with HOST buffers: per step, H2D of the
    tensor slab and of the factors from pinned memory, one MSDT cycle ((N-1) sweeps),
    D2H of every factor and the fitness.  e2e value = step time / (N-1) sweeps."""
    import torch.distributed as dist
    N = cfg.N
    A_host = [m.get_factor(n) for n in range(N)]
    T_host = torch.empty(T.shape, dtype=torch.float64, pin_memory=True)
    T_host.copy_(T)
    T_dev = torch.empty_like(T)
    T_dev.copy_(T)
    m2 = cpd.cp_als_init(T_dev, cfg.shape, cfg.R, A_host, device=local, rank=rank, world=world,
                         nccl_id=nccl_id if world == 1 else _new_id(cpd, dist, rank), stream=stream,
                         ttm_impl=TTM_IMPL[args.ttm_impl])
    outs = [np.empty((cfg.s, cfg.R)) for _ in range(N)]
    pinned_A = [torch.from_numpy(a).pin_memory().numpy() for a in A_host]
    ts = []
    for it in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            T_dev.copy_(T_host, non_blocking=True)
        m2.set_tensor()            # new tensor contents: ||T||^2, exponent, digit planes
        m2.set_factors(pinned_A)
        for _ in range(N - 1):
            m2.msdt_sweep()
        for n in range(N):
            m2.get_factor(n, outs[n])
        m2.fitness()
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= args.warmup:
            ts.append(e0.elapsed_time(e1))
    v = statistics.mean(ts) / (N - 1)
    if world > 1:
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v = float(t.item())
    m2.close()
    h2d = T_host.numel() * 8 + sum(a.size * 8 for a in A_host)
    d2h = sum(a.size * 8 for a in A_host) + 8
    return {"value": v, "unit": "ms/sweep (MSDT)", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "step": f"H2D T slab + factors (pinned), cpd_set_tensor, {N - 1} msdt_sweep, D2H factors + fitness"}


def _new_id(cpd, dist, rank):
    obj = [cpd.cpd_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


if __name__ == "__main__":
    main()
