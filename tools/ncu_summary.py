"""Summarise `ncu --set full` reports into profiles/ (text + traffic json for bench.py)."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum.per_second"]


def rows(rep):
    """Rows of an .ncu-rep (read with ncu -i) or of its raw-page CSV export."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    return [(dict(zip(hdr, x)), dict(zip(hdr, units))) for x in r[2:]]


def main(tag, reps):
    os.makedirs("profiles", exist_ok=True)
    traffic = {}
    tpath = "profiles/ncu_traffic.json"
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    with open(f"profiles/{tag}_ncu_full.txt", "w") as f:
        for name, rep in reps:
            per_launch = []  # DRAM bytes of each captured launch: the traffic entry is their mean
            for d, u in rows(rep):
                f.write(f"== {name}: {d.get('Kernel Name', '')[:120]}\n")
                for k in KEYS:
                    if k in d:
                        f.write(f"  {k:80s} {d[k]:>16s} {u.get(k, '')}\n")
                stalls = sorted(((k, float(v or 0)) for k, v in d.items()
                                 if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")),
                                key=lambda x: -x[1])[:6]
                f.write("  top stalls: " + ", ".join(f"{k[34:-23]}={v:.2f}" for k, v in stalls) + "\n")
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rb = float(d["dram__bytes_read.sum"]) * scale.get(u["dram__bytes_read.sum"], 1)
                wb = float(d["dram__bytes_write.sum"]) * scale.get(u["dram__bytes_write.sum"], 1)
                per_launch.append(rb + wb)
            if per_launch:
                traffic[name] = sum(per_launch) / len(per_launch)
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(open(f"profiles/{tag}_ncu_full.txt").read())


if __name__ == "__main__":
    tag = sys.argv[1]
    reps = [tuple(a.split("=", 1)) for a in sys.argv[2:]]
    main(tag, reps)
