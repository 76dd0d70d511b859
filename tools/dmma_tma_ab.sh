#!/bin/bash
# FP64 DMMA engine: TMA-staged tiles (default) vs the cp.async staging (CPD_DMMA_NO_TMA=1), parity tests
# of the DMMA paths first, then bench lines of the DMMA engine on C2-C5, A/B on one box
TAG=${TAG:-r2i}
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ttm_dmma_tma or ttm_all_positions or msdt_and_dt_sweeps or large_rank or set_tensor or c1_full" > gpurun_out/dmma_tma_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/dmma_tma_tests_$TAG.log
for c in 2 4 3 5; do for off in 0 1; do
  CPD_DMMA_NO_TMA=$off timeout 600 python bench.py --config $c --ttm-impl dmma --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > gpurun_out/dmma_c${c}_notma${off}_$TAG.log 2>&1; echo "c$c notma=$off rc=$?"
  python - <<P
import json
for l in open("gpurun_out/dmma_c${c}_notma${off}_$TAG.log"):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print("C$c notma=$off msdt", round(d["value"], 3), "dt", round(d["sweeps_ms"]["dt"], 3), "ttm ms/launch", round(r.get("avg_launch_ms", 0), 4), "frac", round(r["frac"], 3), d["clocks"]["sm_mhz"])
P
done; done
