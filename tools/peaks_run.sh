#!/bin/bash
# one-off: FP64 peaks on the B200 box
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/peaks_fp64 > gpurun_out/peaks_fp64.json 2>&1
python - >> gpurun_out/peaks_fp64.json 2>&1 <<'PY'
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(2): c = a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print('{"cublas_dgemm_8192_tflops": %.2f}' % (2 * 8192**3 / best / 1e9))
PY
kill $SMI
nproc >> gpurun_out/peaks_fp64.json; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/peaks_fp64.json; free -g >> gpurun_out/peaks_fp64.json
