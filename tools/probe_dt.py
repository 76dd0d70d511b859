import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2010_12056_b200 as cpd
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = synth.config(c)
T = torch.empty(cfg.shape, dtype=torch.float64, device="cuda")
if cfg.kind == "uniform":
    cpd.cpd_gen_tensor(T, cfg.shape, 0, cfg.s, 1, None, 0.0, cfg.seed_noise)
else:
    cpd.cpd_gen_tensor(T, cfg.shape, 0, cfg.s, 0, synth.true_factors(cfg), np.sqrt(cfg.noise_var), cfg.seed_noise)
m = cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), profile_phases=2)
def t(f, name):
    torch.cuda.synchronize(); m.reset_counters(); t0 = time.perf_counter(); f(); dt = time.perf_counter() - t0
    ph = m.phase_ms(); print(f"{name:10s} wall {dt*1e3:8.2f} ms  phases {sum(ph.values()):8.2f} ms  {ph}")
for _ in range(2): t(m.msdt_sweep, "msdt")
for _ in range(3): t(m.dt_sweep, "dt")
for _ in range(3): t(m.msdt_sweep, "msdt")
t(m.pp_init, "pp_init")
for _ in range(2): t(m.pp_approx_sweep, "pp")
for _ in range(2): t(m.dt_sweep, "dt")
