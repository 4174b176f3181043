"""Timing of the iteration phases on one GPU (per-phase events) and of plain
back-to-back iterations (no events between kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2003_11902_b200 import mmas  # noqa: E402
from paper_2003_11902_b200.instances import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
tabu = 0
if cfg.endswith(":ct"):   # full-row configs over the compact tabu (R27)
    cfg, tabu = cfg[:-3], mmas.TABU_COMPACT
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
w = CONFIGS[cfg]
s = torch.cuda.current_stream().cuda_stream
col = mmas.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed, stream=s,
                  local_search=bool(w.local_search), tabu=max(tabu, w.tabu), selection=w.selection)
col.iterate(20)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
col.iterate(iters)
e1.record()
torch.cuda.synchronize()
plain = e0.elapsed_time(e1) / iters * 1e3
col.profile(True)
col.iterate(iters)
t = col.phase_times()
it = t["iterations"]
st = col.stats()
print(f"{cfg} plain step {plain:8.1f} us | profiled: construct {t['construct_ms'] / it * 1e3:8.1f}  "
      f"update {t['update_ms'] / it * 1e3:6.1f}  ls {t['local_search_ms'] / it * 1e3:8.1f}  "
      f"fb/tour {st['fallback_steps'] / st['iterations'] / w.n_ants:.2f}  tours/s {w.n_ants / plain * 1e6:,.0f}")
