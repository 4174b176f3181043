"""Ants-count sweep: construction time per iteration and
per-step cycles of one ant's warp as the colony grows from one warp per SM to many.
usage: python tools/ants_sweep.py [CFG] [m1,m2,...] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2003_11902_b200 import mmas  # noqa: E402
from paper_2003_11902_b200.instances import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
ms = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [148, 296, 592, 1002, 1480, 2960, 5920]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 50
warm = int(sys.argv[4]) if len(sys.argv) > 4 else 10   # steady state (few fallbacks) needs ~300
w = CONFIGS[cfg]
s = torch.cuda.current_stream().cuda_stream
sms = torch.cuda.get_device_properties(0).multi_processor_count
try:
    import pynvml
    pynvml.nvmlInit()
    mhz = pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM)
except Exception:
    mhz = 1965
print(f"{cfg}: n={w.n} cl={w.cand_len}; {sms} SMs, {mhz} MHz")
print(f"{'ants':>6} {'warps/SM':>8} {'construct ms':>12} {'cycles/step':>11} {'tours/s':>12} {'iter ms':>8}")
for m in ms:
    col = mmas.Colony(w.coords(), m, w.cand_len, rho=w.rho, seed=w.mmas_seed, stream=s,
                      local_search=bool(w.local_search), tabu=w.tabu, selection=w.selection)
    col.iterate(warm)
    fb0 = col.stats()["fallback_steps"]
    col.profile(True)
    col.iterate(iters)
    t = col.phase_times()
    it = t["iterations"]
    cons = t["construct_ms"] / it
    tot = (t["construct_ms"] + t["update_ms"] + t["select_ms"] + t["local_search_ms"]) / it
    fb = (col.stats()["fallback_steps"] - fb0) / (iters * m)
    print(f"{m:6d} {m / sms:8.2f} {cons:12.4f} {cons * 1e-3 * mhz * 1e6 / (w.n - 1):11.0f} {m / (tot * 1e-3):12,.0f} "
          f"{tot:8.4f}  fb/tour {fb:.2f}")
    col.close()
