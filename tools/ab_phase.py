"""A/B timing of the iteration variants on one GPU (fused select vs split path)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = CONFIGS[cfg]
s = torch.cuda.current_stream().cuda_stream
for variant in ("fused", "split", "fused", "split"):
    col = mmas.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed, stream=s)
    rec = torch.zeros(col.record_bytes, dtype=torch.uint8, device="cuda")
    def step():
        if variant == "fused":
            col.iterate(1)
        else:
            col.construct(rec.data_ptr()); col.update(rec.data_ptr(), 1)
    for _ in range(20): step()
    torch.cuda.synchronize()
    col.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(300): step()
    e1.record(); torch.cuda.synchronize()
    t = col.phase_times(); it = t["iterations"]
    print(f"{cfg} {variant:6s} step {e0.elapsed_time(e1)/300*1e3:7.1f} us  construct {t['construct_ms']/it*1e3:7.1f}  select {t['select_ms']/it*1e3:5.1f}  update {t['update_ms']/it*1e3:5.1f}  fb/tour {col.stats()['fallback_steps']/col.stats()['iterations']/w.n_ants:.2f}")
    col.close()
