"""Rounds of the cooperative 2-opt (row a8) and how many evaluations each retires or discards
behind its winner, from a -DMMAS_TRACE build (tools/fb_cycles.py build):

    python tools/ls_rounds.py [C5] [iterations]"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MMAS_LIB"] = os.path.join(ROOT, "tools", "libmmas_trace.so")
from paper_2003_11902_b200 import mmas  # noqa: E402
from paper_2003_11902_b200.instances import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = CONFIGS[cfg]
col = mmas.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed, local_search=True, device=0)
L = mmas.lib()
L.mmas_debug_fb_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
buf = (ctypes.c_ulonglong * 16)()
col.sync()
L.mmas_debug_fb_cycles(buf)
col.iterate(iters)
col.sync()
L.mmas_debug_fb_cycles(buf)
st = col.stats()
rounds, ret, disc = buf[2], buf[3], buf[4]
print(json.dumps({"config": cfg, "iterations": iters, "rounds_per_tour": rounds / (iters * w.n_ants),
                  "retired_per_round": ret / max(rounds, 1), "discarded_per_round": disc / max(rounds, 1),
                  "moves_per_tour": st["local_search_moves"] / (iters * w.n_ants),
                  "reversal_len_log2_hist": list(buf[5:15]),
                  "mean_reversal_len": buf[15] / max(sum(buf[5:15]), 1)}))
