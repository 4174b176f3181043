"""Phase timeline of one construct_cl_kernel launch (construction, selection, grid barrier,
fused update), from %globaltimer stamps of a -DMMAS_TRACE build of the library.

    python tools/trace_phases.py build          # here: tools/libmmas_trace.so (nvcc, sm_100a)
    python tools/trace_phases.py [C1|C2] [it]   # on the GPU: iteration `it` (default 400)

Prints, relative to the earliest block entry: the latest table-staged time, the spread of
the blocks' construction end, the last block's selection end, the barrier release and the
kernel end."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tools", "libmmas_trace.so")
sys.path.insert(0, ROOT)


def build():
    from paper_2003_11902_b200 import build as b
    cmd = [b.NVCC, *b.NVCC_FLAGS, "-DMMAS_TRACE", "-I", os.path.join(ROOT, "include"), "-o", SO, *b.SOURCES]
    subprocess.run(cmd, check=True, capture_output=True)
    print(SO)


def run(cfg, it):
    os.environ["MMAS_LIB"] = SO
    import numpy as np
    import torch
    from paper_2003_11902_b200 import mmas
    from paper_2003_11902_b200.instances import CONFIGS
    w = CONFIGS[cfg]
    col = mmas.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed, device=0)
    col.iterate(it)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    flush.zero_()
    torch.cuda.synchronize()
    col.iterate(1)
    col.sync()
    buf = (ctypes.c_ulonglong * (1024 * 8))()
    assert mmas.lib().mmas_debug_trace(buf, 1024 * 8) == 0
    t = np.array(buf, dtype=np.int64).reshape(1024, 8)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    r = (t - t0) / 1000.0   # us
    print(f"{cfg} iteration {it}: {len(t)} blocks (us from the first block's entry)")
    print(f"  entry spread               {r[:, 0].max():8.2f}")
    print(f"  table staged (max)         {r[:, 1].max():8.2f}")
    print(f"  warp 0 done min/med/max    {r[:, 2].min():8.2f} {np.median(r[:, 2]):8.2f} {r[:, 2].max():8.2f}")
    print(f"  block_finish done (max)    {r[:, 3].max():8.2f}   (the last block: + selection)")
    print(f"  barrier released (max)     {r[:, 4].max():8.2f}")
    print(f"  end (max)                  {r[:, 5].max():8.2f}")
    print("  (timestamps of a trace build: its instruction schedule differs from the production build)")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "build":
        build()
    else:
        run(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 400)
