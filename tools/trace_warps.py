"""Finish time of every ant warp of one construct_cl_kernel launch by warp id (a -DMMAS_TRACE
build: %globaltimer when a warp finished its last ant), to see whether the scheduler pairs'
low-id warps (which lose the issue arbiter's priority) are the late ones.

    python tools/trace_phases.py build      # here: tools/libmmas_trace.so
    python tools/trace_warps.py [C2] [it]   # on the GPU"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MMAS_LIB"] = os.path.join(ROOT, "tools", "libmmas_trace.so")


def main(cfg, it):
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
    L = mmas.lib()
    L.mmas_debug_trace_warps.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    L.mmas_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    bw = (ctypes.c_ulonglong * (1024 * 16))()
    bb = (ctypes.c_ulonglong * (1024 * 8))()
    assert L.mmas_debug_trace_warps(bw, 1024 * 16) == 0 and L.mmas_debug_trace(bb, 1024 * 8) == 0
    tb = np.array(bb, dtype=np.int64).reshape(1024, 8)
    tw = np.array(bw, dtype=np.int64).reshape(1024, 16)
    used = tb[:, 0] > 0
    t0 = tb[used, 0].min()
    r = (tw[used] - t0) / 1000.0
    print(f"{cfg} iteration {it}: ant-warp finish times (us from the first block's entry) by warp id")
    for wid in range(16):
        col_ = r[:, wid]
        col_ = col_[col_ > 0]
        if len(col_):
            print(f"  warp {wid:2d} (scheduler {wid % 4}): n {len(col_):4d}  mean {col_.mean():7.1f}  "
                  f"p90 {np.percentile(col_, 90):7.1f}  max {col_.max():7.1f}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 400)
