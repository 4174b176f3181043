"""Cycles per candidate-list fallback (row a3) of the shared-memory-table kernel, from a
-DMMAS_TRACE build (clock64 around every fallback selection, summed on the device).

    python tools/fb_cycles.py build                 # here: tools/libmmas_trace.so
    python tools/fb_cycles.py [C2] [first] [count]  # on the GPU: every variant, iterations
                                                    # first .. first+count-1 (default 5, 20),
                                                    # L2 flushed before each like bench.py

Variants (environment of a child process each): MMAS_FB_COMPACT caps from $CAPS (default
0,200,1008; 0 = the trip scans only); per-U buckets of cycles, phases of the compacted path."""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "tools", "libmmas_trace.so")


def child(cfg, first, count):
    os.environ["MMAS_LIB"] = SO
    import torch
    from paper_2003_11902_b200 import mmas
    from paper_2003_11902_b200.instances import CONFIGS
    w = CONFIGS[cfg]
    col = mmas.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed, device=0)
    L = mmas.lib()
    L.mmas_debug_fb_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    buf = (ctypes.c_ulonglong * 64)()
    if first:
        col.iterate(first)
    col.sync()
    L.mmas_debug_fb_cycles(buf)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ms = 0.0
    for _ in range(count):
        flush.zero_()
        torch.cuda.synchronize()
        ev[0].record(torch.cuda.ExternalStream(col.stream))
        col.iterate(1)
        ev[1].record(torch.cuda.ExternalStream(col.stream))
        col.sync()
        ms += ev[0].elapsed_time(ev[1])
    L.mmas_debug_fb_cycles(buf)
    cyc, cnt = buf[0], buf[1]
    buckets = {f"U<{16 << b}" if b < 7 else "U>=1024": [int(buf[40 + b]), round(buf[32 + b] / max(buf[40 + b], 1))]
               for b in range(8) if buf[40 + b]}
    nc = buf[16]
    compact = {"count": nc, "phases_count_keys_select": [round(buf[17 + k] / max(nc, 1)) for k in range(3)],
               "start_to_entry": round((buf[21] - buf[22]) / max(nc, 1))} if nc else None
    groups = {"hit": [int(buf[49]), round(buf[48] / max(buf[49], 1))], "clean": [int(buf[51]), round(buf[50] / max(buf[51], 1))]}
    print(json.dumps({"fallbacks": cnt, "cycles_per_fallback": cyc / max(cnt, 1), "by_unvisited": buckets, "groups": groups,
                      "compact": compact,
                      "fallbacks_per_tour": cnt / (count * w.n_ants), "ms_per_iteration": ms / count}))


def main():
    if sys.argv[1:2] == ["build"]:
        from paper_2003_11902_b200 import build as b
        cmd = [b.NVCC, *b.NVCC_FLAGS, "-DMMAS_TRACE", "-DMMAS_TRACE_GROUPS", "-I", os.path.join(ROOT, "include"), "-o", SO, *b.SOURCES]
        subprocess.run(cmd, check=True, capture_output=True)
        print(SO)
        return
    if sys.argv[1:2] == ["child"]:
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
        return
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    count = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    for cap in os.environ.get("CAPS", "0,200,1008").split(","):
        if True:
            env = dict(os.environ, MMAS_FB_COMPACT=cap)
            pf = cap
            out = subprocess.run([sys.executable, __file__, "child", cfg, str(first), str(count)], env=env,
                                 capture_output=True, text=True)
            print(f"{cfg} it {first}-{first + count - 1} MMAS_FB_COMPACT={pf}:",
                  out.stdout.strip() or out.stderr[-400:])


if __name__ == "__main__":
    main()
