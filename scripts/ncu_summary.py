"""Summarise an ncu report: key SOL/occupancy numbers, stall reasons, hottest SASS lines.
usage: python scripts/ncu_summary.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
print("kernel:", v[h.index("Kernel Name")] if "Kernel Name" in h else "?")
for name in want:
    if name in h:
        print(f"  {name:60s} {v[h.index(name)]} {raw[1][h.index(name)]}")
# every L2 / DRAM byte and sector counter of the capture (the memory-side roofline evidence)
for name, val, unit in zip(h, v, raw[1]):
    if name in want:
        continue
    if (name.startswith("lts__t_sectors") or name.startswith("lts__t_bytes") or name.startswith("dram__bytes")
            or name.startswith("lts__throughput") or name.startswith("l1tex__t_bytes")) and not name.endswith("_lookup_hit"):
        print(f"  {name:60s} {val} {unit}")
stalls = []
for name, val in zip(h, v):
    if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
        try:
            stalls.append((float(val), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(s for s, _ in stalls) or 1
print("stall samples:", " ".join(f"{n}={s / tot:.0%}" for s, n in sorted(stalls, reverse=True)[:10]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hdr = src[1]
rows = src[2:]
iS, iW, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
print(f"top {top} SASS by stall samples (samples, exec count, instr):")
base = int(rows[0][hdr.index("Address")], 16)
for r in sorted(rows, key=lambda r: -int(r[iW]))[:top]:
    print(f"  {int(r[hdr.index('Address')], 16) - base:05x} {r[iW]:>6} {r[iE]:>10}  {r[iS].strip()[:80]}")
