"""Collect per-launch numbers from ncu --set full captures into profiles/ncu_traffic.json
(read by bench.py for roofline.traffic and the issue roofline).

usage: python scripts/ncu_json.py [--out FILE] CONFIG:KERNEL:report.ncu-rep [...]
KERNEL is the key bench.py looks up (e.g. construct_cl_kernel, pheromone_update_kernel)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
WANT = {"dram__bytes_read.sum": "dram_bytes_read", "dram__bytes_write.sum": "dram_bytes_write",
        "smsp__inst_executed.sum": "inst_executed", "gpu__time_duration.sum": "duration", "sm__inst_executed.sum": "sm_inst_executed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
        "lts__t_bytes.sum": "l2_bytes", "lts__t_sectors_op_read.sum": "l2_sectors_read",
        "lts__t_sectors_op_write.sum": "l2_sectors_write", "lts__t_sectors_op_atom.sum": "l2_sectors_atom",
        "lts__t_sectors_op_red.sum": "l2_sectors_red", "sm__cycles_elapsed.avg": "sm_cycles"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "ns": 1e-3, "us": 1, "usecond": 1,
         "ms": 1e3, "msecond": 1e3, "%": 1, "": 1, "sector": 1, "Ksector": 1e3, "Msector": 1e6, "cycle": 1,
         "Kcycle": 1e3, "Mcycle": 1e6}


def main():
    args = sys.argv[1:]
    out = OUT
    if args and args[0] == "--out":
        out, args = args[1], args[2:]
    d = json.load(open(out)) if os.path.exists(out) else {}
    srcs = []
    for arg in args:
        cfg, kern, rep = arg.split(":", 2)
        if rep.endswith(".txt"):   # a scripts/ncu_summary.py digest: "  metric  value unit" lines
            h, units, v = [], [], []
            for line in open(rep):
                parts = line.split()
                if len(parts) >= 2 and parts[0] in WANT:
                    h.append(parts[0])
                    v.append(parts[1])
                    units.append(parts[2] if len(parts) > 2 else "")
        else:
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            rows = list(csv.reader(io.StringIO(raw)))
            h, units, v = rows[0], rows[1], rows[2]
        e = {}
        for name, key in WANT.items():
            if name in h:
                i = h.index(name)
                val = float(v[i].replace(",", ""))
                if key == "duration":
                    e["duration_us"] = val * SCALE.get(units[i], 1)
                else:
                    e[key] = val * SCALE.get(units[i], 1)
        for k in ("dram_bytes_read", "dram_bytes_write", "inst_executed", "l2_bytes", "l2_sectors_read",
                  "l2_sectors_write", "l2_sectors_atom", "l2_sectors_red"):
            if k in e:
                e[k] = int(round(e[k]))
        d.setdefault(cfg, {})[kern] = e
        srcs.append(os.path.relpath(rep, ROOT))
    d["source"] = ("ncu --set full --clock-control none captures (one launch each): " +
                   ", ".join(sorted(set(srcs) | set(d.get("_reps", [])))) +
                   "; dram__bytes_read/write.sum, smsp__inst_executed.sum (warp instructions), "
                   "gpu__time_duration.sum per launch")
    d["_reps"] = sorted(set(srcs) | set(d.get("_reps", [])))
    json.dump(d, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(d, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
