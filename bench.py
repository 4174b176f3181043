"""bench.py -- candidate tours/s of the MMAS hot path on synthetic pr1002-shaped
instances (BASELINE.json metric), 1..8 B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step = one full MMAS iteration: every ant of
the colony builds a tour, the iteration/global best is selected (with the
all-gather exchange for N > 1) and the pheromone update runs.  Weak scaling:
each GPU builds n_ants (1002 for C2) per step; value = all ranks' tours / the
max-over-ranks device time.  L2 is flushed (256 MiB write) between timed steps,
outside the per-step CUDA-event intervals.

--impl reference times the CPU oracle (oracle/) on the host
cores on a bounded sample of the same workload; it is the slow baseline, not
the product.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2003_11902_b200.instances import CONFIGS  # noqa: E402

METRIC = "candidate tours/sec (pr1002-shaped, 1/2/4/8 B200) and % L2/HBM roofline"
UNIT = "tours/s"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6454.0), "measured"
    return 6650.0, "fallback"


def onchip_peaks():
    """Measured L2 / shared-memory read bandwidth (tools/onchip_peaks.cu, committed in
    profiles/onchip_peaks.json); None if absent."""
    p = os.path.join(ROOT, "profiles", "onchip_peaks.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": sorted(self.reasons)}


def ncu_entry(config, kernel, iteration=None):
    """Per-launch numbers of the committed ncu --set full capture (profiles/ncu_traffic.json,
    written by scripts/ncu_json.py) of this config and kernel, from the capture whose
    iteration is nearest `iteration` (keys "C2@10", "C2@400": the fallback rate -- and so the
    instruction count -- depends on the iteration), else the un-keyed one; (entry, key) or
    (None, None)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None, None
    keyed = []
    for k, v in d.items():
        if k.startswith(config + "@") and isinstance(v, dict) and kernel in v:
            try:
                keyed.append((int(k.split("@", 1)[1]), k))
            except ValueError:
                pass
    if keyed and iteration is not None:
        _, k = min(keyed, key=lambda t: abs(t[0] - iteration))
        return d[k][kernel], k
    if config in d and kernel in d[config]:
        return d[config][kernel], config
    return None, None


def ncu_traffic(ent):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) or None."""
    return None if ent is None else ent["dram_bytes_read"] + ent["dram_bytes_write"]


# the paper's construction-only numbers for the same instance shape (other hardware: context)
PAPER_CONTEXT = {
    "C1": "V100 d198 WRS-BT cl=32 construction 0.19 ms -> 1.04M tours/s (T6 P:1549); ours uses cl=16",
    "C2": "V100 pr1002 WRS-BT cl=32 construction 0.93 ms -> 1.08M tours/s (T6 P:1549)",
    "C2RWM": "the paper's RWM variants are slower than WRS on every instance (T3-T6, P:1269-1273)",
    "C3": "V100 fl3795 WRS-BT cl=32 construction 12.65 ms -> 300k tours/s (T6 P:1549)",
    "C4": "V100 pr2392 WRS-BT full row 52.54 ms -> 46k tours/s (T4 P:1418)",
    "C4CT": "V100 pr2392 WRS-CT full row 39.24 ms -> 61k tours/s (T4 P:1419)",
    "C4RWM": "the paper's RWM variants are slower than WRS on every instance (T3-T4)",
    "C4RWMCT": "the paper's RWM variants are slower than WRS on every instance (T3-T4)",
    "C5": "d18512 with 2-opt: total runtime only in the paper (T9 P:1821), no per-iteration figure",
}


def algorithmic_bytes_per_tour(w):
    """Sec. 8(d): bytes of choice_info / candidate rows an ant's construction reads.
    cl > 0: (n-1) steps x cl candidates x (4 B inv_w + 2 B id);  cl = 0: sum over steps of
    the unvisited entries of the inv_w row, (n-1) n / 2 x 4 B (+ 2 B per list entry with the
    compact tabu)."""
    if w.selection:
        # roulette wheel (R28): tau + heur (8 B) per considered node (+ 2 B id or list
        # entry); the later stages re-read about 1/31 more -- not counted
        if w.cand_len:
            return (w.n - 1) * w.cand_len * 10
        return (w.n - 1) * w.n // 2 * (10 if w.tabu else 8)
    if w.cand_len:
        return (w.n - 1) * w.cand_len * 6
    if w.tabu:   # compact tabu: + the 2 B list entry of every enumerated node (R27)
        return (w.n - 1) * w.n // 2 * 6
    return (w.n - 1) * w.n // 2 * 4


def workload_config(w, args, world):
    """The `config` object of the JSON line -- the workload only, identical for both arms
    (--impl ours / reference) at the same N; how our arm ran it goes to `run`."""
    m_total = w.n_ants * world if args.scaling == "weak" else w.n_ants
    return {"workload": f"{w.name} ({args.config}): n={w.n}, {w.n_ants} ants"
                        + (" per GPU" if args.scaling == "weak" else " in total")
                        + (f" per colony x {w.colonies} colonies" if w.colonies > 1 else "")
                        + f", cl={w.cand_len}, rho={w.rho}, alpha=1, beta=2",
            "n": w.n, "n_ants": w.n_ants, "global_ants": m_total, "cand_len": w.cand_len, "colonies": w.colonies,
            "pheromone": "lean (R30)" if w.pheromone else "dense n x n",
            "scaling": args.scaling, "tabu": "compact" if w.tabu else "bitmask",
            "selection": "roulette wheel" if w.selection else "WRS",
            "local_search": "2-opt" if w.local_search else "none",
            "l2": "flushed between timed steps (256 MiB write, outside the step events)"}


def cpu_baseline_leg(w, budget_s=12.0):
    """The oracle as it stands on this host's cores, bounded to ~budget_s of CPU work."""
    import oracle
    cores = os.cpu_count() or 1
    col = oracle.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed, nthreads=cores,
                        local_search=bool(w.local_search), tabu=w.tabu, selection=w.selection)
    t0 = time.perf_counter()
    iters = 0
    while True:
        col.iterate(1)
        iters += 1
        el = time.perf_counter() - t0
        if el >= budget_s or iters >= 1000:
            break
    return {"value": w.n_ants * iters / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{iters} full oracle iterations of {w.name} (m={w.n_ants}, cl={w.cand_len}) in {el:.1f} s "
                      f"on {cores} host threads"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = CONFIGS[args.config]
    import oracle
    cores = os.cpu_count() or 1
    world = int(os.environ.get("WORLD_SIZE", "1"))
    m_total = w.n_ants * world if args.scaling == "weak" else w.n_ants
    # the same colony (all N ranks' ants; k independent colonies seeded seed + c, R29) on the host
    cols = [oracle.Colony(w.coords(), m_total, w.cand_len, rho=w.rho, seed=w.mmas_seed + c, nthreads=cores,
                          local_search=bool(w.local_search), tabu=w.tabu, selection=w.selection)
            for c in range(w.colonies)]

    def step():
        for col in cols:
            col.iterate(1)
    for _ in range(args.warmup if args.warmup < 3 else 1):
        step()
    # bounded: each step is one full oracle iteration of every colony; cap the timed steps
    t_probe = time.perf_counter()
    step()
    t_iter = time.perf_counter() - t_probe
    steps = int(max(1, min(args.steps, 90.0 // max(t_iter, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    el = time.perf_counter() - t0
    value = m_total * w.colonies * steps / el
    sample = (f"{steps} of the requested {args.steps} steps (full {m_total}-ant oracle iterations of {w.name}"
              + (f", x {w.colonies} colonies" if w.colonies > 1 else "") + ")")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": el / steps * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(w, args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2003_11902_b200 import mmas

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    # one process per GPU; MMAS_DIST_BACKEND=gloo lets several ranks share one GPU (path tests only)
    backend = os.environ.get("MMAS_DIST_BACKEND", "nccl")
    dev = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    w = CONFIGS[args.config]
    # weak (default): n_ants per GPU; strong: n_ants in total, split over the ranks (R21)
    m_total = w.n_ants * world if args.scaling == "weak" else w.n_ants
    coords = w.coords()
    stream = torch.cuda.current_stream().cuda_stream
    col = mmas.Colony(coords, m_total, w.cand_len, rho=w.rho, seed=w.mmas_seed, device=dev,
                      separate_update=args.separate_update,
                      local_search=bool(w.local_search), tabu=w.tabu, selection=w.selection,
                      stream=stream, rank=rank, world=world, colonies=w.colonies,
                      pheromone=w.pheromone)
    rb = col.record_bytes
    local = torch.zeros(rb, dtype=torch.uint8, device="cuda")
    gathered = torch.zeros(world * rb, dtype=torch.uint8, device="cuda")

    # N > 1: the per-iteration exchange goes through the ranks' device memory (CUDA IPC
    # handles gathered once; P2P stores + device flags, include/mmas.h) unless
    # MMAS_EXCHANGE=collective, or the wiring fails on any rank (then the NCCL all-gather).
    exchange = os.environ.get("MMAS_EXCHANGE", "p2p") if world > 1 else "none"

    def wire_p2p(colony):
        ok = 1
        try:
            mine = colony.exchange_ipc_handle()
            handles = [None] * world
            dist.all_gather_object(handles, mine)
            colony.exchange_open_ipc(handles)
        except Exception as e:   # noqa: BLE001 -- any failure: every rank falls back together
            print(f"rank {rank}: peer exchange unavailable ({e}); using the collective", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        return bool(flag.item())

    if exchange == "p2p" and not wire_p2p(col):
        exchange = "collective"

    def step():
        if world == 1:
            col.iterate(1)
        elif exchange == "p2p":
            col.iterate_exchange(1)   # one launch per iteration where eligible (include/mmas.h)
        else:
            col.construct(local.data_ptr())
            if backend == "nccl":
                dist.all_gather_into_tensor(gathered, local)
            else:   # host staging for the CPU backends
                g_cpu = torch.empty(gathered.shape, dtype=gathered.dtype)
                dist.all_gather_into_tensor(g_cpu, local.cpu())
                gathered.copy_(g_cpu)
            col.update(gathered.data_ptr(), world)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MiB > 126 MB L2
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if exchange == "p2p":
        col.exchange_status()   # raises if a device-side wait timed out during the warm-up

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = col.kernel_launches
    # One launch per step (world 1, construction + selection + update fused, no local search):
    # the step's own event pair brackets exactly that kernel on its stream, so it is the live
    # kernel time; the library's phase events would add two more records per step inside the
    # timed region (measured: 0.2027 -> 0.1970 ms per C2 step without them).  Otherwise the
    # phases are timed by the library (mmas_profile).
    single_launch = world == 1 and bool(col.stats()["update_fused"]) and not w.local_search
    col.profile(not single_launch)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record()
            step()
            ev[k][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gpu_launches = col.kernel_launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(np.sum(step_ms))
    if single_launch:
        phases = {"construct_ms": total_ms, "select_ms": 0.0, "update_ms": 0.0, "local_search_ms": 0.0,
                  "iterations": args.steps}
    else:
        phases = col.phase_times()
    col.profile(False)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    K = w.colonies                                  # concurrent colonies (R29): K tours per ant slot
    tours = m_total * K * args.steps
    mid_iter = args.warmup + args.steps // 2   # the ncu capture nearest the timed window
    value = tours / (total_ms * 1e-3)

    # roofline of the dominant kernel (construction), live CUDA-event time on its stream
    cons_ms = phases["construct_ms"] / max(phases["iterations"], 1)
    bytes_per_launch = algorithmic_bytes_per_tour(w) * col.shard()[1] * K
    cons_kernel = ("construct_rwm_kernel" if w.selection else "construct_cl_kernel" if w.cand_len else
                   "construct_ct_kernel" if w.tabu else "construct_full_kernel")
    # world == 1 with the table in shared memory: the update (row a6) runs inside the same
    # launch (construct.cuh fused_update), so that launch also moves the update's 16 n^2 B
    fused = bool(col.stats()["update_fused"]) and (world == 1 or exchange == "p2p")
    # dense: read tau + heur, write tau + inv_w (16 n^2 B); lean (R30): every stored trail read
    # and written once with its 1 / choice_info (2 x the pheromone state)
    upd_bytes = 2 * col.pheromone_bytes if w.pheromone else 16 * w.n * w.n * K
    if fused:
        bytes_per_launch += upd_bytes
    hbm_peak, peak_src = measured_peaks()
    achieved = bytes_per_launch / (cons_ms * 1e-3) / 1e9
    ent, ent_key = ncu_entry(args.config, cons_kernel, mid_iter)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": ncu_traffic(ent), "ncu_capture": ent_key,
                "traffic_note": "DRAM bytes per launch (ncu capture, profiles/ncu_traffic.json); with the "
                                "candidate table in shared memory (C1, C2: TMA-staged once per launch) or "
                                "L2-resident rows, HBM traffic is far below the algorithmic bytes",
                "kernel": cons_kernel + (" (+ fused pheromone update)" if fused else ""),
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                "kernel_ms": cons_ms, "kernel_share_of_step": cons_ms / (total_ms / args.steps),
                "algorithmic_bytes_per_launch": bytes_per_launch,
                "note": "algorithmic bytes per tour: see algorithmic_bytes_per_tour() and DESIGN.md Sec. 5; the "
                        "construction kernels are issue/latency-bound (ALU + the per-step dependent chain), so "
                        "the issue and chain views below are the ones that bound them (SURVEY 8(d))"}
    # (1b) the on-chip resource the candidate rows actually come from: shared memory (table
    # staged per launch: C1, C2) or L2 (the rest), against the measured read bandwidth
    pk = onchip_peaks() or {}
    if pk:
        smem_table = bool(w.cand_len) and not w.selection and w.n * 32 * 6 <= 200 * 1024
        res = "smem" if smem_table else "l2"
        peak_on = pk["smem_read_gbs" if smem_table else "l2_read_gbs"]
        cand_bytes = algorithmic_bytes_per_tour(w) * col.shard()[1] * K
        ach_on = cand_bytes / (cons_ms * 1e-3) / 1e9
        roofline["onchip"] = {"resource": res, "achieved": ach_on, "peak": peak_on, "unit": "GB/s",
                              "frac": ach_on / peak_on,
                              "peak_source": "measured: profiles/onchip_peaks.json (tools/onchip_peaks.cu)",
                              "note": "the construction's algorithmic candidate/row bytes over the launch time "
                                      "against the measured read bandwidth of the resource they are read from"}
    # (2) issue roofline: warp instructions per launch (ncu capture of the same launch configuration)
    # over the live kernel time, against 4 schedulers x SMs x the SM clock sampled during the run
    sm_mhz = clk.summary().get("sm_mhz") or 0.0
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    if ent and ent.get("l2_bytes") is not None:
        # measured L2 traffic of the same-regime capture over the live kernel time (north_star:
        # "achieved L2 and HBM GB/s"); the read sectors are the candidate / row loads that miss L1
        l2_ach = ent["l2_bytes"] / (cons_ms * 1e-3) / 1e9
        roofline["l2_measured"] = {"bytes_per_launch": ent["l2_bytes"],
                                   "read_sectors": ent.get("l2_sectors_read"),
                                   "achieved": l2_ach, "unit": "GB/s",
                                   "peak": pk.get("l2_read_gbs"),
                                   "frac": l2_ach / pk["l2_read_gbs"] if pk.get("l2_read_gbs") else None,
                                   "capture": ent_key,
                                   "note": "lts__t_bytes.sum of the ncu capture (same config, nearest iteration) / "
                                           "live kernel time, against the measured L2 read bandwidth"}
    if ent and ent.get("inst_executed") and sm_mhz:
        ach = ent["inst_executed"] / (cons_ms * 1e-3) / 1e9
        ipk = 4 * nsm * sm_mhz * 1e6 / 1e9
        roofline["issue"] = {"achieved": ach, "peak": ipk, "unit": "Ginst/s (warp)", "frac": ach / ipk,
                             "inst_per_launch": ent["inst_executed"], "capture": ent_key,
                             "note": "smsp__inst_executed.sum of one captured launch / live kernel time; "
                                     "peak = 4 issue slots x %d SMs x %.0f MHz" % (nsm, sm_mhz)}
    # (3) chain model: every ant's n-1 dependent steps; time per step of one resident warp
    warps_per_sm = col.shard()[1] * K / nsm
    roofline["chain"] = {"ns_per_step": cons_ms * 1e6 / (w.n - 1),
                         "cycles_per_step": cons_ms * 1e-3 * sm_mhz * 1e6 / (w.n - 1) if sm_mhz else None,
                         "ant_warps_per_sm": warps_per_sm,
                         "note": "kernel time / (n-1): the per-step latency of an ant's warp when all ants are "
                                 "resident at once (warps_per_sm <= 64); tools/micro_step.cu measures the "
                                 "chain alone at ~145-160 cycles/step"}
    update_ms = phases["update_ms"] / max(phases["iterations"], 1)
    if fused:
        update_roof = {"kernel": "fused into " + cons_kernel, "fused": True, "algorithmic_bytes_per_launch": upd_bytes,
                       "note": "one launch per iteration: construction, grid barrier (the last block selects the "
                               "iteration best), then every warp updates its rows from tau/heur rows TMA-prefetched "
                               "into shared memory during the construction tail; its bytes are counted in "
                               "roofline.algorithmic_bytes_per_launch"}
    else:
        update_roof = {"kernel": "pheromone_update_kernel", "kernel_ms": update_ms,
                       "traffic": ncu_traffic(ncu_entry(args.config, "pheromone_update_kernel", mid_iter)[0]),
                       "achieved_gbs": upd_bytes / (update_ms * 1e-3) / 1e9,
                       "frac": upd_bytes / (update_ms * 1e-3) / 1e9 / hbm_peak,
                       "algorithmic_bytes_per_launch": upd_bytes}

    # e2e through the C ABI with host buffers: create from host coords (H2D), then per step
    # iterate + read the global best back to the host (D2H), all inside the timed region.
    # e2e through the C ABI with host buffers, at N GPUs: every rank creates its shard from
    # pinned host coords (H2D), then per step construct + exchange + update (iterate at N = 1)
    # and reads the global best length back to the host (D2H); max over ranks.
    e2e = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    pinned = torch.from_numpy(coords.copy()).pin_memory().numpy()
    out_steps = args.steps
    best_host = torch.full((out_steps,), -1, dtype=torch.int64).pin_memory()   # per-step results

    def e2e_colony():
        c = mmas.Colony(pinned, m_total, w.cand_len, rho=w.rho, seed=w.mmas_seed, device=dev,
                        separate_update=args.separate_update,
                        local_search=bool(w.local_search), tabu=w.tabu, selection=w.selection,
                        stream=stream, rank=rank, world=world, colonies=w.colonies,
                      pheromone=w.pheromone)
        if exchange == "p2p":
            wire_p2p(c)
        return c

    # untimed warm-up of the same path (create, a few iterations, read-back, destroy)
    cw = e2e_colony()
    for _ in range(min(3, args.warmup)):
        cw.iterate(1) if world == 1 else (cw.iterate_exchange(1) if exchange == "p2p" else None)
    cw.sync()
    cw.close()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c2 = e2e_colony()
    t_created = time.perf_counter()
    for k in range(out_steps):
        if world == 1:
            c2.iterate(1)
        elif exchange == "p2p":
            c2.iterate_exchange(1)
        else:
            c2.construct(local.data_ptr())
            if backend == "nccl":
                dist.all_gather_into_tensor(gathered, local)
            else:
                g_cpu = torch.empty(gathered.shape, dtype=gathered.dtype)
                dist.all_gather_into_tensor(g_cpu, local.cpu())
                gathered.copy_(g_cpu)
            c2.update(gathered.data_ptr(), world)
        # the step's result (global best length, 8 B) copied to pinned host memory on the
        # stream: no per-step host round trip; the host reads them after the final sync
        c2.best_length_async(best_host.data_ptr() + 8 * k)
    t_enqueued = time.perf_counter()
    _, final_len = c2.best_tour()
    el = time.perf_counter() - t0
    c2.close()
    bh = best_host.numpy()
    assert bh[-1] == final_len and np.all(bh > 0) and np.all(np.diff(bh) <= 0), "e2e per-step results"
    if world > 1:
        te = torch.tensor([el], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te.item())
    e2e = {"value": m_total * K * out_steps / el, "unit": UNIT,
           "h2d_bytes_per_step": 16 * w.n / out_steps, "d2h_bytes_per_step": 8 + 2 * w.n / out_steps,
           "seconds": {"total": el, "create": t_created - t0, "steps_enqueued": t_enqueued - t_created},
           "note": "timed on every rank, max over ranks: mmas_create from pinned host coords (H2D), per "
                   "step mmas_iterate(1) (N = 1) or mmas_construct + all-gather + mmas_update (N > 1) + "
                   "mmas_best_length_async (8-byte D2H of the step's global best into pinned host memory, "
                   "no per-step sync), final mmas_best_tour (sync + D2H of the route); the per-step "
                   "lengths are checked (non-increasing, last = final); a plain back-to-back loop with no L2 "
                   "flush between steps (value flushes 256 MiB before every step), so e2e can exceed value"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(w)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": workload_config(w, args, world),
                "run": {"parallelism": f"ant-sharded x{world}" if world > 1 else "single GPU",
                        "exchange": {"p2p": "peer memory: CUDA IPC buffers, P2P record stores + device flags",
                                     "collective": f"{backend} all-gather of the records",
                                     "none": "none (one GPU)"}[exchange],
                        "timed_iterations": [args.warmup, args.warmup + args.steps - 1],
                        "pheromone_bytes": col.pheromone_bytes,
                        "iteration_launches": "one (construction + selection + update fused)" if fused else
                                              "construction (+ selection) then update",
                        "paper_context": PAPER_CONTEXT.get(args.config, "") + " (other hardware, context only)"},
                "roofline": roofline, "update_roofline": update_roof,
                "phases_ms_per_step": {"construct": cons_ms, "select": phases["select_ms"] / max(phases["iterations"], 1),
                                       "update": update_ms,
                                       "local_search": phases["local_search_ms"] / max(phases["iterations"], 1)},
                "construction_only_tours_per_s": w.n_ants * K / (cons_ms * 1e-3),
                "gpu_launches": gpu_launches, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
                "fallback_steps_per_tour": col.stats()["fallback_steps"] / max(col.stats()["iterations"], 1) / col.shard()[1] / K,
                "local_search_moves_per_tour": col.stats()["local_search_moves"] / max(col.stats()["iterations"], 1) / col.shard()[1]}
        print(json.dumps(line), flush=True)
    col.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: n_ants per GPU (default); strong: n_ants in total, split over the GPUs")
    ap.add_argument("--separate-update", action="store_true",
                    help="run the pheromone update as its own kernel (A/B against the fused launch)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
