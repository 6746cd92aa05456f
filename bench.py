#!/usr/bin/env python
"""bench.py -- agent mechanical updates/s of the B200-native BioDynaMo mechanical step.

One bench "step" is one full pass of the hot path (grid rebuild, 27-box search, force,
displacement, position update) over the whole population.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl bdm|reference]

Default workload: BASELINE.json configs[2] (cfg3, 2e7 agents, Gaussian spheroid) -- the config
BASELINE.json's metric ("at 1/2/4/8 B200") is quoted on; it fits one GPU.  Rank 0 prints ONE
JSON line.  --impl reference times the CPU oracle (oracle/, the base contract's reference arm)
on a bounded sample of the same workload.
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

import bdm_inputs  # noqa: E402

METRIC = "agent mechanical updates/sec at 1/2/4/8 B200; achieved HBM GB/s vs peak"
UNIT = "agent-updates/s"
WORKLOADS = {
    1: "cfg1 (BASELINE configs[0]): 4096 agents U[0,160)^3 um, D~U[8,12)",
    2: "cfg2 (BASELINE configs[1]): 1e6 agents, 100^3 lattice 10 um, jitter U[-2,2), D~U[9,11)",
    3: "cfg3 (BASELINE configs[2]): 2e7 agents, Gaussian spheroid sigma=992.2 um, D=lognormal(10,0.15) clipped [6,16]",
    4: "cfg4 (BASELINE configs[3]): 2e8 agents uniform 8:1:1 slab at 1e-3 um^-3, D~U[8,12)",
    5: "cfg5 (BASELINE configs[4]): 1e9 agents uniform 1e4^3 um, D~U[8,12)",
}

# fp64-pipe instruction costs per unit of work (counted from the SASS of k_force)
FP64_PER_CANDIDATE = 9
FP64_PER_CONTACT = 44
FP64_PER_AGENT = 40


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_inputs(cfg: int, n: int | None):
    return bdm_inputs.make_config(cfg, n)


# ------------------------------------------------------------------------------------ oracle arm
def host_cores() -> int:
    """The host cores this process may run on (torchrun sets OMP_NUM_THREADS=1 for its workers, so the
    oracle's "all cores" runs pass this count explicitly instead of relying on the OpenMP default)."""
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def oracle_sample_run(pos, diam, stride: int, nthreads: int = 0):
    """The CPU oracle as it stands on a bounded sample: the whole population is the environment
    (the oracle rebuilds its grid over all N agents) and every stride-th agent id is updated.
    nthreads 0: all host cores."""
    import oracle

    threads = nthreads or host_cores()
    sample = np.arange(0, len(diam), stride, dtype=np.int64)
    t0 = time.perf_counter()
    oracle.step(pos, diam, sample=sample, record=False, nthreads=threads)
    dt = time.perf_counter() - t0
    return len(sample), dt, threads


def host_info():
    """nproc, CPU model and RAM of the host the oracle runs on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    ram = round(int(ln.split()[1]) / 2 ** 20, 1)
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "ram_gib": ram}


def cpu_baseline(pos, diam, what, stride_1t):
    """The CPU oracle as it stands: ONE full step of the whole population (every
    agent updated, grid rebuilt) with OpenMP on all host cores, and a single-threaded run on a
    bounded sample (every stride-th agent updated; the grid over all agents is still built, so that
    figure includes the whole index build)."""
    import oracle

    threads = host_cores()
    t0 = time.perf_counter()
    oracle.step(pos, diam, record=False, nthreads=threads)
    t_all = time.perf_counter() - t0
    m, t_1, _ = oracle_sample_run(pos, diam, stride_1t, nthreads=1)
    n = len(diam)
    return {"value": n / t_all, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"one full oracle step of {what} (all {n} agents updated, grid rebuilt), OpenMP on "
                      f"{threads} threads, {t_all:.1f} s wall",
            "single_thread": {"value": m / t_1, "unit": UNIT, "cores": 1,
                              "sample": f"every {stride_1t}th agent id updated ({m} agents) with {what} as "
                                        f"environment, 1 thread; includes the oracle's full grid build; "
                                        f"{t_1:.1f} s wall"},
            **host_info()}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    pos, diam = make_inputs(args.config, args.n)
    n = len(diam)
    stride = args.cpu_stride
    for _ in range(args.warmup):
        oracle_sample_run(pos, diam, stride)
    tot_agents, tot_t, threads = 0, 0.0, 1
    for _ in range(args.steps):
        m, dt, threads = oracle_sample_run(pos, diam, stride)
        tot_agents += m
        tot_t += dt
    value = tot_agents / tot_t
    sample = (f"every {stride}th agent id of the {n}-agent workload updated per step (the oracle rebuilds its "
              f"grid over all {n} agents each step); value = sampled agent-updates / oracle wall time")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_obj(args, n, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                             **host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_obj(args, n, world):
    return {"workload": WORKLOADS[args.config], "n_agents": n, "config_index": args.config,
            "parallelism": f"x-slabs x{world}" if world > 1 else "1 GPU",
            "l2": "inputs larger than L2 (32 B/agent state)" if n * 32 > 126e6 else "L2 flushed between steps",
            "params": "k=10 gamma=4 adherence=0.1 dt=1 eta=1 max_disp=3 (DESIGN.md R1-R5)"}


# ------------------------------------------------------------------------------------ GPU arm
def run_bdm(args):
    import torch

    import paper_2006_06775_b200 as bdm

    world, rank, local = dist_env()
    if world > 1 or args.slabs:
        return run_dist(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    n = config_size(args.config, args.n)
    big = n > BIG_N
    pos_d, diam_d, pos_h, diam_h = device_inputs(bdm, torch, args.config, n, dev, stream)

    # work units of one step (algorithmic fp64 ops), from one recorded step at the start state; for
    # the 1e8-1e9-agent configs on a 2e7-agent sub-volume of the same density (per-agent averages)
    prm = bdm.bdm_params_default(device=local)
    prm.flags |= bdm.BDM_RECORD
    if big:
        sp, sd, _, _ = device_inputs(bdm, torch, args.config, SUB_N, dev, stream, scale_from=n)
        hr = bdm.bdm_init(sp, sd, prm, stream=stream)
        del sp, sd
    else:
        hr = bdm.bdm_init(pos_d, diam_d, prm, stream=stream)
    bdm.bdm_mech_step(hr, 1)
    st = bdm.bdm_get_agent_stats(hr)
    scale = n / (SUB_N if big else n)
    n_cand = int(st["n_cand"].sum().item() * scale)
    n_ct = int(st["n_ct"].sum().item() * scale)
    hr.close()
    del st
    torch.cuda.empty_cache()
    h = bdm.bdm_init(pos_d, diam_d, bdm.bdm_params_default(device=local), stream=stream)
    del pos_d, diam_d  # the handle holds its own copy (frees 32 B/agent for the 1e9-agent config)
    torch.cuda.empty_cache()
    bdm.bdm_set_timing(h, True)
    flush = None
    if n * 32 <= 126e6:  # state fits in L2: flush it between timed steps
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:  # sampled from warm-up through the timed region
        time.sleep(0.3)
        for _ in range(args.warmup):
            bdm.bdm_mech_step(h, 1)
        bdm.bdm_sync(h)
        bdm.bdm_get_timing(h)  # reset sums
        torch.cuda.synchronize()
        prof = os.environ.get("BDM_PROFILE_TIMED") == "1"  # ncu --profile-from-start off: the timed steps only
        if prof:
            torch.cuda.profiler.start()
        if flush is None:  # state larger than L2: time the K steps as one bdm_mech_step(K) call
            evs[0][0].record(stream)
            bdm.bdm_mech_step(h, args.steps)
            evs[0][1].record(stream)
            evs = evs[:1]
        else:  # state fits in L2: flush it between steps, time each step
            for k in range(args.steps):
                flush.add_(1)
                evs[k][0].record(stream)
                bdm.bdm_mech_step(h, 1)
                evs[k][1].record(stream)
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
    bdm.bdm_sync(h)
    path_kind = bdm.bdm_get_path_stats(h)["half"]  # 1 half-shell passes, 2 the same band by band (ring), 0 k_force
    half_path = path_kind in (1, 2)  # (packed new boxes exist only on the half-shell path, ring or not)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tm = bdm.bdm_get_timing(h)
    total_s = sum(step_ms) / 1e3
    value = n * args.steps / total_s

    peaks, peak_kind = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp64_peak = 148 * 64 * sm_max * 1e6  # fp64 lanes x clock
    force_s = tm["force_ms"] / 1e3 / max(tm["steps"], 1)
    ops = FP64_PER_CANDIDATE * n_cand + FP64_PER_CONTACT * n_ct + FP64_PER_AGENT * n
    achieved = ops / force_s
    grid_s = tm["grid_ms"] / 1e3 / max(tm["steps"], 1)
    rebuild_bpa = REBUILD_BYTES_PER_AGENT if half_path else 160
    rebuild_bytes = rebuild_bpa * n
    rebuild = {"bound": "hbm", "achieved": rebuild_bytes / grid_s / 1e9, "peak": float(peaks["hbm_gbs"]),
               "unit": "GB/s", "frac": rebuild_bytes / grid_s / 1e9 / float(peaks["hbm_gbs"]),
               "ms_per_step": grid_s * 1e3, "bytes_per_agent": rebuild_bpa}
    traffic = None
    tf = os.path.join(ROOT, "profiles", "r02_force_traffic.json")
    if args.config == 3 and os.path.exists(tf):  # measured DRAM bytes of the force kernel (committed capture)
        with open(tf) as f:
            t = json.load(f)
        traffic = t["dram_bytes_read"] + t["dram_bytes_write"]

    h.close()
    torch.cuda.empty_cache()
    # end-to-end through the C ABI with host buffers (pinned), copies inside the timed region
    if pos_h is None:  # device-generated config: bring the inputs to (pinned) host memory once
        pd, dd, _, _ = device_inputs(bdm, torch, args.config, n, dev, stream)
        pos_h, diam_h = pd.cpu().numpy(), dd.cpu().numpy()
        del pd, dd
        torch.cuda.empty_cache()
    e2e = run_e2e(bdm, torch, pos_h, diam_h, local, args)

    cpu = None
    if not args.no_cpu_baseline:
        if big:  # the oracle on a 2e7-agent sub-volume of the same density
            ps, ds = sub_volume(args.config, n)
            what = f"a {SUB_N}-agent sub-volume of the workload at the same density"
        else:
            ps, ds = pos_h, diam_h
            what = f"the whole {n}-agent workload"
        cpu = cpu_baseline(ps, ds, what, args.cpu_stride_1t)

    step_hbm = None
    tr = os.path.join(ROOT, "profiles", "r02_rebuild_traffic.json")
    if traffic and os.path.exists(tr):  # the whole step's measured DRAM bytes (ncu) over its event time
        with open(tr) as f:
            t = json.load(f)
        sb = traffic + t["dram_bytes_read"] + t["dram_bytes_write"]
        ach = sb / (total_s / args.steps) / 1e9
        step_hbm = {"bytes_per_step": sb, "achieved_gbs": ach, "peak_gbs": float(peaks["hbm_gbs"]),
                    "frac": ach / float(peaks["hbm_gbs"]),
                    "source": "ncu DRAM bytes of the force phase (profiles/r02_force_traffic.json) + rebuild "
                              "(profiles/r02_rebuild_traffic.json), cfg3 steady state, over the timed ms/step"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_obj(args, n, 1),
            "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": fp64_peak / 1e12, "unit": "TFLOP/s",
                         "frac": achieved / fp64_peak, "traffic": traffic,
                         "kernel": {1: "force phase: k_half_search + k_half_sum",
                                    2: "force phase: k_half_search + k_half_sum, band by band over a ring of pair rows"
                                    }.get(path_kind, "k_force"),
                         "traffic_source": "profiles/r02_force_traffic.json" if traffic else None,
                         "ms_per_launch": force_s * 1e3,
                         "passes_ms": {"search": tm["search_ms"] / max(tm["steps"], 1),
                                       "sum": tm["sum_ms"] / max(tm["steps"], 1)},
                         "note": "the method's fp64-pipe ops (9 per 27-box candidate + 44 per contact + 40 per "
                                 "agent, DESIGN.md §6.2) over the force phase's event time (both passes); peak = "
                                 f"148 SM x 64 fp64 lanes x {sm_max:.0f} MHz ({peak_kind} sm_max_mhz)",
                         "units": {"candidates": n_cand, "contacts": n_ct, "agents": n}},
            "roofline_rebuild": rebuild, "step_hbm": step_hbm,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": tm["launches"],
            "clocks": clk.summary(), "step_ms": [round(x, 4) for x in step_ms]}
    print(json.dumps(line), flush=True)
    return 0


def run_dist(args):
    """N ranks (one per GPU) of libbdm's distributed runtime (bdm_init_dist): every rank
    generates its id share, the library redistributes the agents by x-slab (work-balanced cuts) and
    steps them with NCCL halo exchange + migration.  Timed: K steps after W warm-up steps, barrier +
    synchronize on both sides, CUDA events on each rank's stream, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2006_06775_b200 as bdm
    from paper_2006_06775_b200 import dist as bdist

    world, rank, local = dist_env()
    os.environ.setdefault("NCCL_DEBUG", "INFO")  # (init logging: the rank count of each communicator)
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        if world > 1:
            dist.init_process_group("nccl", device_id=dev)
        elif "MASTER_ADDR" in os.environ and "WORLD_SIZE" in os.environ:  # (1 rank under torchrun: its store)
            dist.init_process_group("gloo")
        else:  # (--slabs at N = 1: a 1-rank group for the barriers)
            dist.init_process_group("gloo", rank=0, world_size=1, init_method="tcp://127.0.0.1:%d" % free_port())
    stream = torch.cuda.Stream(device=dev)
    n = config_size(args.config, args.n)
    big = n > BIG_N
    # algorithmic work units per agent (candidates, contacts) from one recorded single-GPU step on
    # rank 0: the whole population when it fits, else a 2e7-agent sub-volume of the same density
    units = torch.zeros(2, dtype=torch.float64, device=dev)
    if rank == 0:
        prm = bdm.bdm_params_default(device=local)
        prm.flags |= bdm.BDM_RECORD
        m = SUB_N if big else n
        sp, sd, _, _ = device_inputs(bdm, torch, args.config, m, dev, torch.cuda.current_stream(),
                                     scale_from=n if big else None)
        hr = bdm.bdm_init(sp, sd, prm)
        bdm.bdm_mech_step(hr, 1)
        st = bdm.bdm_get_agent_stats(hr)
        units[0] = float(st["n_cand"].sum().item()) / m
        units[1] = float(st["n_ct"].sum().item()) / m
        hr.close()
        del st, sp, sd
        torch.cuda.empty_cache()
    dist.broadcast(units, 0) if world > 1 else None
    uid = bdist.broadcast_uid(dist, bdm, dev) if world > 1 else bdm.bdm_nccl_unique_id()
    if args.slab_of > 1:  # one rank's x-slab of the config at slab_of ranks, alone on this GPU (memory / rate)
        ids, pos, diam = slab_share(bdm, torch, args.config, n, args.slab_of, dev, stream)
        n = int(ids.shape[0])
    else:
        ids, pos, diam = bdist.rank_inputs(bdm, torch, bdm_inputs, args.config, n, rank, world, dev, stream)
    t0 = time.perf_counter()
    h = bdm.bdm_init_dist(ids, pos, diam, bdm.bdm_params_default(), rank=rank, world=world, uid=uid, device=local,
                          stream=stream)
    setup_s = time.perf_counter() - t0
    del ids, pos, diam
    torch.cuda.empty_cache()
    bdm.bdm_set_timing(h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        bdm.bdm_mech_step(h, args.warmup)
        bdm.bdm_sync(h)
        bdm.bdm_get_timing(h)  # reset the sums
        s0 = bdm.bdm_get_stats(h)
        dist.barrier()
        torch.cuda.synchronize(dev)
        prof = os.environ.get("BDM_PROFILE_TIMED") == "1"
        if prof:
            torch.cuda.profiler.start()
        e0.record(stream)
        bdm.bdm_mech_step(h, args.steps)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if prof:
            torch.cuda.profiler.stop()
        dist.barrier()
    tm = bdm.bdm_get_timing(h)
    s1 = bdm.bdm_get_stats(h)
    free_b, total_b = torch.cuda.mem_get_info(dev)
    import resource

    mem = {"gpu_used_gib": round((total_b - free_b) / 2 ** 30, 2), "gpu_total_gib": round(total_b / 2 ** 30, 2),
           "host_maxrss_gib": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20, 2),
           "note": "rank 0 after the timed steps: device memory in use (libbdm's buffers + torch's cache), host peak RSS"}
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = n * args.steps / (ms / 1e3)
    agg = torch.tensor([s1["launches"] - s0["launches"], s1["host_syncs"] - s0["host_syncs"],
                        s1["exchange_bytes"] - s0["exchange_bytes"], s1["migrated"] - s0["migrated"]],
                       dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(agg, op=dist.ReduceOp.SUM)
    own = s1["n_agents"]
    cuts = bdm.bdm_get_cuts(h)
    # end to end through the public API with HOST buffers: per batch every rank uploads its id share
    # from pinned memory (bdm_init_dist: validation, cuts, redistribution), runs one step and reads its
    # owned agents' displacements back (bdm_get_local into pinned memory)
    h.close()
    torch.cuda.empty_cache()
    ids_d, pos_d, diam_d = bdist.rank_inputs(bdm, torch, bdm_inputs, args.config, n, rank, world, dev, stream)
    pin_ids = ids_d.cpu().pin_memory()
    pin_pos = pos_d.cpu().pin_memory()
    pin_diam = diam_d.cpu().pin_memory()
    del ids_d, pos_d, diam_d
    torch.cuda.empty_cache()
    e2e_s, h2d, d2h = 0.0, 0, 0
    uid = bdist.broadcast_uid(dist, bdm, dev) if world > 1 else bdm.bdm_nccl_unique_id()
    he = bdm.bdm_init_dist(pin_ids.numpy(), pin_pos.numpy(), pin_diam.numpy(), bdm.bdm_params_default(), rank=rank,
                           world=world, uid=uid, device=local, stream=stream)
    for rep in range(args.e2e_steps + 1):
        dist.barrier()
        torch.cuda.synchronize(dev)
        w0 = time.perf_counter()
        if rep > 0:
            bdm.bdm_set_agents_dist(he, pin_ids.numpy(), pin_pos.numpy(), pin_diam.numpy())
        bdm.bdm_mech_step(he, 1)
        ids_o, dp_o = bdm.bdm_get_local(he, bdm.BDM_LAST_DISPLACEMENTS)
        wall = time.perf_counter() - w0
        if rep > 0:  # (the first batch, loaded by bdm_init_dist, is a warm-up)
            e2e_s += wall
            h2d += pin_ids.numel() * 8 + pin_pos.numel() * 8 + pin_diam.numel() * 8
            d2h += ids_o.size * 8 + dp_o.size * 8
    he.close()
    et = torch.tensor([e2e_s, h2d, d2h], dtype=torch.float64, device=dev)
    mx = et.clone()
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(et, op=dist.ReduceOp.SUM)
    steps_e2e = max(args.e2e_steps, 1)
    e2e = {"value": n * steps_e2e / float(mx[0].item()), "unit": UNIT,
           "h2d_bytes_per_step": int(et[1].item() / steps_e2e), "d2h_bytes_per_step": int(et[2].item() / steps_e2e),
           "steps": steps_e2e,
           "path": "per rank: host id share (pinned) -> bdm_set_agents_dist (validation, cuts, redistribution) "
                   "-> bdm_mech_step(1) -> bdm_get_local(displacements, host); wall clock, max over ranks"}
    if rank == 0:
        peaks, peak_kind = load_peaks()
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        fp64_peak = 148 * 64 * sm_max * 1e6
        ops = (FP64_PER_CANDIDATE * units[0].item() + FP64_PER_CONTACT * units[1].item() + FP64_PER_AGENT) * own
        steps_t = max(tm["steps"], 1)
        force_s = tm["force_ms"] / 1e3 / steps_t
        achieved = ops / force_s if force_s > 0 else 0.0
        traffic = None
        tf = os.path.join(ROOT, "profiles", "r02_force_traffic.json")
        if not os.path.exists(tf):
            tf = os.path.join(ROOT, "profiles", "r02_force_traffic.json")
        if args.config == 3 and os.path.exists(tf):
            with open(tf) as f:
                tr = json.load(f)
            traffic = int((tr["dram_bytes_read"] + tr["dram_bytes_write"]) * own / tr.get("n_agents", 20_000_000))
        cpu = None
        if not args.no_cpu_baseline:
            if big:
                ps, ds = sub_volume(args.config, n)
                what = f"a {SUB_N}-agent sub-volume of the workload at the same density"
            else:
                ps, ds = bdm_inputs.make_config(args.config, n if n != bdm_inputs.CFG_N[args.config] else None)
                what = f"the whole {n}-agent workload"
            cpu = cpu_baseline(ps, ds, what, args.cpu_stride_1t)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(config_obj(args, n, world), cuts=[int(c) for c in cuts[1:-1]],
                               **({"slab_of": args.slab_of, "note": f"rank 0's x-slab of the {args.config} population at "
                                   f"{args.slab_of} ranks, alone on one GPU (no neighbours: no exchange traffic)"}
                                  if args.slab_of > 1 else {})),
                "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": fp64_peak / 1e12, "unit": "TFLOP/s",
                             "frac": achieved / fp64_peak, "traffic": traffic,
                             "traffic_source": (os.path.relpath(tf, ROOT) + " scaled to rank 0's owned agents")
                             if traffic else None,
                             "kernel": "rank 0 force phase: k_half_search + k_half_sum",
                             "ms_per_launch": force_s * 1e3,
                             "passes_ms": {"search": tm["search_ms"] / steps_t, "sum": tm["sum_ms"] / steps_t},
                             "note": "rank 0's owned agents x the per-agent fp64-pipe ops of the recorded step "
                                     "(9 per candidate + 44 per contact + 40 per agent, DESIGN.md §6.2) over its "
                                     "force-phase event time; peak = 148 SM x 64 fp64 lanes x sm_max_mhz"},
                "mem": mem,
                "dist": {"host_syncs": int(agg[1].item()), "launches": int(agg[0].item()),
                         "exchange_bytes": int(agg[2].item()), "migrated": int(agg[3].item()),
                         "setup_s": setup_s, "rank0_agents": own,
                         "note": "libbdm distributed runtime: NCCL send/recv of fixed-capacity messages, "
                                 "device-resident counts, one host round trip per chunk of <= 16 steps"},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(agg[0].item()),
                "clocks": clk.summary(), "timing": "CUDA events on each rank's stream, max over ranks"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    dist.destroy_process_group()
    return 0


def slab_share(bdm, torch, cfg, n_full, slabs, dev, stream):
    """The first of `slabs` equal x-slabs of a uniform counter-hash config (4, 5), generated on the device
    in id chunks (kernel K0) and filtered: what rank 0 of `slabs` ranks owns."""
    assert cfg in (4, 5), "--slab-of needs a uniform counter-hash config (4 or 5)"
    lo, hi = bdm_inputs.box_of(cfg, n_full)
    xcut = lo[0] + (hi[0] - lo[0]) / slabs
    keep_i, keep_p, keep_d = [], [], []
    step = 50_000_000
    for a in range(0, n_full, step):
        m = min(step, n_full - a)
        p = torch.empty((m, 3), dtype=torch.float64, device=dev)
        d = torch.empty(m, dtype=torch.float64, device=dev)
        bdm.bdm_generate_uniform(cfg, a, m, lo, hi, 8.0, 12.0, p, d, stream)
        torch.cuda.synchronize(dev)
        sel = p[:, 0] < xcut
        keep_i.append(torch.nonzero(sel).squeeze(1) + a)
        keep_p.append(p[sel])
        keep_d.append(d[sel])
        del p, d, sel
    return torch.cat(keep_i).to(torch.int64), torch.cat(keep_p).contiguous(), torch.cat(keep_d).contiguous()


def free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


BIG_N = 50_000_000  # above this: device generation, statistics and CPU baseline on a sub-volume
SUB_N = 20_000_000


def config_size(cfg, n):
    if n is not None:
        return n
    return bdm_inputs.CFG_N[cfg]


def sub_volume(cfg, n_full):
    """Host population: the first SUB_N ids of a counter-hash config in a box shrunk so that the
    density is unchanged (cfg4 / cfg5 are uniform)."""
    lo, hi = bdm_inputs.box_of(cfg, n_full)
    f = (SUB_N / n_full) ** (1.0 / 3.0)
    hi = tuple(lo[a] + (hi[a] - lo[a]) * f for a in range(3))
    return bdm_inputs.uniform_population(cfg, np.arange(SUB_N), lo, hi, 8.0, 12.0)


def device_inputs(bdm, torch, cfg, n, dev, stream, scale_from=None):
    """(pos_d, diam_d, pos_h, diam_h): counter-hash configs (1, 4, 5) are generated on the device by
    bdm_generate_uniform (kernel K0, bit-identical to bdm_inputs); cfg2 / cfg3 on the host."""
    if cfg in (1, 4, 5):
        nfull = scale_from or n
        lo, hi = bdm_inputs.box_of(cfg, nfull) if cfg != 1 else bdm_inputs.box_of(1)
        if scale_from:
            f = (n / scale_from) ** (1.0 / 3.0)
            hi = tuple(lo[a] + (hi[a] - lo[a]) * f for a in range(3))
        pos = torch.empty((n, 3), dtype=torch.float64, device=dev)
        diam = torch.empty(n, dtype=torch.float64, device=dev)
        bdm.bdm_generate_uniform(cfg, 0, n, lo, hi, 8.0, 12.0, pos, diam, stream)
        torch.cuda.synchronize()
        return pos, diam, None, None
    pos_h, diam_h = make_inputs(cfg, n if n != bdm_inputs.CFG_N[cfg] else None)
    return torch.from_numpy(pos_h).to(dev), torch.from_numpy(diam_h).to(dev), pos_h, diam_h


# rebuild kernels, algorithmic bytes per agent: column pass 32 | key + histogram
# 32 + 8 | scatter 12 + 12 | place 12 + 32 gather + 32 + 4 + 16 (fp32 copy) = 192 B/agent (the
# ragged box table adds ~12 B per box, not counted)
# key+hist 12 (packed new box written by the last sum pass) or 40 (BDM_PBOX=0: the state), scatter 24,
# place 96 (column pass fused into the sum pass)
REBUILD_BYTES_PER_AGENT = 132 if os.environ.get("BDM_PBOX", "1") != "0" else 160


def run_e2e(bdm, torch, pos_h, diam_h, local, args):
    """Same metric through the public C ABI with HOST buffers: every batch pays its pinned H2D
    (bdm_set_agents), one step and the D2H of its displacements (bdm_get_displacements).  Three
    handles on three streams (BDM_E2E_LANES), each driven by its own host thread (ctypes releases the
    GIL), take batches round-robin, so one batch's upload overlaps the others' steps and downloads
    (H2D and D2H use separate copy engines) -- a serving pipeline; the timed region is the wall time
    of all batches."""
    import threading

    n = len(diam_h)
    pin_pos = torch.from_numpy(pos_h).pin_memory()
    pin_diam = torch.from_numpy(diam_h).pin_memory()
    ppos, pdiam = pin_pos.numpy(), pin_diam.numpy()
    lanes = []
    lanes_n = int(os.environ.get("BDM_E2E_LANES", "3"))
    free, _ = torch.cuda.mem_get_info(local)
    lanes_n = max(1, min(lanes_n, int(free // (n * 200))))  # each lane is a handle of ~135-160 B/agent
    for _ in range(lanes_n):
        out = torch.empty((n, 3), dtype=torch.float64).pin_memory()
        st = torch.cuda.Stream(device=local)
        h = bdm.bdm_init(ppos, pdiam, bdm.bdm_params_default(device=local))
        bdm.bdm_set_stream(h, st)
        lanes.append((h, out.numpy(), out))

    def one(h, pout):
        bdm.bdm_set_agents(h, ppos, pdiam)  # H2D of this batch's inputs
        bdm.bdm_mech_step(h, 1)
        bdm.bdm_get_displacements(h, pout)  # D2H of the batch's result (synchronises its stream)

    for h, pout, _ in lanes:
        one(h, pout)
    torch.cuda.synchronize()
    batches = max(lanes_n, lanes_n * args.e2e_steps)

    def worker(k):
        h, pout, _ = lanes[k]
        for _ in range(k, batches, lanes_n):
            one(h, pout)

    w0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(k,)) for k in range(lanes_n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    for h, _, _ in lanes:
        h.close()
    # the link's own bound for this traffic: plain pinned copies of the same sizes, both directions
    # at once (separate copy engines), timed the same way
    copy_bound = None
    try:
        dev_in = torch.empty(pos_h.nbytes + diam_h.nbytes, dtype=torch.uint8, device=local)
        dev_out = torch.empty(n * 3 * 8, dtype=torch.uint8, device=local)
        host_in = torch.empty(dev_in.numel(), dtype=torch.uint8).pin_memory()
        host_out = lanes[0][2].view(torch.uint8).view(-1)
        s_in, s_out = torch.cuda.Stream(device=local), torch.cuda.Stream(device=local)
        reps = 4
        torch.cuda.synchronize()
        c0 = time.perf_counter()
        for _ in range(reps):
            with torch.cuda.stream(s_in):
                dev_in.copy_(host_in, non_blocking=True)
            with torch.cuda.stream(s_out):
                host_out.copy_(dev_out, non_blocking=True)
        torch.cuda.synchronize()
        link = (time.perf_counter() - c0) / reps
        copy_bound = {"value": n / link, "unit": UNIT,
                      "note": "pinned H2D of the inputs and D2H of the result alone (concurrent, no step): "
                              "the PCIe ceiling of this e2e path"}
        del dev_in, dev_out, host_in
    except RuntimeError:  # (no room for the extra buffers at the largest configs)
        pass
    return {"value": n * batches / wall, "unit": UNIT, "h2d_bytes_per_step": int(pos_h.nbytes + diam_h.nbytes),
            "d2h_bytes_per_step": int(n * 3 * 8), "steps": batches, "wall_s": wall,
            "copy_bound": copy_bound,
            "path": f"{lanes_n} host threads x (bdm_set_agents(host pinned) -> bdm_mech_step(1) -> "
                    "bdm_get_displacements(host pinned)) on as many streams, batches round-robin; wall clock"}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--n", type=int, default=None, help="override N (testing only)")
    ap.add_argument("--impl", default="bdm", choices=["bdm", "reference"])
    ap.add_argument("--cpu-stride", type=int, default=10, help="reference arm: every k-th agent updated per step")
    ap.add_argument("--cpu-stride-1t", type=int, default=200, help="single-threaded oracle sample stride")
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slabs", action="store_true", help="use the distributed runtime even at one rank")
    ap.add_argument("--slab-of", type=int, default=1,
                    help="with --slabs at one rank: run only rank 0's x-slab of a uniform config at this many ranks")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "bdm":
        print("note: timing rules need >= 3 warm-up steps; raising warmup to 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    world, _, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:  # not under torchrun: launch the N ranks ourselves
        from paper_2006_06775_b200 import dist as bdist

        return bdist.relaunch(os.path.abspath(__file__), sys.argv[1:], args.gpus)
    return run_bdm(args)


if __name__ == "__main__":
    sys.exit(main())
