#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (run here, on the CPU box, from gpurun_out/ captures).

  python tools/ncu_summary.py launches <launches.csv>        per-kernel share of the launch list
  python tools/ncu_summary.py kernel <prof.ncu-rep>          key metrics + stall reasons + hot SASS
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        agg[r[ki].split("(")[0].replace("void ", "")[:70]].append(float(r[vi].replace(",", "")) * UNIT[r[ui]])
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':70s} {'n':>4s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:70s} {len(v):4d} {sum(v):10.3f} {sum(v) / len(v):9.4f} {sum(v) / tot:6.3f}")
    print(f"total {tot:.3f} ms over {sum(len(v) for v in agg.values())} launches (cold-cache, serialised)")


def kernel(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    for row in r[2:]:
        d = dict(zip(r[0], row))
        print("kernel:", d.get("Kernel Name", "")[:120])
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sector_hit_rate.pct",
                "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
                "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
        units = dict(zip(r[0], r[1]))
        for k in keys:
            if k in d:
                print(f"  {k:62s} {d[k]:>16s} {units.get(k, '')}")
        st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(d[k]))
              for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")]
        st = [x for x in st if x[1] > 0.1]
        print("  stall reasons (warps per issue):", ", ".join(f"{k} {v:.2f}" for k, v in sorted(st, key=lambda x: -x[1])))
        # the source page holds one table per captured kernel, each starting with a "Kernel Name" row
        for part in src.split('"Kernel Name"')[1:]:
            rows = list(csv.reader(io.StringIO('"Kernel Name"' + part)))
            base = lambda n: n.split("(")[0].split("<")[0].split("::")[-1].replace("void ", "").strip()
            if len(rows) <= 2 or base(rows[0][1]) != base(d.get("Kernel Name", "")):
                continue
            h = rows[1]
            si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")

            def num(v):
                try:
                    return int(float(v.replace(",", "")))
                except ValueError:
                    return 0

            data = [x for x in rows[2:] if len(x) > max(si, wi, ei)]
            for x in data:
                x[wi], x[ei] = num(x[wi]), num(x[ei])
            tot = sum(x[wi] for x in data) or 1
            print(f"  hottest SASS of {rows[0][1].split('(')[0].strip()} (share of its stall samples):")
            for x in sorted(data, key=lambda x: -x[wi])[:20]:
                print(f"    {100 * x[wi] / tot:5.1f}%  exec {x[ei] / 1e6:8.2f}M  {x[si].strip()[:70]}")
            break


if __name__ == "__main__":
    {"launches": launches, "kernel": kernel}[sys.argv[1]](sys.argv[2])
