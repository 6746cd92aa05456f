#!/usr/bin/env python
"""Instruction-count histogram of an ncu capture (source page, SASS), per kernel: groups SASS lines
by execution count (~ one basic block), largest instruction share first.
  python tools/sass_hist.py <prof.ncu-rep> [n_groups] [--kernel SUBSTR] [--dump MIN_EXEC [MAX_EXEC]]"""
import csv, collections, io, subprocess, sys
path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
ksel = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else ""
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for part in raw.split('"Kernel Name"')[1:]:
    r = list(csv.reader(io.StringIO('"Kernel Name"' + part)))
    name = r[0][1]
    if ksel not in name:
        continue
    h = r[1]; rows = [x for x in r[2:] if len(x) == len(h)]
    ie = h.index("Instructions Executed"); src = h.index("Source"); st = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[ie]) for x in rows); sst = sum(int(x[st]) for x in rows) or 1
    print(f"== {name[:90]}\ntotal inst {tot:,}  stall samples {sst:,}")
    b = collections.Counter(); bs = collections.Counter(); nb = collections.Counter()
    for x in rows:
        e = int(x[ie]); b[e] += e; bs[e] += int(x[st]); nb[e] += 1
    for e, v in sorted(b.items(), key=lambda kv: -kv[1])[:n]:
        print(f"exec {e:10d} n_instr {nb[e]:4d} inst share {v / tot:6.3f} stall share {bs[e] / sst:6.3f}")
    if "--dump" in sys.argv:
        k = sys.argv.index("--dump")
        lo = int(sys.argv[k + 1])
        hi = int(sys.argv[k + 2]) if len(sys.argv) > k + 2 and sys.argv[k + 2].isdigit() else 1 << 62
        for x in rows:
            if lo <= int(x[ie]) <= hi:
                print(f"{int(x[ie]):9d} {x[st]:>6s} {x[src]}")
