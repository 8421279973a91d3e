"""Split a kernel's SASS (ncu source page, address order) into segments at
BAR / WARPSYNC-free barrier instructions and print per segment: executed
warp-instructions, stall samples and the top stall reasons, plus the CUDA
lines that dominate the segment.  python tools/ncu_phases.py REPORT KERNEL"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
sass = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and r and r[0].startswith("0x"):
        d = dict(zip(hdr, r))
        sass.append(d)
if not sass:
    print(out[:2000])
    sys.exit(1)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
seg = collections.Counter()
segs = []
cur = {"start": sass[0]["Address"], "inst": 0.0, "samples": 0.0, "r": collections.Counter(), "ops": collections.Counter()}
for d in sass:
    src = d["Source"].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    try:
        n = float(d.get("Instructions Executed", 0) or 0)
        s = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
    except ValueError:
        n = s = 0
    cur["inst"] += n
    cur["samples"] += s
    cur["ops"][op.split(".")[0]] += n
    for k in reasons:
        try:
            cur["r"][k] += float(d.get(k, 0) or 0)
        except ValueError:
            pass
    if op.startswith("BAR") and n > 0:
        cur["end"] = d["Address"]
        segs.append(cur)
        cur = {"start": d["Address"], "inst": 0.0, "samples": 0.0, "r": collections.Counter(), "ops": collections.Counter()}
cur["end"] = sass[-1]["Address"]
segs.append(cur)
T = sum(s["samples"] for s in segs) or 1
I = sum(s["inst"] for s in segs) or 1
for i, s in enumerate(segs):
    if s["samples"] / T < 0.01 and s["inst"] / I < 0.01:
        continue
    top = ", ".join(f"{k[6:]}={100 * v / max(s['samples'], 1):.0f}%" for k, v in s["r"].most_common(5))
    ops = ", ".join(f"{k}:{100 * v / max(s['inst'], 1):.0f}" for k, v in s["ops"].most_common(6))
    print(f"seg {i:2d} {s['start']}..{s['end']}  time {100 * s['samples'] / T:5.1f}%  inst {100 * s['inst'] / I:5.1f}%  | {top}\n         ops {ops}")
