"""Executed warp-instructions of one kernel in an ncu report, by CUDA source
line and by SASS opcode (needs -lineinfo and --import-source):
    python tools/ncu_inst.py REPORT KERNEL_REGEX [N_LINES] [UNITS_SYMBOLS]
UNITS_SYMBOLS (optional) divides the counts into per-symbol figures."""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
div = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
by_line, by_op, src_txt = collections.Counter(), collections.Counter(), {}
fname, cur = "", None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" or r[0] == "Function Name":
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]))
        src_txt[cur] = r[1].strip()[:90]
        continue
    if r[0] == "" and len(r) > 7 and r[2].startswith("0x"):
        try:
            n = float(r[7])
        except ValueError:
            continue
        op = r[3].strip().split()[0] if r[3].strip() else "?"
        if op.startswith("@"):
            op = r[3].strip().split()[1]
        by_op[op.split(".")[0]] += n
        if cur:
            by_line[cur] += n
tot = sum(by_op.values())
print(f"total warp-instructions {tot:.4g}  (/{div:g} = {tot / div:.1f})")
print("-- by opcode")
for op, n in by_op.most_common(28):
    print(f"  {op:10s} {100 * n / tot:5.1f}%  {n / div:10.1f}")
print("-- by source line")
for k, n in by_line.most_common(top):
    print(f"  {100 * n / tot:5.1f}% {n / div:9.1f}  {k[0]}:{k[1]:<5} {src_txt.get(k, '')}")
