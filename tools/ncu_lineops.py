"""Per-CUDA-source-line executed instructions split into FP math / memory / other, with stall
samples, from an ncu report (needs -lineinfo):  python tools/ncu_lineops.py rep kernel-regex [top]"""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
FP = ("FFMA", "FADD", "FMUL", "FFMA2", "FADD2", "FMUL2")
MEM = ("LDS", "STS", "LDG", "STG", "LDC", "LDCU", "RED", "ATOM", "LDL", "STL", "UBLKPF", "LDGSTS")
per = collections.defaultdict(lambda: [0, 0, 0, 0, ""])  # fp, mem, other, samples, text
cur = None
fname = ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] in ("Address", "Line", "#"):
        hdr = r
        continue
    if len(r) < 8:
        continue
    if r[0].isdigit() and r[2] == "-":      # a CUDA source line row
        cur = (fname, int(r[0]))
        per[cur][4] = r[1].strip()[:90]
        continue
    if r[0] == "" and r[2].startswith("0x") and cur is not None:  # a SASS row under the current line
        toks = r[3].split()
        op = toks[0] if toks else ""
        if op.startswith("@"):
            op = toks[1]
        base = op.split(".")[0]
        try:
            n = float(r[7]); s = float(r[4])
        except ValueError:
            continue
        k = 0 if base in FP else (1 if base in MEM else 2)
        per[cur][k] += n
        per[cur][3] += s
tot = sum(v[0] + v[1] + v[2] for v in per.values()) or 1
tots = sum(v[3] for v in per.values()) or 1
print(f"total inst {tot:.0f}  fp {sum(v[0] for v in per.values())/tot:.1%}  mem {sum(v[1] for v in per.values())/tot:.1%}  other {sum(v[2] for v in per.values())/tot:.1%}")
key = (lambda kv: -(kv[1][2])) if len(sys.argv) > 4 and sys.argv[4] == "other" else (lambda kv: -(kv[1][0] + kv[1][1] + kv[1][2]))
for (f, l), v in sorted(per.items(), key=key)[:top]:
    n = v[0] + v[1] + v[2]
    print(f"{100*n/tot:5.1f}% inst (fp {100*v[0]/tot:4.1f} mem {100*v[1]/tot:4.1f} oth {100*v[2]/tot:4.1f})  stall {100*v[3]/tots:5.1f}%  {f}:{l:<5} {v[4]}")
