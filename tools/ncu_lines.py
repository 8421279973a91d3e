"""Per-CUDA-source-line stall samples from an ncu report (needs -lineinfo)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res, fname = [], ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[2] == "-" and r[0].isdigit():
        try:
            res.append((float(r[4]), float(r[7] or 0), fname, int(r[0]), r[1].strip()[:100]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
for s, inst, f, l, src in sorted(res, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 35]:
    print(f"{100*s/tot:5.1f}%  inst={inst:>12.0f}  {f}:{l:<5} {src}")
