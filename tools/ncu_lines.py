"""Per CUDA-source-line totals of an ncu source page (cuda,sass): warp
instructions executed, thread instructions, stall samples.
usage: python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
rows = []
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            rows.append((f, int(r[0]), r[1].strip()[:70], int(r[7]), int(r[8]), int(r[6])))
        except ValueError:
            pass
ti = sum(r[3] for r in rows) or 1
ts = sum(r[5] for r in rows) or 1
print(f"total warp inst {ti:.4g}")
for r in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{r[0][:18]:18s}:{r[1]:<5d} inst {r[3]/ti:6.3f} thr/inst {r[4]/max(r[3],1):5.1f} "
          f"stall {r[5]/ts:6.3f}  {r[2]}")
