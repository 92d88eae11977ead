"""Group an ncu SASS source page into runs of equal execution count (code regions)."""
import csv, subprocess, sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.003
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))[2:]
tot = sum(int(r[5]) for r in rows)
samp = sum(int(r[2]) for r in rows) or 1
print("total warp inst %.4g, samples %d" % (tot, samp))
prev = None; groups = []
for r in rows:
    ex = int(r[5])
    if prev is None or abs(ex - prev) > 0.02 * max(prev, 1):
        groups.append([r[0][-5:] + " " + r[1].strip()[:38], 0, ex, 0, 0])
    g = groups[-1]; g[1] += 1; g[3] += ex; g[4] += int(r[2]); prev = ex
for g in groups:
    if g[3] > thr * tot:
        print(f"{g[0]:46s} n={g[1]:4d} exec={g[2]:>12d} share={g[3]/tot:.3f} stall={g[4]/samp:.3f}")
