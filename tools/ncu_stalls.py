"""Summarise warp-stall sampling of an ncu report by instruction group.

    python tools/ncu_stalls.py report.ncu-rep [--top 30] [--exec N]

Groups instructions by execution count (the per-key-tile softmax body runs once per tile
per warp), prints the stall-reason totals per group and the top instructions."""
import argparse
import csv
import collections
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--exec", type=int, default=0, help="only instructions executed exactly N times")
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
col = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
f = lambda r, k: float(r[col[k]] or 0)
groups = collections.defaultdict(lambda: collections.Counter())
for r in data:
    ex = int(float(r[col["Instructions Executed"]] or 0))
    g = groups[ex]
    g["_n"] += 1
    for k in reasons:
        g[k] += f(r, k)
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"total samples {tot:.0f}")
big = sorted(groups.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "_n"))[:8]
for ex, g in big:
    s = sum(v for k, v in g.items() if k != "_n")
    top = ", ".join(f"{k[6:]} {v:.0f}" for k, v in g.most_common(8) if k != "_n")
    print(f"exec {ex:>9} n_instr {g['_n']:>5} samples {s:>6.0f}: {top}")
sel = [r for r in data if not args.exec or int(float(r[col["Instructions Executed"]] or 0)) == args.exec]
for r in sorted(sel, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:args.top]:
    rs = sorted(((f(r, k), k[6:]) for k in reasons), reverse=True)[:3]
    print(r[col["Address"]][-5:], f"{f(r, 'Warp Stall Sampling (All Samples)'):5.0f}", r[col["Source"]][:60].ljust(60),
          " ".join(f"{k}:{v:.0f}" for v, k in rs if v))
