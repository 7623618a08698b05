"""Summarise ncu output into profiles/ (tracked evidence).

    python tools/ncu_summary.py launches <launches.csv> <out.csv>   # compact per-launch table
    python tools/ncu_summary.py full <report.ncu-rep> <out.md> [--traffic profiles/attention_traffic.json]

`launches` keeps ID, kernel, grid, duration (us), tensor-pipe %, DRAM read/write (MB) per launch
of a `--metrics gpu__time_duration.sum,...` capture (cold-cache, serialised: compare shares).
`full` extracts the headline metrics of each profiled launch of a `--set full` capture and,
with --traffic, writes the mean DRAM bytes per launch that bench.py reports as roofline.traffic.
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    idx = {h: i for i, h in enumerate(rows[0])}
    seq = collections.OrderedDict()
    for r in rows[1:]:
        if r[idx["ID"]] == "ID":
            continue
        d = seq.setdefault(int(r[idx["ID"]]), {"kernel": r[idx["Kernel Name"]].split("(")[0],
                                               "grid": r[idx["Grid Size"]]})
        d[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "us", "tensor_pct", "dram_read_MB", "dram_write_MB"])
        for k, d in seq.items():
            w.writerow([k, d["kernel"], d["grid"], round(d.get("gpu__time_duration.sum", 0) / 1e3, 2),
                        round(d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0), 1),
                        round(d.get("dram__bytes_read.sum", 0) / 1e6, 2),
                        round(d.get("dram__bytes_write.sum", 0) / 1e6, 2)])
    print(f"{len(seq)} launches -> {dst}")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "smsp__warps_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def full(rep, dst, traffic=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary of `{rep.split('/')[-1]}`", ""]
    dram = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"## {d['Kernel Name'][:100]}")
        for k in KEYS:
            if k in d:
                lines.append(f"- `{k}` = {d[k]} {u.get(k, '')}")
        try:
            dram.append(float(d["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]]
                        + float(d["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]])
        except (KeyError, ValueError):
            pass
        lines.append("")
    open(dst, "w").write("\n".join(lines) + "\n")
    print(f"{len(rows) - 2} profiled launches -> {dst}")
    if traffic and dram:
        json.dump({"dram_bytes_per_launch": sum(dram) / len(dram), "launches": len(dram),
                   "source": rep.split("/")[-1]}, open(traffic, "w"), indent=1)
        print(f"traffic {sum(dram) / len(dram):.4g} B/launch -> {traffic}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None)
