"""Oracle timing (SURVEY.md §8(d) "Oracle timing"): the fp64 oracle as it stands, timed on
the host cores at C3 (T = 5), C3T1 (T = 1) and the full C1, once on all cores and once on ONE
core (BLAS threads pinned with threadpoolctl).  Every timed step is a WHOLE oracle memory step
(bench.oracle_step: soft split + embedding of the new frames, every block against a full memory,
back-projection + composite).  A reported baseline, not the target.

    python tools/oracle_timing.py [--steps 3] [--configs C3,C3T1,C1] [--out FILE.jsonl]

One JSON line per (config, cores).  Test infrastructure: it imports oracle/ through bench.py's
cpu-baseline helpers and never touches the GPU.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (oracle_memory / oracle_step / cpu_threads)
from vi_synth import CONFIGS  # noqa: E402


def time_config(name, steps, one_core):
    from threadpoolctl import threadpool_limits
    cfg = CONFIGS[name]
    w, mem = bench.oracle_memory(cfg)
    limits = 1 if one_core else None
    with threadpool_limits(limits=limits):
        cores = 1 if one_core else bench.cpu_threads()
        bench.oracle_step(cfg, w, mem, seed=99)          # untimed warm-up
        ts = [bench.oracle_step(cfg, w, mem, seed=s) for s in range(steps)]
    total = sum(ts)
    return {"config": name, "cores": cores, "affinity_cores": len(os.sched_getaffinity(0)), "steps": steps,
            "frames_per_step": cfg.t_new, "s_per_step": [round(t, 3) for t in ts],
            "frames_per_s": steps * cfg.t_new / total, "kind": "oracle (fp64, plain NumPy)",
            "label": "reported baseline, not the target",
            "work": f"{cfg.layers} blocks, {cfg.t_new} new frames x {cfg.tokens} tokens against "
                    f"{cfg.mem_frames} memory frames, split/embed + composite"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--configs", default="C3,C3T1,C1")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    out = open(args.out, "w") if args.out else None
    for name in args.configs.split(","):
        for one_core in (False, True):
            t0 = time.perf_counter()
            line = time_config(name, args.steps, one_core)
            line["wall_s"] = round(time.perf_counter() - t0, 1)
            s = json.dumps(line)
            print(s, flush=True)
            if out:
                out.write(s + "\n")
                out.flush()


if __name__ == "__main__":
    main()
