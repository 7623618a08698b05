#!/usr/bin/env python
"""Online baseline (Eq. 2) vs Memory model (Eq. 3) at the C3 shape.

The paper's speed claim (Memory ~3x faster than Online for DSTT/FuseFormer)
comes from the Online baseline recomputing a whole window for every output frame: for
frame f it runs the transformer jointly over the window f-k .. f and keeps only frame f's
prediction, while the Memory model computes only frame f's queries against the
cached K/V of f-k .. f-1.  Both run here through the same kernels: Online = a
context with M = 0 and a chunk of k+1 frames per output frame; Memory = M = k, one frame
per step.  Same context (k+1 frames), same synthetic inputs; frames/s per stream (graph
replays, CUDA events, L2 flushed between steps).

    python tools/online_vs_memory.py [--k 10] [--steps 30]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def time_steps(cfg, n, steps, flush):
    import torch

    from paper_2403_16161_b200 import vi
    from vi_synth import make_features, make_weights
    ctx = vi.Context.from_synth(cfg)
    ctx.set_weights(make_weights(cfg, seed=0))
    stream = torch.cuda.ExternalStream(ctx.stream())
    feats = torch.from_numpy(make_features(cfg, n, seed=0)).to(torch.bfloat16).cuda()
    out = torch.empty_like(feats)
    for _ in range(cfg.mem_frames + 3):
        ctx.run_step(feats, n, out)
    ctx.sync()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(k))
            ev[k][0].record(stream)
        ctx.run_step(feats, n, out)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    ctx.close()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def main():
    import torch

    from vi_synth import CONFIGS
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_online_vs_memory.jsonl"))
    args = ap.parse_args()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    k = args.k
    online_ms = time_steps(CONFIGS["C3"].replace(t_new=k + 1, mem_frames=0), k + 1, args.steps, flush)
    memory_ms = time_steps(CONFIGS["C3"].replace(t_new=1, mem_frames=k), 1, args.steps, flush)
    line = {"config": f"C3 shape, context k+1 = {k + 1} frames", "online_ms_per_output_frame": online_ms,
            "memory_ms_per_output_frame": memory_ms, "online_fps": 1e3 / online_ms, "memory_fps": 1e3 / memory_ms,
            "memory_vs_online_speedup": online_ms / memory_ms,
            "paper_context": "x3 for DSTT / FuseFormer, x2 for E2FGVI on RTX 2080 Ti (P:24, P:252)"}
    print(json.dumps(line), flush=True)
    with open(args.out, "w") as f:
        f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
