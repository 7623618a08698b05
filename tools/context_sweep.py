#!/usr/bin/env python
"""Context sweep and memory footprint of the memory step (SURVEY §8(d) "Extra sweeps").

The paper's claim is that the memory makes the per-frame attention linear
in the context instead of quadratic: with M memory frames and T new frames per step the
attention FLOPs per frame are 4 P (M + T) P D L, i.e. linear in M + T.  This runs the
FuseFormer-shaped step (BASELINE configs[2]) for M in {0, 1, 2, 5, 10, 20} at T = 1 (Eq. 3
exactly) and T = 5, on one GPU, with the memory full, and reports per configuration:
frames/s, step latency (median of CUDA-event-timed graph replays, L2 flushed between
steps), attention FLOPs and device time (kernel self-timing), the log-log slope of
attention FLOPs and time against M + T, and the context's device memory (Table 3 analogue,
P:258-272) -- the K/V slabs (2 L S P D bf16) and everything it owns.

    python tools/context_sweep.py [--steps 50] [--out profiles/r01_context_sweep.jsonl]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_one(cfg, steps, flush):
    import torch

    from paper_2403_16161_b200 import vi
    from vi_synth import make_features, make_weights
    T, P, D, L = cfg.t_new, cfg.tokens, cfg.d_model, cfg.layers
    ctx = vi.Context.from_synth(cfg)
    ctx.set_weights(make_weights(cfg, seed=0))
    stream = torch.cuda.ExternalStream(ctx.stream())
    feats = [torch.from_numpy(make_features(cfg, T, first_frame=i * T, seed=0)).to(torch.bfloat16).cuda()
             for i in range(2)]
    out = torch.empty_like(feats[0])
    for i in range(math.ceil(cfg.mem_frames / T) + 3):      # memory full from here on
        ctx.run_step(feats[i % 2], T, out)
    ctx.sync()
    ctx.profile(1)
    ctx.profile_read()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(k))
            ev[k][0].record(stream)
        ctx.run_step(feats[k % 2], T, out)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(0)
    ms = [a.elapsed_time(b) for a, b in ev]
    slab, total = ctx.footprint()
    ctx.close()
    nk = (cfg.mem_frames + T) * P
    attn_flop_step = 4.0 * T * P * nk * D * L
    attn_ms = prof["attention"][0] / steps
    return {"M": cfg.mem_frames, "T": T, "keys_per_block": nk, "step_ms_p50": statistics.median(ms),
            "frames_per_s": T / (statistics.median(ms) * 1e-3),
            "attn_gflop_per_frame": attn_flop_step / T / 1e9, "attn_ms_per_step": attn_ms,
            "attn_tflops": attn_flop_step / (attn_ms * 1e-3) / 1e12 if attn_ms > 0 else None,
            "slab_MB": slab / 1e6, "ctx_device_MB": total / 1e6}


def slope(xs, ys):
    lx, ly = [math.log(x) for x in xs], [math.log(y) for y in ys]
    mx, my = sum(lx) / len(lx), sum(ly) / len(ly)
    return sum((a - mx) * (b - my) for a, b in zip(lx, ly)) / sum((a - mx) ** 2 for a in lx)


def main():
    import torch

    from vi_synth import CONFIGS
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_context_sweep.jsonl"))
    args = ap.parse_args()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    rows = []
    for T in (1, 5):
        for M in (0, 1, 2, 5, 10, 20):
            cfg = CONFIGS["C3"].replace(t_new=T, mem_frames=M)
            r = run_one(cfg, args.steps, flush)
            rows.append(r)
            print(json.dumps(r), flush=True)
    summary = {}
    for T in (1, 5):
        sel = [r for r in rows if r["T"] == T and r["M"] >= 1]
        ctx = [r["M"] + T for r in sel]
        summary[f"T{T}"] = {
            "loglog_slope_attn_flops_vs_context": slope(ctx, [r["attn_gflop_per_frame"] for r in sel]),
            "loglog_slope_attn_time_vs_context": slope(ctx, [r["attn_ms_per_step"] for r in sel]),
            "loglog_slope_step_time_vs_context": slope(ctx, [r["step_ms_p50"] for r in sel])}
    print(json.dumps({"summary": summary}), flush=True)
    with open(args.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
        f.write(json.dumps({"summary": summary, "device": torch.cuda.get_device_name(0),
                            "note": "C3 shape (8 blocks, 4 heads, D 512, 720 tok/frame), memory full, "
                                    "L2 flushed between steps, median of CUDA-event-timed graph replays"}) + "\n")


if __name__ == "__main__":
    main()
