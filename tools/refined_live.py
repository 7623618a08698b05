#!/usr/bin/env python
"""Refined dual-model live run at BASELINE configs[4].

FuseFormer-shaped online inpainter (8 blocks, 4 heads, D 512, 720 tokens/frame, memory
span M = 10, one frame per step) on a 300-frame synthetic 432x240 stream (feature maps
60x108x128 ~N(0,1), one moving rectangle covering 10-30 % zeroed), with and without an
identical-shape refining inpainter that re-inpaints the last 20 frames jointly every 5
frames and overwrites their K/V in the online memory (vi_memory_read -> vi_refine_commit).
Both on one GPU (one live stream per GPU; `--gpus N` under torchrun runs N independent
streams), the online context on a high-priority stream, the refiner in its own host thread.

Reports per stream: online frames/s and per-frame latency (live-paced loop), refiner
windows and commits, the refiner's lag behind the online frame, and the online fps
ratio refiner-on / refiner-off (the paper's Refined-vs-Memory FPS comparison, P:178-220,
context only: 2080 Ti numbers).

    python tools/refined_live.py [--frames 300] [--out profiles/r02_refined_live.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2403_16161_b200 import streams
    from paper_2403_16161_b200.refined import RefinedRun
    from vi_synth import CONFIGS, make_features, make_weights
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=300)
    ap.add_argument("--window", type=int, default=20)
    ap.add_argument("--every", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_refined_live.jsonl"))
    ap.add_argument("--refined-span", type=int, default=10, help="s' of Eq. 4's refined memory")
    ap.add_argument("--refined-rate", type=int, default=10, help="r' of Eq. 4's refined references")
    ap.add_argument("--refined-refs", type=int, default=2, help="refined references kept")
    args = ap.parse_args()
    info = streams.DistInfo.from_env()
    torch.cuda.set_device(info.local_rank)
    streams.init("nccl", info, torch.device("cuda", info.local_rank))
    cfg = CONFIGS["C3T1"]                      # T = 1, M = 10: Eq. 3 / Eq. 4's online inpainter
    w = make_weights(cfg, seed=0)
    seed = streams.stream_seed(info.rank)
    feats = torch.from_numpy(make_features(cfg, args.frames, seed=seed, masked="moving")).to(torch.bfloat16).cuda()
    out = torch.empty_like(feats)
    lines = []
    # (refiner, Eq. 4 inputs): the Memory model; Refined with the round-1 hand-off (commits
    # overwrite online frames only); Eq. 4 in full (online span + refined span s' + refined
    # references every r'); and the FPS side of the paper's input ablation (Table 4):
    # Eq. 4 without refined references, and with the refined span cut to the watermark frame
    variants = [("memory", False, None, 0, 0),
                ("refined_overwrite_only", True, None, 0, 0),
                ("refined_eq4", True, args.refined_span, args.refined_rate, args.refined_refs),
                ("refined_eq4_no_refined_refs", True, args.refined_span, 0, 0),
                ("refined_eq4_span0", True, 0, args.refined_rate, args.refined_refs)]
    for name, refiner, sr, rr, RR in variants:
        kw = dict(window=args.window, every=args.every, refiner=refiner, device_online=info.local_rank,
                  refined_span=sr, refined_rate=rr, max_refined_refs=RR)
        run = RefinedRun(cfg, w, **kw)
        run.run(feats[:25], out[:25])           # warm-up: graphs captured, memory filled
        run.close()
        run = RefinedRun(cfg, w, **kw)
        secs = run.run(feats, out)
        secs = streams.max_over_ranks([secs], torch.device("cuda", info.local_rank))[0]
        st = run.stats
        line = {"metric": "refined live run: online frames/s per stream", "config": "C5 (BASELINE configs[4])",
                "variant": name, "refiner": refiner, "refined_span": sr, "refined_rate": rr, "refined_refs": RR,
                "online_memory_slots": run.online.S, "watermark": st["watermark"],
                "frames": args.frames, "streams": info.world,
                "online_fps_per_stream": args.frames / secs, "online_ms_per_frame": 1e3 * secs / args.frames,
                "refiner_windows": st["windows"], "refine_commits": st["commits"],
                "commits_not_resident": st["not_resident"],
                "refiner_ms_per_window": 1e3 * st["refine_s"] / st["windows"] if st["windows"] else None,
                "refiner_lag_frames_median": statistics.median(st["lag_frames"]) if st["lag_frames"] else None,
                "window": args.window, "every": args.every, "online_mem_frames": cfg.mem_frames,
                "data": "synthetic 60x108x128 features, moving 10-30% rectangle mask, seeded N(0,0.02) weights"}
        run.close()
        lines.append(line)
        if info.rank == 0:
            print(json.dumps(line), flush=True)
    if info.rank == 0:
        ratio = lines[2]["online_fps_per_stream"] / lines[0]["online_fps_per_stream"]
        summ = {"online_fps_ratio_refined_eq4_vs_memory": ratio,
                "paper_context": "FuseFormer + Memory 31.0 FPS on 1 RTX 2080 Ti vs + Refined 21.3 FPS on 2 "
                                 "(DAVIS, P:185-186; SURVEY §6); here one B200 hosts both inpainters"}
        print(json.dumps(summ), flush=True)
        with open(args.out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")
            f.write(json.dumps(summ) + "\n")


if __name__ == "__main__":
    main()
