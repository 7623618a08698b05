#!/usr/bin/env python
"""Benchmark of the memory step (BASELINE.json metric: "memory-step frames/s per stream at
720-tok/frame shape; attn % bf16 peak") on the FuseFormer-shaped config (configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3|C3T1]

One step = vi_memory_push(5) + soft split/embedding + 8 memory blocks (3600 queries over
the 10800 keys of a full 15-slot ring per block) + back-projection/composite, on 5 new
frames, through libvi.so.  N GPUs = N independent live streams, one per GPU (weak
scaling, no data-path collective: the streams are independent problems).  Inputs are
resident in HBM; L2 is flushed (256 MiB write) between timed steps.  Rank 0 prints one
JSON line.  --impl reference times the fp64 CPU oracle (oracle/) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "memory-step frames/s per stream at 720-tok/frame shape; attn % bf16 peak"
UNIT = "frames/s"


def peaks():
    """Roofline denominators: the driver-measured MEASURED_PEAKS.json (bf16 dense burst, HBM
    copy); without it the profiling guide's fallback figures, labelled "fallback"."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 1590.0, 6650.0, "fallback (B200_PROFILING.md: no MEASURED_PEAKS.json)"


WORKLOADS = {"C3": "FuseFormer-shaped memory step (BASELINE.json configs[2])",
             "C3T1": "FuseFormer-shaped memory step, one new frame per step (Eq. 3; configs[2] shape, T=1)",
             "C2": "STTN-shaped memory step (BASELINE.json configs[1])",
             "C4": "E2FGVI-shaped memory step, 5x9-token window attention (BASELINE.json configs[3])"}


def gemm_flop_per_step(cfg):
    """Algorithmic GEMM FLOPs of one step (the back-projection's hi/lo split not counted)."""
    M, D, F, Pd, L = cfg.t_new * cfg.tokens, cfg.d_model, cfg.ffn_hidden, cfg.patch_dim, cfg.layers
    return 2.0 * M * (D * Pd + L * (3 * D * D + D * D + 2 * F * D) + Pd * D)


def patch_bytes_per_step(cfg):
    """ALGORITHMIC HBM bytes of the patch kernels of one step (SURVEY §8(d) / §8(a) rows a1, a10,
    a13: bf16 features, tokens, patch vectors and F3N hidden): split = read the map + write the
    tokens; composite = read the patch vectors + write the map; F3N per block = read the hidden
    (fold) + write the re-split hidden (unfold), the small fold map itself not counted.  C3:
    66.6 MB per frame, 333 MB per 5-frame step."""
    T, P, Pd = cfg.t_new, cfg.tokens, cfg.patch_dim
    fmap = T * cfg.feat_h * cfg.feat_w * cfg.feat_c * 2
    tok = T * P * Pd * 2
    b = (fmap + tok) + (tok + fmap)
    if cfg.ffn_kind == 1:
        b += cfg.layers * 2 * (T * P * cfg.ffn_hidden * 2)
    return float(b)


def patch_bytes_implementation(cfg):
    """The bytes this implementation's patch kernels move per step (the F3N hidden u and the
    back-projection output Yp are kept fp32 for precision; the fold map read by
    the unfold counted): reported beside the algorithmic figure."""
    T, P, Pd = cfg.t_new, cfg.tokens, cfg.patch_dim
    fmap = T * cfg.feat_h * cfg.feat_w * cfg.feat_c * 2
    b = fmap + T * P * Pd * 2                       # split: read features, write tokens
    b += T * P * Pd * 4 + fmap                      # composite: read fp32 Yp, write features
    if cfg.ffn_kind == 1:
        C = cfg.ffn_hidden // (cfg.kh * cfg.kw)
        fold = T * cfg.feat_h * cfg.feat_w * C * 2
        b += cfg.layers * ((T * P * cfg.ffn_hidden * 4 + fold) + (fold + T * P * cfg.ffn_hidden * 2))
    return float(b)


def workload_config(cfg, args=None, world=1):
    return {"workload": f"{cfg.name}: {WORKLOADS[cfg.name]}",
            "layers": cfg.layers, "heads": cfg.heads, "d_model": cfg.d_model, "tokens_per_frame": cfg.tokens,
            "new_frames_per_step": cfg.t_new, "mem_frames": cfg.mem_frames,
            "keys_per_block": cfg.slots * cfg.tokens, "queries_per_block": cfg.t_new * cfg.tokens,
            "keys_per_query": cfg.slots * (cfg.win_h * cfg.win_w if cfg.win_h else cfg.tokens),
            "feature_map": [cfg.feat_h, cfg.feat_w, cfg.feat_c],
            "ffn": f"F3N {cfg.ffn_hidden}" if cfg.ffn_kind == 1 else f"MLP-GELU {cfg.ffn_hidden}",
            "l2": "flushed between timed steps (256 MiB write)",
            "parallelism": (f"heads sharded over {world} GPUs (NCCL all-gather per block), 1 stream"
                            if args is not None and args.tp else f"{world} independent live streams, 1 per GPU")}


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                s, m = float(f[1]), float(f[2])
            except ValueError:
                continue
            smax = m
            sm.append(s)
            names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        load = [s for s in sm if smax and s > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return len(os.sched_getaffinity(0))


def oracle_memory(cfg, seed=0):
    """A full memory for the oracle: per block, the K/V of cfg.mem_frames resident frames,
    projected (oracle.qkv) from seeded random block inputs (the values do not change the
    work; the oracle's own stream would need mem_frames / T extra steps to fill it)."""
    from oracle import vi_oracle as O
    from vi_synth import make_weights, rng_for
    w = make_weights(cfg, seed=seed)
    rng = rng_for(seed, "oracle-mem")
    mem = []
    for l in range(cfg.layers):
        kv = []
        for j in range(cfg.mem_frames):
            _, _, K, V = O.qkv(rng.standard_normal((cfg.tokens, cfg.d_model)), w, l, cfg)
            kv.append((K, V))
        mem.append(kv)
    return w, mem


def oracle_step(cfg, w, mem, seed=0, layers=None):
    """One WHOLE memory step of the fp64 oracle (no extrapolation): soft split + embedding of
    the T new frames, every block against its full memory, back-projection + composite.
    `layers` < cfg.layers runs only the first blocks (used for the 1-core sample).  Returns
    the seconds it took."""
    from oracle import vi_oracle as O
    from vi_synth import make_features
    feats = make_features(cfg, cfg.t_new, first_frame=cfg.mem_frames, seed=seed)
    t0 = time.perf_counter()
    _, X = O.embed(feats, w, cfg)
    for l in range(cfg.layers if layers is None else layers):
        X, _ = O.block_memory(X, mem[l], w, l, cfg, cfg.t_new)
    O.compose(X, w, cfg, cfg.t_new)
    return time.perf_counter() - t0


def run_reference(args, cfg):
    """--impl reference: the fp64 oracle as it stands, on the host cores, on this arm's config
    and metric.  Every timed step is a whole oracle memory step (5 frames through all blocks
    against a full memory); the run is bounded in time: it stops after the step that crosses
    REF_BUDGET_S seconds (at least one step), and prints the steps it actually timed."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    budget = float(os.environ.get("REF_BUDGET_S", "90"))
    w, mem = oracle_memory(cfg)
    warm = min(args.warmup, 1)                   # nothing to warm up in NumPy beyond one step
    for _ in range(warm):
        oracle_step(cfg, w, mem)
    steps = []
    while len(steps) < args.steps and (not steps or sum(steps) < budget):
        steps.append(oracle_step(cfg, w, mem, seed=len(steps)))
    total = sum(steps)
    value = len(steps) * cfg.t_new / total
    cores = cpu_threads()
    sample = (f"{len(steps)} whole oracle steps (of {args.steps} requested; time budget {budget:.0f} s): soft split + "
              f"embedding of {cfg.t_new} frames, all {cfg.layers} blocks against a full {cfg.mem_frames}-frame "
              f"memory, composite; {warm} untimed warm-up step")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": len(steps),
            "steps_requested": args.steps, "warmup": warm, "ms_per_step": 1000 * total / len(steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args, args.gpus), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg):
    """The oracle timed beside the GPU (rank 0, N = 1): one whole step on all host cores, and
    one block (+ split/embedding + composite) on ONE core, scaled to a step (stated)."""
    from threadpoolctl import threadpool_limits
    w, mem = oracle_memory(cfg)
    t_all = oracle_step(cfg, w, mem)
    with threadpool_limits(limits=1):
        t1_block = oracle_step(cfg, w, mem, layers=1)
        t1_embed = oracle_step(cfg, w, mem, layers=0)
    t1_step = t1_embed + cfg.layers * (t1_block - t1_embed)
    return {"value": cfg.t_new / t_all, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
            "sample": f"1 whole step ({cfg.t_new} frames, {cfg.layers} blocks against a full {cfg.mem_frames}-frame "
                      f"memory, split/embed and composite): {t_all:.1f} s on all cores",
            "one_core": {"value": cfg.t_new / t1_step, "unit": UNIT, "cores": 1,
                         "sample": f"split/embed + 1 block + composite on 1 core ({t1_block:.1f} s), the block time "
                                   f"x{cfg.layers} (scaled, not run)"}}


def run_ours(args, cfg):
    import torch

    from paper_2403_16161_b200 import streams, vi
    from vi_synth import make_features, make_weights

    info = streams.DistInfo.from_env()
    world, rank, local = info.world, info.rank, info.local_rank
    torch.cuda.set_device(local)
    streams.init("nccl", info, torch.device("cuda", local))

    T, P, D = cfg.t_new, cfg.tokens, cfg.d_model
    if args.tp:
        # one live stream, heads sharded over the N ranks (NCCL all-gather of the head
        # outputs inside every block): strong scaling of one stream's step latency
        nccl_id = streams.broadcast_bytes(vi.tp_unique_id() if rank == 0 else None, torch.device("cuda", local))
        ctx = vi.Context.from_synth(cfg, device=local, tp_size=world, tp_rank=rank, nccl_id=nccl_id)
        n_streams = 1
    else:
        ctx = vi.Context.from_synth(cfg, device=local)   # one independent live stream per GPU
        n_streams = world
    w = make_weights(cfg, seed=0)
    ctx.set_weights(w)
    stream = torch.cuda.ExternalStream(ctx.stream())
    dt = torch.bfloat16
    nchunks = 4
    seed = streams.stream_seed(0 if args.tp else streams.stream_ids(rank, world, world)[0])
    feats = [torch.from_numpy(make_features(cfg, T, first_frame=i * T, seed=seed)).to(dt).cuda()
             for i in range(nchunks)]
    out = torch.empty_like(feats[0])
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()

    warm = max(args.warmup, math.ceil(cfg.mem_frames / T) + 1)   # the memory is full from here on
    for i in range(warm):
        ctx.run_step(feats[i % nchunks], T, out)
    ctx.sync()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    # the timed steps run uninstrumented (profile mode 0): the kernels' self-timing (one
    # atomic per CTA, ~960 CTAs per split-merge launch) lengthened the C3 step by ~20 us
    # (1.301 vs 1.282 ms, same box); the attention's device time comes from an instrumented
    # 20-step sub-run of the same workload below (profile modes 1 and 4)
    ctx.profile(int(os.environ.get("VI_PROFILE_MODE", "0")))
    # untimed: records + uploads this profile mode's step graphs, one per (ring state, input
    # buffer) pair, so that no graph is captured inside the timed region (C3T1: 11 x 4)
    for k in range(nchunks * (cfg.mem_frames + T)):
        ctx.run_step(feats[k % nchunks], T, out)
    ctx.profile_read()                 # (and resets the kernel self-timing)
    l0 = ctx.launches()
    streams.barrier()
    torch.cuda.synchronize()
    # an untimed ~25 ms device sleep lets the host queue the steps ahead of the GPU, so a host
    # hiccup (the clock sampler's process, GC) never leaves the stream idle inside a step
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(5e7))
    k0 = nchunks * (cfg.mem_frames + T)   # (continues the warm-up's buffer / ring-state cycle)
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(k))                   # untimed L2 flush
            starts[k].record(stream)
        ctx.run_step(feats[(k0 + k) % nchunks], T, out)
        ends[k].record(stream)
    torch.cuda.synchronize()
    streams.barrier()
    launches = ctx.launches() - l0
    prof = ctx.profile_read()
    ctx.profile(0)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)

    # end to end through the public API with host (pinned) buffers, copies inside
    # (vi_run_step_async: the copies of a step overlap the neighbouring steps' compute, the
    # way a live stream feeds the library; every step's H2D and D2H are inside the timed region)
    e2e_steps = max(3, min(args.steps, 50))
    host_in = [f.cpu().pin_memory() for f in feats]
    host_out = [torch.empty(out.shape, dtype=dt).pin_memory() for _ in range(e2e_steps)]
    # untimed: creates the copy streams and staging slots, and captures the step graph of every
    # (ring state, staging slot) pair (two staging slots alternate)
    for k in range(2 * (cfg.mem_frames + T)):
        ctx.run_step_async(host_in[k % nchunks], T, host_out[k % e2e_steps])
    ctx.sync()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        ctx.run_step_async(host_in[k % nchunks], T, host_out[k])
    ctx.sync()                                           # every result has landed in host memory
    e2e_s = time.perf_counter() - t0
    clk = clocks.stop()

    # secondary rooflines and determinism (outside the timed region): the GEMMs' own device
    # time (self-timing inside the graph), the HBM-bound patch kernels' (CUDA events around
    # eager launches), and two replays of one step compared bitwise (no atomics anywhere)
    extra_steps = 20
    sub = {}
    for mode in (3, 2, 4, 1):
        ctx.profile(mode)
        ctx.profile_read()
        for k in range(extra_steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(k))
            ctx.run_step(feats[k % nchunks], T, out)
        sub[mode] = ctx.profile_read()
    ctx.profile(0)
    # run-to-run determinism: two fresh contexts, the same weights and frames -> bitwise
    # identical outputs after the memory is full (no atomics on the path)
    outs = []
    for _ in range(2):
        nid = None
        if args.tp:           # an NCCL id serves one communicator: a fresh one per context
            nid = streams.broadcast_bytes(vi.tp_unique_id() if rank == 0 else None, torch.device("cuda", local))
        c2 = vi.Context.from_synth(cfg, device=local, tp_size=world if args.tp else 1, tp_rank=rank if args.tp else 0,
                                   nccl_id=nid)
        c2.set_weights(w)
        o2 = torch.empty_like(out)
        for k in range(math.ceil(cfg.mem_frames / T) + 2):
            c2.run_step(feats[k % nchunks], T, o2)
        c2.sync()
        outs.append(o2)
        c2.close()
    deterministic = bool(torch.equal(outs[0], outs[1]))

    total_ms, e2e_s = streams.max_over_ranks([total_ms, e2e_s], torch.device("cuda", local))
    value = streams.aggregate_fps(T * args.steps, n_streams, total_ms / 1e3)
    e2e_value = streams.aggregate_fps(T * e2e_steps, n_streams, e2e_s)
    bf16_peak, hbm_peak, peak_src = peaks()
    # attention device time per step: from the timed region when it ran instrumented
    # (VI_PROFILE_MODE=1), else from the instrumented sub-run (profile mode 1, same workload)
    if prof["attention"][0] > 0:
        attn_step_ms, attn_src = prof["attention"][0] / args.steps, "kernel self-timing inside the timed steps"
    else:
        attn_step_ms = sub[1]["attention"][0] / extra_steps
        attn_src = (f"kernel self-timing in an instrumented {extra_steps}-step sub-run (profile mode 1; "
                    "the timed steps run uninstrumented)")
    attn_ms = attn_step_ms * args.steps
    per_block_ms = attn_step_ms / cfg.layers if attn_step_ms > 0 else float("nan")
    nq, nk = T * P, cfg.slots * (cfg.win_h * cfg.win_w if cfg.win_h else P)   # keys a query sees
    attn_flop = 4.0 * nq * nk * D / (world if args.tp else 1)   # this rank's share when head-sharded
    achieved = attn_flop / (per_block_ms * 1e-3) / 1e12 if attn_ms > 0 else float("nan")
    # which attention path engine.cu takes for this shape (mirrors its dispatch)
    heads_local = cfg.heads // world if args.tp else cfg.heads
    if cfg.win_h:
        attn_kernel = "attn_sk2_kernel, one CTA per (head, window, query pair)"
    elif ((nq + 255) // 256) * heads_local * 4 < 148:
        attn_kernel = "attn_tc2_kernel KV split + attn_combine_kernel"
    else:
        attn_kernel = "attn_sk2_kernel, persistent stream-K, column-split softmax"
    traffic = None                     # ncu DRAM bytes per launch, captured on the default C3 run
    if args.config == "C3" and not args.tp:
        try:
            with open(os.path.join(ROOT, "profiles", "attention_traffic.json")) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.tp else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) features, N(0,0.02) weights)",
        "config": workload_config(cfg, args, world),
        "fps_per_stream": value / n_streams,
        "step_latency_ms": {"p50": statistics.median(step_ms), "p5": sorted(step_ms)[int(0.05 * len(step_ms))],
                            "p95": sorted(step_ms)[min(len(step_ms) - 1, int(0.95 * len(step_ms)))],
                            "max": max(step_ms)},
        "roofline": {"kernel": f"memory attention ({attn_kernel}), per block",
                     "bound": "tensor", "achieved": achieved, "peak": bf16_peak, "unit": "TFLOP/s",
                     "frac": achieved / bf16_peak, "traffic": traffic,
                     "flop_per_launch": attn_flop, "avg_launch_ms": per_block_ms,
                     "peak_source": f"{peak_src} bf16 dense (burst)",
                     "share_of_step": attn_ms / total_ms, "timing": attn_src},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": host_in[0].numel() * 2,
                "d2h_bytes_per_step": host_out[0].numel() * 2,
                "api": "vi_run_step_async (pinned host buffers; copies overlap neighbouring steps)"},
        # per-frame latency of a live source: frame i of a T-frame chunk waits for the T-1-i
        # frames after it (batching delay), then for the step; at a 25 fps source and at a source
        # delivering frames as fast as this run processes them
        "frame_latency_ms": {
            "step_p50": statistics.median(step_ms),
            "source_25fps": {"first_frame": (T - 1) * 40.0 + statistics.median(step_ms),
                             "mean": (T - 1) / 2 * 40.0 + statistics.median(step_ms)},
            "source_at_processing_rate": {
                "first_frame": (T - 1) * total_ms / (args.steps * T) + statistics.median(step_ms),
                "mean": (T - 1) / 2 * total_ms / (args.steps * T) + statistics.median(step_ms)}},
        "gpu_launches": launches,
        "clocks": clk,
    }
    # the attention kernel alone (profile mode 4: its split-merge kernel untimed), per block
    kern_ms = sub[4]["attention"][0] / (extra_steps * cfg.layers)
    if kern_ms > 0:
        line["roofline"]["kernel_only"] = {
            "avg_launch_ms": kern_ms, "achieved": attn_flop / (kern_ms * 1e-3) / 1e12,
            "frac": attn_flop / (kern_ms * 1e-3) / 1e12 / bf16_peak,
            "merge_kernel_ms": max(per_block_ms - kern_ms, 0.0),
            "note": "the attention kernel's own launch window (20-step sub-run, profile mode 4); the headline "
                    "avg_launch_ms / frac above also count the split-merge kernel that follows it"}
    gemm_ms = max(sub[3]["gemm"][0] / extra_steps, 1e-9)    # GEMMs' own device time (profile mode 3 sub-run)
    line["device_time_ms_per_step"] = {"attention": attn_ms / args.steps, "gemm": gemm_ms,
                                       "other": total_ms / args.steps - attn_ms / args.steps - gemm_ms,
                                       "gemm_source": "self-timed in a separate 20-step sub-run (profile mode 3)"}
    # patch kernels: their own device time inside the step graph (profile mode 3 self-timing,
    # the fixed 7x7 / stride-3 kernels) when every patch launch of the step was timed, else the
    # CUDA events around eager launches (mode 2: includes each launch's ramp without overlap)
    n_patch = 2 + (2 * cfg.layers if cfg.ffn_kind == 1 else 0)
    if os.environ.get("VI_PATCH_TIME_ONLY"):   # one patch kernel kind self-timed (engine.cu patch_timing)
        print(f"patch kind {os.environ['VI_PATCH_TIME_ONLY']}: {sub[3]['patch'][0] / extra_steps:.4f} ms/step "
              f"({sub[3]['patch'][1] / extra_steps:.0f} launches)", file=sys.stderr)
    self_timed = sub[3]["patch"][1] == n_patch * extra_steps
    patch_ms = max((sub[3] if self_timed else sub[2])["patch"][0] / extra_steps, 1e-9)
    patch_ms_events = sub[2]["patch"][0] / extra_steps
    gflop, pbytes = gemm_flop_per_step(cfg) / (world if args.tp else 1), patch_bytes_per_step(cfg)
    line["secondary_rooflines"] = {
        "gemms (embed, QKV, O, FFN1, FFN2, back; self-timed in the graph)": {
            "bound": "tensor", "achieved": gflop / (gemm_ms * 1e-3) / 1e12, "peak": bf16_peak, "unit": "TFLOP/s",
            "frac": gflop / (gemm_ms * 1e-3) / 1e12 / bf16_peak, "flop_per_step": gflop, "ms_per_step": gemm_ms},
        "patch kernels (soft split, F3N fold/unfold, soft composite)": {
            "bound": "hbm", "achieved": pbytes / (patch_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": pbytes / (patch_ms * 1e-3) / 1e9 / hbm_peak, "bytes_per_step": pbytes,
            "bytes": "algorithmic (SURVEY §8(d): bf16 intermediates)", "ms_per_step": patch_ms,
            "implementation_bytes_per_step": patch_bytes_implementation(cfg),
            "implementation_frac": patch_bytes_implementation(cfg) / (patch_ms * 1e-3) / 1e9 / hbm_peak,
            "timing": ("kernel self-timing inside the step graph" if self_timed
                       else "CUDA events around eager launches"),
            "ms_per_step_eager_events": patch_ms_events}}
    line["deterministic"] = deterministic
    if os.environ.get("VI_PROFILE_MODE") == "2":
        line["profile_ms_per_step"] = {k: v[0] / args.steps for k, v in prof.items()}
        line["profile_launches_per_step"] = {k: v[1] / args.steps for k, v in prof.items()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tp", action="store_true",
                    help="one stream with its heads sharded over the N ranks (NCCL all-gather per block)")
    args = ap.parse_args()
    if os.environ.get("VI_BENCH_WATCHDOG"):   # debugging: dump every thread's stack, then exit
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["VI_BENCH_WATCHDOG"]), exit=True)
    from vi_synth import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
