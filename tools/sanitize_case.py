"""Small end-to-end runs for compute-sanitizer: BASELINE configs[0] (C1,
fp32 SIMT path, 4 steps wrapping the ring) and a reduced FuseFormer-shaped case (C3S, bf16
tensor-core path: embed / QKV / stream-K or KV-split attention / F3N / composite GEMMs and
patch kernels, 3 steps) and one block of the C3 shape (the persistent stream-K attention with its
split-unit merges), each with a refine commit; steps replay captured CUDA graphs.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2403_16161_b200 import vi
    from vi_synth import CONFIGS, make_features, make_kv, make_weights
    torch.cuda.set_device(0)
    cases = (("C1", CONFIGS["C1"]), ("C3S", CONFIGS["C3S"].replace(layers=1)), ("C3", CONFIGS["C3"].replace(layers=1)))
    only = sys.argv[1:]
    for name, cfg in cases:
        if only and name not in only:
            continue
        ctx = vi.Context.from_synth(cfg)
        ctx.set_weights(make_weights(cfg, seed=0, variant="sensitive"))
        dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
        for i in range(4 if name == "C1" else 3):
            f = torch.from_numpy(make_features(cfg, cfg.t_new, first_frame=i * cfg.t_new, seed=0)).to(dt).cuda()
            out = torch.empty_like(f)
            ctx.run_step(f, cfg.t_new, out)
            if i == 1:
                k, v = make_kv(cfg, 1, 0)
                kk, vv = (torch.from_numpy(a).to(dt).contiguous() for a in (k, v))
                ctx.commit(0, kk, vv)
        ctx.sync()
        print(f"{name}: ok, out mean {out.float().abs().mean().item():.4f}", flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
