"""Dump the patch kernels' outputs of one C3 (or C3S) memory step, for the bitwise A/B of
the unfold variants (VI_PATCH_V=0: per-vector gathers; 1, the default: one warp per token).  usage: VI_PATCH_V=<v> python tools/patch_dump.py <config> <out.npz>

Saves the soft split tokens, the F3N hidden g of every block and the soft composite output of
two steps as raw bit patterns (uint16 for bf16 / uint32 for fp32)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch

from gpu_harness import GpuStream
from vi_synth import CONFIGS, make_features, make_weights


def bits(t: torch.Tensor) -> np.ndarray:
    t = t.contiguous()
    return (t.view(torch.int16) if t.dtype == torch.bfloat16 else t.view(torch.int32)).cpu().numpy()


def main():
    cfg = CONFIGS[sys.argv[1]]
    s = GpuStream(cfg, make_weights(cfg, seed=1))
    out = {}
    for step in range(2):
        feats = make_features(cfg, cfg.t_new, first_frame=step * cfg.t_new, seed=5)
        y, st = s.step(feats, stages=True)
        out[f"s{step}_tp"] = bits(st["tp"])
        out[f"s{step}_out"] = bits(y)
        for l, d in enumerate(st["layers"]):
            out[f"s{step}_l{l}_g"] = bits(d["g"])
            out[f"s{step}_l{l}_x"] = bits(d["x"])
    np.savez(sys.argv[2], **out)


if __name__ == "__main__":
    main()
