"""Helpers for the GPU parity tests: drive a libvi context step by step through the C-ABI
and collect the same stage tensors the oracle reports."""
from __future__ import annotations

import numpy as np
import torch

from vi_synth import make_features


def tdev(a: np.ndarray, dtype: str) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    return (t.to(torch.bfloat16) if dtype == "bf16" else t).cuda()


def host(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64)


def tdtype(cfg):
    return torch.bfloat16 if cfg.dtype == "bf16" else torch.float32


class GpuStream:
    """A vi_ctx fed the same per-step inputs as oracle.OracleStream."""

    def __init__(self, cfg, weights, max_new_frames=None):
        from paper_2403_16161_b200 import vi
        self.vi = vi
        self.cfg = cfg
        self.ctx = vi.Context.from_synth(cfg, max_new_frames=max_new_frames)
        self.ctx.set_weights(weights)
        T = max_new_frames or cfg.t_new
        self.x = torch.zeros(T * cfg.tokens, cfg.d_model, dtype=torch.float32, device="cuda")

    def step(self, feats: np.ndarray, stages: bool = True):
        cfg, ctx = self.cfg, self.ctx
        n = feats.shape[0]
        first, ev = ctx.push(n)
        f = tdev(feats, cfg.dtype)
        x = self.x[: n * cfg.tokens]
        dt = tdtype(cfg)
        st = {"first": first, "evicted": ev, "layers": []}
        if stages:
            tok = torch.empty(n, cfg.tokens, cfg.patch_dim, dtype=dt, device="cuda")
            ctx.soft_split(f, n, tok, 0)
            st["tp"] = tok
        ctx.soft_split(f, n, x, 1)
        if stages:
            ctx.sync()
            st["x0"] = x.clone()
        for l in range(cfg.layers):
            ctx.memory_step(l, x, x)
            if stages:
                d = {}
                names = [("o", cfg.d_model, dt), ("g", cfg.ffn_hidden, dt)]
                if not getattr(cfg, "win_h", 0):      # Q is window-major under window attention
                    names.append(("q", cfg.d_model, dt))
                if cfg.ffn_kind == 1:
                    names.append(("u", cfg.ffn_hidden, torch.float32))
                for name, width, bdt in names:
                    buf = torch.empty(n * cfg.tokens, width, dtype=bdt, device="cuda")
                    ctx.debug_read(name, buf)
                    d[name] = buf
                ctx.sync()
                d["x"] = x.clone()
                st["layers"].append(d)
        out = torch.empty(n, cfg.feat_h, cfg.feat_w, cfg.feat_c, dtype=dt, device="cuda")
        ctx.soft_composite(x, n, out, 1)
        ctx.sync()
        st["x"] = x.clone()
        st["out"] = out
        return out, st

    def kv(self, layer: int, slot: int):
        dt = tdtype(self.cfg)
        k = torch.empty(self.cfg.tokens, self.cfg.d_model, dtype=dt, device="cuda")
        v = torch.empty_like(k)
        self.ctx.debug_read("k", k, layer, slot)
        self.ctx.debug_read("v", v, layer, slot)
        return k, v
