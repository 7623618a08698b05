"""Where does the bf16 path's error come from?  One block, first step (no memory): compare the
GPU's stored tensors (h, Q, K, V, O through vi_debug_read) with the bf16-storage emulation, and
the GPU's attention output with fp64 attention recomputed from the GPU's OWN Q, K, V (isolates
the attention kernel's arithmetic: P in bf16, exp2 approximations, fp32 accumulation).

    python tools/parity_diag.py [variant ...]        (GPU; test infrastructure: uses oracle/)
"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import vi_oracle as O  # noqa: E402
from vi_synth import CONFIGS, make_features, make_weights  # noqa: E402
import gpu_harness  # noqa: E402


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def attn64(Q, K, V, H):
    return O.attention(Q, K, V, H)


def main(variants):
    for variant in variants:
        for cname, layers, steps in (("C3S", 1, 1), ("C3S", 1, 3)):
            cfg = CONFIGS[cname].replace(layers=layers)
            w = make_weights(cfg, seed=1, variant=variant)
            g = gpu_harness.GpuStream(cfg, w)
            e = O.emulate_bf16_storage(cfg, w)
            o = O.OracleStream(cfg, w)
            n = cfg.t_new
            for i in range(steps):
                feats = make_features(cfg, n, first_frame=i * n, seed=1)
                e.push(n); o.push(n)
                _, est = e.step(feats)
                _, ost = o.step(feats)
                _, gst = g.step(feats)
            rows = n * cfg.tokens
            h = torch.empty(rows, cfg.d_model, dtype=torch.bfloat16, device="cuda")
            g.ctx.debug_read("h", h)   # after the step: LN2 output of the last block (h buffer reused)
            el, ol, gl = est["layers"][-1], ost["layers"][-1], gst["layers"][-1]
            gq = host(gl["q"])
            # K/V of the chunk's frames and of the memory frames, in slot order = temporal here
            ks, vs = [], []
            for fid in e.mem.window() + list(range(e.mem.cur_first, e.mem.next_id)):
                k_, v_ = g.kv(layers - 1, fid % g.ctx.S)
                ks.append(host(k_)); vs.append(host(v_))
            gk, gv = np.concatenate(ks), np.concatenate(vs)
            ek = np.concatenate([e.frame_kv(layers - 1, f)[0] for f in e.mem.window() + list(range(e.mem.cur_first, e.mem.next_id))])
            go = host(gl["o"])
            o_from_gpu_qkv = attn64(gq, gk, gv, cfg.heads)
            print(f"[{variant} {cname} steps={steps}] q: gpu vs emu {O.rel_err(gq, el['q']):.2e} "
                  f"(differing elements {np.count_nonzero(gq != el['q'])}/{gq.size}); k: gpu vs emu {O.rel_err(gk, ek):.2e}")
            print(f"   o: gpu vs fp64(gpu q,k,v) {O.rel_err(go, o_from_gpu_qkv):.3e} | gpu vs emu {O.rel_err(go, el['o'], den_ref=ol['o']):.3e}"
                  f" | emu vs oracle {O.rel_err(el['o'], ol['o']):.3e} | gpu vs oracle {O.rel_err(go, ol['o']):.3e}")
            print(f"   fp64(gpu q,k,v) vs emu o {O.rel_err(o_from_gpu_qkv, el['o'], den_ref=ol['o']):.3e}; "
                  f"x: gpu vs emu {O.rel_err(host(gst['x']), est['x'], den_ref=ost['x']):.3e}")
            g.ctx.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["paper", "sensitive", "sharp"])
