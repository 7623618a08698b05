"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no split, projection, attention,
normalisation or composite).  It only draws random numbers and rounds them to the
storage precision of the path under test, so that both sides of a parity check
start from bit-identical inputs.  Neither ``oracle/`` nor the CUDA package import
each other; both may import this module.

Workload recipe: the paper measures on DAVIS / YouTube-VOS
at an unstated resolution (§4.1 "Settings").  No dataset is in
the container, so frames are replaced by feature maps shaped like a 432x240 video after
the backbones' 4x down-sampling (60x108 cells), drawn ~N(0,1); pretrained weights
("we reuse the weights of the pre-trained models") are replaced by seeded
N(0, 0.02) weights (BASELINE.json configs).  Masks (X = Y (1-M)) enter only the
out-of-scope CNN encoder; where a config asks for them they zero the features under a
random rectangle covering 10-30% of the frame, down-sampled 4x.
"""
from __future__ import annotations

import dataclasses
import zlib
from typing import Dict, Optional

import numpy as np

__all__ = ["Config", "CONFIGS", "rng_for", "round_bf16", "make_weights", "make_features",
           "make_kv", "WEIGHT_NAMES"]


@dataclasses.dataclass(frozen=True)
class Config:
    """Shape of one memory-step workload (BASELINE.json ``configs``)."""
    name: str
    layers: int
    heads: int
    d_model: int
    ffn_hidden: int
    ffn_kind: int          # 0 = MLP (GELU), 1 = F3N (fold/unfold inside the FFN)
    feat_h: int
    feat_w: int
    feat_c: int
    kh: int
    kw: int
    sh: int
    sw: int
    ph: int
    pw: int
    t_new: int             # frames per memory step (T)
    mem_frames: int        # M, the memory span s of Eq. 3
    dtype: str             # "bf16" (tensor-core path) or "fp32" (SIMT path)
    pos_embed: int = 0
    ref_rate: int = 0      # r of Eq. 3's reference frames M_{1,r} (0 = span only)
    max_refs: int = 0      # reference slots kept (the oldest reference leaves first)
    win_h: int = 0         # window attention: win_h x win_w token windows (0 = global attention)
    win_w: int = 0
    refined_mem: int = 0   # Eq. 4's refined memory M-bar (0 = off)
    refined_span: int = 0  # s' of Eq. 4 (refined frames t-s'..t)
    refined_rate: int = 0  # r' of Eq. 4 (refined reference frames, 0 = none)
    max_refined_refs: int = 0

    @property
    def oh(self) -> int:
        return (self.feat_h + 2 * self.ph - self.kh) // self.sh + 1

    @property
    def ow(self) -> int:
        return (self.feat_w + 2 * self.pw - self.kw) // self.sw + 1

    @property
    def tokens(self) -> int:
        return self.oh * self.ow

    @property
    def patch_dim(self) -> int:
        return self.kh * self.kw * self.feat_c

    @property
    def head_dim(self) -> int:
        return self.d_model // self.heads

    @property
    def slots(self) -> int:
        return (self.mem_frames + self.t_new + (self.max_refs if self.ref_rate > 0 else 0) +
                ((self.refined_span + 1 + (self.max_refined_refs if self.refined_rate > 0 else 0))
                 if self.refined_mem else 0))

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS: Dict[str, Config] = {
    # BASELINE.json configs[0]: tiny fp32 oracle check (24 tokens/frame, 1 new + 3 memory frames)
    "C1": Config("C1", 1, 2, 64, 128, 0, 12, 18, 16, 7, 7, 3, 3, 3, 3, 1, 3, "fp32"),
    # configs[1]: STTN-shaped, non-overlapping 5x9-cell patches -> 12x12 = 144 tokens
    "C2": Config("C2", 8, 4, 256, 1024, 0, 60, 108, 256, 5, 9, 5, 9, 0, 0, 5, 10, "bf16"),
    # configs[2]: FuseFormer-shaped, the metric config (720 tokens/frame, F3N 1960 = 49 x 40)
    "C3": Config("C3", 8, 4, 512, 1960, 1, 60, 108, 128, 7, 7, 3, 3, 3, 3, 5, 10, "bf16"),
    # C3 in the paper's strict Eq. 3 mode: one new frame per step (also C5's online model)
    "C3T1": Config("C3T1", 8, 4, 512, 1960, 1, 60, 108, 128, 7, 7, 3, 3, 3, 3, 1, 10, "bf16"),
    # configs[3]: E2FGVI-shaped, window attention over 5x9-token windows (16 per frame), 16 blocks
    "C4": Config("C4", 16, 4, 512, 1960, 1, 60, 108, 128, 7, 7, 3, 3, 3, 3, 5, 10, "bf16", win_h=5, win_w=9),
    # a reduced C3 that the fp64 oracle finishes in seconds: 2 blocks, 30x54 map -> 10x18=180 tokens
    "C3S": Config("C3S", 2, 4, 512, 1960, 1, 30, 54, 128, 7, 7, 3, 3, 3, 3, 2, 3, "bf16"),
}

WEIGHT_NAMES = ("embed_w", "embed_b", "pos", "ln1_g", "ln1_b", "wqkv", "bqkv", "wo", "bo",
                "ln2_g", "ln2_b", "w1", "b1", "w2", "b2", "back_w", "back_b")


def rng_for(seed: int, tag: str) -> np.random.Generator:
    """Independent, reproducible stream per (seed, tensor tag)."""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(zlib.crc32(tag.encode()),)))


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returned as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32).copy()
    nan = np.isnan(a)
    out[nan] = np.nan
    return out


def _normal(seed: int, tag: str, shape, std: float) -> np.ndarray:
    return (rng_for(seed, tag).standard_normal(shape) * std).astype(np.float32)


def make_weights(cfg: Config, seed: int = 0, variant: str = "paper") -> Dict[str, np.ndarray]:
    """Seeded weights in nn.Linear layout ([out, in]), float32.

    variant "paper": every matrix and bias ~N(0, 0.02) (BASELINE.json configs);
    LN gains 1 + N(0, 0.02), LN shifts N(0, 0.02).
    variant "sensitive": matrices ~N(0, 1/fan_in) so that attention logits have std ~1
    and the memory measurably changes the output (SURVEY §8(c) parity protocol 3).
    variant "sharp": like "sensitive" but Wq scaled x5 (logits std >> 1: exercises
    the online-softmax rescaling).
    Matrices are rounded to bf16 for the bf16 path (the GPU stores them in bf16);
    biases and LN parameters stay fp32 (the GPU keeps them in fp32).
    """
    L, D, F, Pd, P = cfg.layers, cfg.d_model, cfg.ffn_hidden, cfg.patch_dim, cfg.tokens

    def mat(tag, shape, fan_in):
        std = 0.02 if variant == "paper" else 1.0 / np.sqrt(fan_in)
        w = _normal(seed, tag, shape, std)
        if variant == "sharp" and tag == "wqkv":
            w[:, :D, :] *= 5.0
        return round_bf16(w) if cfg.dtype == "bf16" else w

    def vec(tag, shape, base=0.0):
        return (base + _normal(seed, tag, shape, 0.02)).astype(np.float32)

    w = {
        "embed_w": mat("embed_w", (D, Pd), Pd),
        "embed_b": vec("embed_b", (D,)),
        "pos": (_normal(seed, "pos", (P, D), 0.02) if cfg.pos_embed else None),
        "ln1_g": vec("ln1_g", (L, D), 1.0),
        "ln1_b": vec("ln1_b", (L, D)),
        "wqkv": mat("wqkv", (L, 3 * D, D), D),
        "bqkv": vec("bqkv", (L, 3 * D)),
        "wo": mat("wo", (L, D, D), D),
        "bo": vec("bo", (L, D)),
        "ln2_g": vec("ln2_g", (L, D), 1.0),
        "ln2_b": vec("ln2_b", (L, D)),
        "w1": mat("w1", (L, F, D), D),
        "b1": vec("b1", (L, F)),
        "w2": mat("w2", (L, D, F), F),
        "b2": vec("b2", (L, D)),
        "back_w": mat("back_w", (Pd, D), D),
        "back_b": vec("back_b", (Pd,)),
    }
    return w


def _rect_mask(rng: np.random.Generator, h: int, w: int) -> np.ndarray:
    """A random rectangle covering 10-30% of an h x w grid, aspect U(0.5, 2)."""
    area = rng.uniform(0.10, 0.30) * h * w
    aspect = rng.uniform(0.5, 2.0)
    rh = int(min(h, max(1, round(np.sqrt(area / aspect)))))
    rw = int(min(w, max(1, round(area / rh))))
    y0 = int(rng.integers(0, h - rh + 1))
    x0 = int(rng.integers(0, w - rw + 1))
    m = np.zeros((h, w), dtype=bool)
    m[y0:y0 + rh, x0:x0 + rw] = True
    return m


def _moving_rect_mask(seed: int, fid: int, h: int, w: int) -> np.ndarray:
    """One rectangle per stream (10-30% of the grid, aspect U(0.5, 2)) moving with a constant
    velocity and reflecting at the borders (object-removal style masks)."""
    rng = rng_for(seed, "moving-mask")
    area = rng.uniform(0.10, 0.30) * h * w
    aspect = rng.uniform(0.5, 2.0)
    rh = int(min(h, max(1, round(np.sqrt(area / aspect)))))
    rw = int(min(w, max(1, round(area / rh))))
    y0, x0 = rng.uniform(0, h - rh), rng.uniform(0, w - rw)
    vy, vx = rng.uniform(-1.5, 1.5), rng.uniform(-1.5, 1.5)

    def reflect(p, span):
        if span <= 0:
            return 0
        q = p % (2 * span)
        return int(round(q if q <= span else 2 * span - q))
    y, x = reflect(y0 + vy * fid, h - rh), reflect(x0 + vx * fid, w - rw)
    m = np.zeros((h, w), dtype=bool)
    m[y:y + rh, x:x + rw] = True
    return m


def make_features(cfg: Config, n_frames: int, first_frame: int = 0, seed: int = 0,
                  masked=False) -> np.ndarray:
    """Feature maps [n, H, W, C] (channels-last) ~N(0,1), one independent draw per frame id.

    With ``masked`` the cells under a random 10-30% rectangle are zeroed (a stand-in for
    the encoder seeing X = Y (1-M)); ``masked="moving"``: one rectangle per stream
    moving across the frames with reflecting borders.
    """
    out = np.empty((n_frames, cfg.feat_h, cfg.feat_w, cfg.feat_c), dtype=np.float32)
    for i in range(n_frames):
        fid = first_frame + i
        out[i] = _normal(seed, f"feat{fid}", (cfg.feat_h, cfg.feat_w, cfg.feat_c), 1.0)
        if masked == "moving":
            out[i][_moving_rect_mask(seed, fid, cfg.feat_h, cfg.feat_w)] = 0.0
        elif masked:
            m = _rect_mask(rng_for(seed, f"mask{fid}"), cfg.feat_h, cfg.feat_w)
            out[i][m] = 0.0
    return round_bf16(out) if cfg.dtype == "bf16" else out


def make_kv(cfg: Config, seed: int, frame_id: int, scale: float = 1.0):
    """Arbitrary per-layer K/V rows [L, P, D] for one frame (refine-commit payloads)."""
    shape = (cfg.layers, cfg.tokens, cfg.d_model)
    k = _normal(seed, f"k{frame_id}", shape, scale)
    v = _normal(seed, f"v{frame_id}", shape, scale)
    if cfg.dtype == "bf16":
        k, v = round_bf16(k), round_bf16(v)
    return k, v
