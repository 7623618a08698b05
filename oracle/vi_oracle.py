"""fp64 CPU oracle of the memory step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  It shares no code with the CUDA
path (``paper_2403_16161_b200``) and never receives a value produced by it.

It is a plain, slow, obviously-correct restatement of what the paper's "Memory" model
(§3.4, Eq. 3) computes, with the readings listed in DESIGN.md
("Readings of the paper").  Citations: ``P:n`` = /root/reference/PAPER.md line n.

Structure (deliberately different from the GPU path):
  * the memory caches each frame's *block input representation* per transformer
    block, exactly as the paper describes ("save in memory the successive outputs of
    these transformers for each predicted frame"; "each frame is saved in the
    memory as much times as there are transformers", P:99 / Fig. 2 caption) and
    re-projects K/V from it every step; the GPU caches projected K/V instead;
  * attention is computed per head with explicit score and probability matrices over
    keys in temporal (frame-id) order; the GPU walks the ring-buffer slot order;
  * everything is float64; inputs are whatever the caller passes (the bf16 path's
    tests pass bf16-representable values, see vi_synth.round_bf16).

Pinned by tests/test_oracle_*.py (torch library routines, closed forms, SPEC worked
examples, the memory-equivalence invariants I1/I2 and brute force).  Every function
here has at least one pin; none is "parity unpinned".
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
from scipy.special import erf

# status codes of the C-ABI (include/vi.h), restated here for the bookkeeping model
VI_OK = 0
VI_NOT_RESIDENT = 1
VI_E_ARG = -1
VI_E_PROTOCOL = -4

LN_EPS = 1e-5  # SURVEY Q1 / SPEC S:61


# ----------------------------------------------------------------------------------
# Patch geometry: soft split / soft composite (FuseFormer overlapping patches)
# P:53 "the idea of having the patches overlapping"; "cut into patches";
# P:166 FuseFormer patches "blended together".  Reading Q6: nn.Unfold semantics
# (symmetric zero padding), patch vector ordered (ky, kx, c), tokens row-major (oy, ox).
# ----------------------------------------------------------------------------------

def out_size(n: int, k: int, s: int, p: int) -> int:
    """Number of window positions along one side: (n + 2p - k) // s + 1."""
    return (n + 2 * p - k) // s + 1


def soft_split(F: np.ndarray, kh: int, kw: int, sh: int, sw: int, ph: int, pw: int) -> np.ndarray:
    """Overlapping unfold of channels-last maps F[T,H,W,C] -> tokens [T, oh*ow, kh*kw*C].

    Tp[t, oy*ow+ox, (ky*kw+kx)*C + c] = F[t, oy*sh-ph+ky, ox*sw-pw+kx, c], 0 outside.
    """
    F = np.asarray(F, dtype=np.float64)
    T, H, W, C = F.shape
    oh, ow = out_size(H, kh, sh, ph), out_size(W, kw, sw, pw)
    out = np.zeros((T, oh * ow, kh * kw * C), dtype=np.float64)
    for oy in range(oh):
        for ox in range(ow):
            tok = oy * ow + ox
            for ky in range(kh):
                y = oy * sh - ph + ky
                if y < 0 or y >= H:
                    continue
                for kx in range(kw):
                    x = ox * sw - pw + kx
                    if x < 0 or x >= W:
                        continue
                    j = (ky * kw + kx) * C
                    out[:, tok, j:j + C] = F[:, y, x, :]
    return out


def coverage(H: int, W: int, kh: int, kw: int, sh: int, sw: int, ph: int, pw: int) -> np.ndarray:
    """How many (token, ky, kx) windows cover each cell: the composite's divisor."""
    oh, ow = out_size(H, kh, sh, ph), out_size(W, kw, sw, pw)
    cnt = np.zeros((H, W), dtype=np.int64)
    for oy in range(oh):
        for ox in range(ow):
            for ky in range(kh):
                y = oy * sh - ph + ky
                if y < 0 or y >= H:
                    continue
                for kx in range(kw):
                    x = ox * sw - pw + kx
                    if 0 <= x < W:
                        cnt[y, x] += 1
    return cnt


def soft_composite(Yp: np.ndarray, H: int, W: int, C: int, kh: int, kw: int, sh: int, sw: int,
                   ph: int, pw: int) -> np.ndarray:
    """Overlap-add of patch vectors back onto the map, divided by the cover count.

    out[t,y,x,c] = (sum over (tok,ky,kx) landing on (y,x) of Yp[t,tok,(ky*kw+kx)*C+c]) / cnt[y,x].
    Padding positions are discarded.  A cell no window covers is a configuration error.
    """
    Yp = np.asarray(Yp, dtype=np.float64)
    T = Yp.shape[0]
    oh, ow = out_size(H, kh, sh, ph), out_size(W, kw, sw, pw)
    assert Yp.shape[1] == oh * ow and Yp.shape[2] == kh * kw * C, Yp.shape
    acc = np.zeros((T, H, W, C), dtype=np.float64)
    cnt = np.zeros((H, W), dtype=np.int64)
    for oy in range(oh):
        for ox in range(ow):
            tok = oy * ow + ox
            for ky in range(kh):
                y = oy * sh - ph + ky
                if y < 0 or y >= H:
                    continue
                for kx in range(kw):
                    x = ox * sw - pw + kx
                    if x < 0 or x >= W:
                        continue
                    j = (ky * kw + kx) * C
                    acc[:, y, x, :] += Yp[:, tok, j:j + C]
                    cnt[y, x] += 1
    if (cnt == 0).any():
        raise ValueError("soft_composite: a cell is covered by no window (config error)")
    return acc / cnt[None, :, :, None]


# ----------------------------------------------------------------------------------
# Transformer block pieces ("same general pipeline as the original vision
# transformer"; readings Q1-Q5: pre-norm, biases, 1/sqrt(d) scale, exact-erf GELU,
# FuseFormer Fusion-FFN = FFN1 -> fold/count -> unfold -> GELU -> FFN2).
# ----------------------------------------------------------------------------------

def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float = LN_EPS) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * np.asarray(g, np.float64) + np.asarray(b, np.float64)


def gelu(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def linear(x: np.ndarray, w: np.ndarray, b: Optional[np.ndarray]) -> np.ndarray:
    """nn.Linear convention: y = x W^T + b, W stored [out, in]."""
    y = np.asarray(x, np.float64) @ np.asarray(w, np.float64).T
    if b is not None:
        y = y + np.asarray(b, np.float64)
    return y


def softmax_rows(S: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction."""
    S = np.asarray(S, dtype=np.float64)
    E = np.exp(S - S.max(axis=-1, keepdims=True))
    return E / E.sum(axis=-1, keepdims=True)


def attention(Q: np.ndarray, K: np.ndarray, V: np.ndarray, heads: int,
              allowed: Optional[np.ndarray] = None, row_chunk: int = 1024,
              return_lse: bool = False):
    """Multi-head softmax(Q_h K_h^T / sqrt(d)) V_h, one explicit head at a time.

    Q [nq, D], K/V [nk, D]; ``allowed`` optional boolean [nq, nk] (True = key visible).
    Returns O [nq, D] (and lse [heads, nq] = log sum exp of the scaled scores).
    P:121 "the query vector ... only contain patches from this last frame", "the key and
    value vectors must still represent all the frames selected".
    """
    Q = np.asarray(Q, np.float64); K = np.asarray(K, np.float64); V = np.asarray(V, np.float64)
    nq, D = Q.shape
    d = D // heads
    O = np.zeros((nq, D), dtype=np.float64)
    lse = np.zeros((heads, nq), dtype=np.float64)
    scale = 1.0 / math.sqrt(d)
    for h in range(heads):
        cols = slice(h * d, (h + 1) * d)
        kh, vh = K[:, cols], V[:, cols]
        for r0 in range(0, nq, row_chunk):
            r1 = min(nq, r0 + row_chunk)
            S = (Q[r0:r1, cols] @ kh.T) * scale
            if allowed is not None:
                S = np.where(allowed[r0:r1], S, -np.inf)
            m = S.max(axis=-1, keepdims=True)
            E = np.exp(S - m)
            l = E.sum(axis=-1, keepdims=True)
            O[r0:r1, cols] = (E / l) @ vh
            lse[h, r0:r1] = (m + np.log(l))[:, 0]
    return (O, lse) if return_lse else O


def f3n_mix(u: np.ndarray, cfg) -> np.ndarray:
    """FuseFormer Fusion-FFN hidden mixing (reading Q5): per frame, view the hidden
    vector of each token as (ky, kx, c) with c = F / (kh*kw), fold onto the feature map
    with overlap-count normalisation, then unfold again with the same geometry."""
    T = u.shape[0]
    F = u.shape[-1]
    cf = F // (cfg.kh * cfg.kw)
    assert cf * cfg.kh * cfg.kw == F
    g = (cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
    folded = soft_composite(u.reshape(T, -1, F), cfg.feat_h, cfg.feat_w, cf, *g)
    return soft_split(folded, *g)


def ffn(h2: np.ndarray, w: Dict[str, np.ndarray], l: int, cfg, n_frames: int,
        store=None) -> Tuple[np.ndarray, np.ndarray]:
    """FFN of block l on LN2 output h2 [n*P, D]; returns (u, g) and the caller adds W2.
    (``store``: the emulation's rounding of the stored hidden g, see ``qkv``.)"""
    u = linear(h2, w["w1"][l], w["b1"][l])
    if cfg.ffn_kind == 1:
        g = gelu(f3n_mix(u.reshape(n_frames, cfg.tokens, -1), cfg).reshape(u.shape))
    else:
        g = gelu(u)
    return u, _st(store, g)


def embed(feats: np.ndarray, w: Dict[str, np.ndarray], cfg) -> Tuple[np.ndarray, np.ndarray]:
    """Soft split + patch embedding: X0 = SoftSplit(F) We^T + be (+ pos)."""
    Tp = soft_split(feats, cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
    n = Tp.shape[0]
    X = linear(Tp.reshape(n * cfg.tokens, -1), w["embed_w"], w["embed_b"])
    if w.get("pos") is not None:
        X = X + np.tile(np.asarray(w["pos"], np.float64), (n, 1))
    return Tp, X


def compose(X: np.ndarray, w: Dict[str, np.ndarray], cfg, n_frames: int) -> Tuple[np.ndarray, np.ndarray]:
    """Back-projection + soft composite to the feature map [n, H, W, C]."""
    Yp = linear(X, w["back_w"], w["back_b"]).reshape(n_frames, cfg.tokens, -1)
    out = soft_composite(Yp, cfg.feat_h, cfg.feat_w, cfg.feat_c,
                         cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
    return Yp, out


def _st(store, a):
    return a if store is None else store(a)


def qkv(x: np.ndarray, w, l: int, cfg, store=None):
    """LN1 and the Q/K/V projection of block l.  ``store`` (default None: plain fp64) is a
    storage-rounding function applied where the bf16 design stores a tensor (here the LN1
    output h and Q, K, V) -- the bf16-storage EMULATION used only to derive logit-scaled
    tolerance bars (see ``emulate_bf16_storage``); never the oracle itself."""
    h = _st(store, layer_norm(x, w["ln1_g"][l], w["ln1_b"][l]))
    D = cfg.d_model
    y = linear(h, w["wqkv"][l], w["bqkv"][l])
    Q, K, V = y[:, :D], y[:, D:2 * D], y[:, 2 * D:]
    if store is not None:
        Q, K, V = store(Q), store(K), store(V)
    return h, Q, K, V


# ----------------------------------------------------------------------------------
# One transformer block of the Memory model (Eq. 3): queries = the new frames only,
# keys/values = memory frames (span s) + the new frames.
# ----------------------------------------------------------------------------------

def token_windows(cfg) -> Optional[np.ndarray]:
    """Window id of every token of a frame for window attention (E2FGVI-style, BASELINE
    configs[3]: non-overlapping win_h x win_w token windows on the oh x ow token grid, row-major
    window order), or None for global attention (cfg.win_h = 0)."""
    wh, ww = getattr(cfg, "win_h", 0), getattr(cfg, "win_w", 0)
    if not wh:
        return None
    oy, ox = np.divmod(np.arange(cfg.tokens), cfg.ow)
    return (oy // wh) * (cfg.ow // ww) + (ox // ww)


def block_memory(x: np.ndarray, mem_kv: Sequence[Tuple[np.ndarray, np.ndarray]], w, l: int, cfg,
                 n_frames: int, chunk_causal: bool = False, store=None) -> Tuple[np.ndarray, Dict[str, np.ndarray]]:
    """x [n*P, D] = block-l input of the chunk; mem_kv = [(K_j, V_j)] in frame-id order.
    With window attention (cfg.win_h > 0) a query sees only the keys of its own token window,
    in every frame of the memory and the chunk."""
    P = cfg.tokens
    h1, Q, Kc, Vc = qkv(x, w, l, cfg, store)
    K = np.concatenate([k for k, _ in mem_kv] + [Kc], axis=0)
    V = np.concatenate([v for _, v in mem_kv] + [Vc], axis=0)
    allowed = None
    if chunk_causal and n_frames > 1:
        nm = len(mem_kv) * P
        qf = np.repeat(np.arange(n_frames), P)
        kf = np.concatenate([np.full(nm, -1), np.repeat(np.arange(n_frames), P)])
        allowed = kf[None, :] <= qf[:, None]
    win = token_windows(cfg)
    if win is not None:
        wq = np.tile(win, n_frames)
        wk = np.tile(win, len(mem_kv) + n_frames)
        same = wq[:, None] == wk[None, :]
        allowed = same if allowed is None else (allowed & same)
    O, lse = attention(Q, K, V, cfg.heads, allowed=allowed, return_lse=True)
    O = _st(store, O)
    xa = x + linear(O, w["wo"][l], w["bo"][l])
    h2 = _st(store, layer_norm(xa, w["ln2_g"][l], w["ln2_b"][l]))
    u, g = ffn(h2, w, l, cfg, n_frames, store)
    xo = xa + linear(g, w["w2"][l], w["b2"][l])
    st = dict(h1=h1, q=Q, k=Kc, v=Vc, o=O, lse=lse, x_attn=xa, h2=h2, u=u, g=g, x=xo)
    return xo, st


def joint_forward(feats: np.ndarray, w, cfg, mode: str = "causal",
                  frame_mask: Optional[np.ndarray] = None) -> Dict[str, object]:
    """Eq. 1/2-style joint pass over a window of frames, all predicted together.

    mode "causal": frame i's queries see frames j <= i (frame-level block-causal mask);
    mode "full": bidirectional (the offline/refiner window of Eq. 1);
    mode "mask": frame i's queries see the frames j with frame_mask[i, j] (boolean [n, n]).
    Returns per-layer K/V [L][n, P, D] and the composite output [n, H, W, C].
    """
    n = feats.shape[0]
    P, D = cfg.tokens, cfg.d_model
    Tp, X = embed(feats, w, cfg)
    fr = np.repeat(np.arange(n), P)
    if mode == "mask":
        allowed = np.asarray(frame_mask, bool)[fr[:, None], fr[None, :]]
    else:
        allowed = (fr[None, :] <= fr[:, None]) if mode == "causal" else None
    ks, vs, xs = [], [], [X]
    for l in range(cfg.layers):
        h1, Q, K, V = qkv(X, w, l, cfg)
        ks.append(K.reshape(n, P, D)); vs.append(V.reshape(n, P, D))
        O = attention(Q, K, V, cfg.heads, allowed=allowed)
        X = X + linear(O, w["wo"][l], w["bo"][l])
        h2 = layer_norm(X, w["ln2_g"][l], w["ln2_b"][l])
        _, g = ffn(h2, w, l, cfg, n)
        X = X + linear(g, w["w2"][l], w["b2"][l])
        xs.append(X)
    Yp, out = compose(X, w, cfg, n)
    return dict(k=ks, v=vs, x=xs, yp=Yp, out=out)


# ----------------------------------------------------------------------------------
# The memory itself (set model).  Reading Q11: the memory of Eq. 3 keeps frames
# f-s .. f-1 (span s = M); older frames are removed ("removing information
# from ancient frames").  Reading Q13: refined entries (Eq. 4)
# overwrite online ones and are applied at the next frame boundary.
# ----------------------------------------------------------------------------------

class OracleMemory:
    """Resident-set bookkeeping + per-(layer, frame) cache, no arrays of slots (the slot
    numbers of ``state()`` follow the documented mapping, for comparison with the GPU ring).

    Regions (all plain sets of frame ids):
      * online span: the frames f-M .. f-1 of Eq. 3 (span s = M) and the chunk;
      * Eq. 3 references M_{1,r}^{f-1} (reading Q12): multiples of r that left the span, the R
        newest kept;
      * Eq. 4's refined memory M-bar (reading Q22; SPEC select_refined S:467-475):
        refined frames t-s' .. t (refined span; t = the newest frame whose refine commit has
        been applied, the watermark) and the R' newest refined frames with id a multiple of r'
        (refined references), each frame at most once (an online-span frame with a refined
        entry stays there: refined wins)."""

    def __init__(self, mem_frames: int, max_new: int, ref_rate: int = 0, max_refs: int = 0,
                 refined_span: Optional[int] = None, refined_rate: int = 0, max_refined_refs: int = 0):
        self.M = mem_frames
        self.T_max = max_new
        # Eq. 3's reference frames M_{1,r}^{f-1}: multiples of r stay after they
        # leave the span, in R reference slots, the oldest leaving first (DESIGN reading Q12)
        self.r = ref_rate if max_refs > 0 else 0
        self.R = max_refs if ref_rate > 0 else 0
        self.refs: Dict[int, int] = {}     # reference frame id -> its slot (S .. S+R-1)
        # Eq. 4's refined memory (None: off)
        self.refd = refined_span is not None
        self.sr = refined_span if self.refd else 0
        self.rr = refined_rate if (self.refd and max_refined_refs > 0) else 0
        self.RR = max_refined_refs if (self.refd and refined_rate > 0) else 0
        self.t = -1                        # watermark
        self.online: set = set()
        self.rspan: set = set()            # refined span frames (not in the online span)
        self.rrefs: Dict[int, int] = {}    # refined reference id -> its slot
        self.next_id = 0
        self.cur_first = 0     # first id of the chunk pushed last
        self.cur_n = 0
        self.refined: set = set()
        self.pending: Dict[int, object] = {}
        self.stepped = False   # has the chunk pushed last gone through all blocks?

    @property
    def resident(self) -> set:
        return self.online | set(self.refs) | self.rspan | set(self.rrefs)

    def mark_stepped(self):
        self.stepped = True

    @property
    def S(self) -> int:
        return self.M + self.T_max

    @property
    def SR(self) -> int:
        return self.sr + 1 if self.refd else 0

    @property
    def slots(self) -> int:
        return self.S + self.R + self.SR + self.RR

    def _ref_cand(self, j: int) -> bool:
        return self.RR > 0 and self.rr > 0 and j % self.rr == 0

    def push(self, n: int, on_evict=None, on_commit=None) -> Tuple[int, List[int]]:
        if n < 1 or n > self.T_max:
            raise ValueError("push: n out of range")
        f = self.next_id
        S = self.S
        evicted = []
        before = set(self.resident)    # a frame can only be reported evicted if it was resident
        tn = max([self.t] + list(self.pending)) if self.refd else self.t

        def drop(j):
            self.online.discard(j)
            self.rspan.discard(j)
            self.refs.pop(j, None)
            self.rrefs.pop(j, None)
            self.refined.discard(j)
            self.pending.pop(j, None)
            if j in before:
                evicted.append(j)
            if on_evict:
                on_evict(j)

        def keep_refined_ref(j) -> bool:
            """Give j a refined-reference slot: the lowest free one, else the oldest
            reference's if j is newer (the oldest leaves); False: j is not kept."""
            b = S + self.R + self.SR
            free = [k for k in range(b, b + self.RR) if k not in self.rrefs.values()]
            if free:
                self.rrefs[j] = min(free)
                return True
            if not self.rrefs or min(self.rrefs) > j:
                return False
            oldest = min(self.rrefs)
            slot = self.rrefs[oldest]
            drop(oldest)
            self.rrefs[j] = slot
            return True

        # 1. refined span frames below t - s' (t: the watermark after this push's commits)
        for j in sorted(x for x in self.rspan if x < tn - self.sr):
            self.rspan.discard(j)
            if not (self._ref_cand(j) and keep_refined_ref(j)):
                self.rspan.add(j)
                drop(j)
        # 2. frames leaving the online span
        for j in sorted(x for x in self.online if x < f - self.M):
            self.online.discard(j)
            has_refined = j in self.refined or j in self.pending
            if self.refd and has_refined and j >= tn - self.sr:
                self.rspan.add(j)
                continue
            if self.refd and has_refined and self._ref_cand(j) and keep_refined_ref(j):
                continue
            if self.r > 0 and j % self.r == 0:
                free = [k for k in range(S, S + self.R) if k not in self.refs.values()]
                if free:
                    slot = min(free)
                else:
                    oldest = min(self.refs)
                    slot = self.refs[oldest]
                    drop(oldest)
                self.refs[j] = slot
            else:
                self.online.add(j)
                drop(j)
        # 3. queued commits: resident frames are overwritten; with the refined memory, others
        # land in it when Eq. 4 selects them
        for j in sorted(self.pending):
            land = j in self.resident
            if not land and self.refd:
                if j >= tn - self.sr:
                    self.rspan.add(j)
                    land = True
                elif self._ref_cand(j):
                    land = keep_refined_ref(j)
            if land:
                self.refined.add(j)
                if on_commit:
                    on_commit(j, self.pending[j])
        self.pending.clear()
        self.t = tn
        evicted.sort()
        for j in range(f, f + n):
            self.online.add(j)
        self.next_id = f + n
        self.cur_first, self.cur_n = f, n
        self.stepped = False
        return f, evicted

    def _check_past(self, fid: int) -> int:
        if fid < 0:
            return VI_E_ARG
        if fid >= self.next_id or (fid >= self.cur_first and not self.stepped):
            # a future frame, or a frame of the chunk whose step has not completed yet
            # ("t >= f -> protocol error"; reading Q13: never tear a frame)
            return VI_E_PROTOCOL
        if fid not in self.resident:
            return VI_NOT_RESIDENT
        return VI_OK

    def _may_land(self, fid: int) -> bool:
        """A past, non-resident frame's refine commit can still be used (refined memory on):
        it is within s' of the watermark the commit would raise it to, or a refined-reference
        candidate newer than the oldest refined reference held (or a slot is free)."""
        if not self.refd:
            return False
        tw = max([self.t, fid] + list(self.pending))
        if fid >= tw - self.sr:
            return True
        return self._ref_cand(fid) and (len(self.rrefs) < self.RR or fid > min(self.rrefs))

    def evict(self, fid: int, on_evict=None) -> int:
        st = self._check_past(fid)
        if st == VI_OK:
            self.online.discard(fid)
            self.rspan.discard(fid)
            self.refs.pop(fid, None)
            self.rrefs.pop(fid, None)
            self.refined.discard(fid)
            self.pending.pop(fid, None)
            if on_evict:
                on_evict(fid)
        return st

    def commit(self, fid: int, payload) -> int:
        st = self._check_past(fid)
        if st == VI_NOT_RESIDENT and self._may_land(fid):
            st = VI_OK
        if st == VI_OK:
            self.pending[fid] = payload
        return st

    def window(self) -> List[int]:
        """Memory frames the current chunk attends to, in temporal order (Eq. 3 / Eq. 4)."""
        return sorted(j for j in self.resident if j < self.cur_first)

    def state(self) -> Tuple[List[int], List[int], int]:
        """(slot_id[slots], refined[slots], valid mask): online span slot = id mod S (SURVEY
        §8(c)), then the reference slots, refined span slot = S + R + id mod (s'+1), then the
        refined reference slots."""
        S = self.S
        slot_id, ref, mask = [-1] * self.slots, [0] * self.slots, 0
        for j in self.resident:
            if j in self.refs:
                s = self.refs[j]
            elif j in self.rrefs:
                s = self.rrefs[j]
            elif j in self.rspan:
                s = S + self.R + j % self.SR
            else:
                s = j % S
            assert slot_id[s] == -1, "two resident frames share a slot"
            slot_id[s] = j
            ref[s] = int(j in self.refined)
            mask |= 1 << s
        return slot_id, ref, mask


class OracleStream:
    """A live stream through the Memory model (Eq. 3), one chunk of n new frames per step."""

    def __init__(self, cfg, w: Dict[str, np.ndarray], chunk_causal: bool = False, store=None):
        self.cfg = cfg
        self.w = w
        self.store = store     # None: the oracle; a rounding function: the bf16-storage emulation
        self.mem = OracleMemory(cfg.mem_frames, cfg.t_new, getattr(cfg, "ref_rate", 0), getattr(cfg, "max_refs", 0),
                                refined_span=(cfg.refined_span if getattr(cfg, "refined_mem", 0) else None),
                                refined_rate=getattr(cfg, "refined_rate", 0),
                                max_refined_refs=getattr(cfg, "max_refined_refs", 0))
        self.chunk_causal = chunk_causal
        # (layer, frame id) -> ("x", block input [P, D]) or ("kv", K [P, D], V [P, D])
        self.entries: Dict[Tuple[int, int], tuple] = {}

    # -- bookkeeping -------------------------------------------------------------
    def push(self, n: int):
        def drop(j):
            for l in range(self.cfg.layers):
                self.entries.pop((l, j), None)

        def apply(j, payload):
            K, V = payload
            for l in range(self.cfg.layers):
                self.entries[(l, j)] = ("kv", np.asarray(K[l], np.float64), np.asarray(V[l], np.float64))
        return self.mem.push(n, on_evict=drop, on_commit=apply)

    def evict(self, fid: int) -> int:
        def drop(j):
            for l in range(self.cfg.layers):
                self.entries.pop((l, j), None)
        return self.mem.evict(fid, on_evict=drop)

    def commit(self, fid: int, K: np.ndarray, V: np.ndarray) -> int:
        return self.mem.commit(fid, (np.array(K, np.float64), np.array(V, np.float64)))

    def memory_kv(self, l: int) -> List[Tuple[np.ndarray, np.ndarray]]:
        out = []
        for j in self.mem.window():
            e = self.entries[(l, j)]
            if e[0] == "kv":
                out.append((e[1], e[2]))
            else:
                _, _, K, V = qkv(e[1], self.w, l, self.cfg, self.store)
                out.append((K, V))
        return out

    # -- one memory step ---------------------------------------------------------------
    def step(self, feats: np.ndarray) -> Tuple[np.ndarray, Dict[str, object]]:
        """Process the chunk pushed last: feats [n, H, W, C] -> output maps [n, H, W, C]."""
        cfg = self.cfg
        n = feats.shape[0]
        assert n == self.mem.cur_n, "step() must follow push(n)"
        P = cfg.tokens
        Tp, X = embed(feats, self.w, cfg)
        stages: Dict[str, object] = dict(tp=Tp, x0=X.copy(), layers=[])
        for l in range(cfg.layers):
            mem = self.memory_kv(l)
            for i in range(n):   # cache this block's input for the chunk's frames
                self.entries[(l, self.mem.cur_first + i)] = ("x", X[i * P:(i + 1) * P].copy())
            X, st = block_memory(X, mem, self.w, l, cfg, n, self.chunk_causal, self.store)
            stages["layers"].append(st)
        Yp, out = compose(X, self.w, cfg, n)
        stages["x"] = X
        stages["yp"] = Yp
        stages["out"] = out
        self.mem.mark_stepped()
        return out, stages

    def frame_kv(self, l: int, fid: int) -> Tuple[np.ndarray, np.ndarray]:
        """K/V of a resident frame at block l as the oracle would attend to them."""
        e = self.entries[(l, fid)]
        if e[0] == "kv":
            return e[1], e[2]
        _, _, K, V = qkv(e[1], self.w, l, self.cfg, self.store)
        return K, V


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp64 values to the nearest bf16 (round-to-nearest-even), returned as fp64.
    Two steps: fp64 -> fp32 (RNE) -> bf16 (RNE on the fp32 bit pattern); this double
    rounding is what a GPU storing an fp32 accumulator as bf16 does."""
    a32 = np.ascontiguousarray(np.asarray(a, np.float64).astype(np.float32))
    u = a32.view(np.uint32).astype(np.uint64)
    r = (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)
    r = np.where(np.isnan(a32), np.float32(np.nan), r)
    return r.astype(np.float64)


def emulate_bf16_storage(cfg, w: Dict[str, np.ndarray], chunk_causal: bool = False) -> "OracleStream":
    """The bf16-STORAGE EMULATION (GPU-free, test infrastructure for tolerance bars only):
    the oracle stream with every tensor the bf16 design STORES in bf16 rounded to bf16 at
    that point -- the GEMM A operands h = LN1(x), O (attention output), h2 = LN2(x) and the
    FFN hidden g, and Q, K, V (the query buffer and the K/V ring-buffer memory; BASELINE
    north_star "in bf16 with fp32 accumulate", reading Q15).  The softmax
    probabilities P (bf16 in the GPU's TMEM) are NOT rounded: that rounding, the fp32
    accumulation order and the exp2 approximations are the GPU's own arithmetic, which the
    tests hold to the plain bar against this emulation.  Everything else stays exact fp64.
    Its distance from the plain oracle is the error storage alone causes at the given logit
    scale (a logit s moves by ~|s| 2^-8); tests derive the bars of the logit-sensitive
    weight variants from it."""
    return OracleStream(cfg, w, chunk_causal=chunk_causal, store=bf16_round)


def mac_counts(P: int, n_mem: int, n_new: int, D: int) -> int:
    """Score MACs of one memory-step block: Nq * Nk * D."""
    return (n_new * P) * ((n_mem + n_new) * P) * D


def rel_err(got: np.ndarray, ref: np.ndarray, den_ref: Optional[np.ndarray] = None) -> float:
    """Tolerance metric (reading Q18): max_i |g_i - o_i| / max(|d_i|, rms(d)), d = ref (or
    ``den_ref``: distances to an emulation are normalised by the oracle's values, so that
    rel_err(g, o) <= rel_err(g, e; den_ref=o) + rel_err(e, o) holds element by element)."""
    got = np.asarray(got, np.float64); ref = np.asarray(ref, np.float64)
    d = ref if den_ref is None else np.asarray(den_ref, np.float64)
    rms = math.sqrt(float(np.mean(d * d))) if d.size else 0.0
    den = np.maximum(np.abs(d), rms if rms > 0 else 1e-300)
    return float(np.max(np.abs(got - ref) / den)) if ref.size else 0.0
