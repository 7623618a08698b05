"""Refined dual-model live run (§3.5, Eq. 4; BASELINE configs[4]).

Two contexts of libvi.so work side by side on one live stream:
  * the Online Inpainter: the Memory model, one memory step per incoming frame (T = 1,
    memory span M), on a high-priority CUDA stream;
  * the Refining Inpainter: every `every` frames it re-inpaints the past window of the last
    `window` frames jointly (T = window, M = 0: the window attention of the original
    model, "it can work directly on windows"), on a normal-priority stream, and hands
    its per-block K/V of those frames to the online context (vi_memory_read ->
    vi_refine_commit), which overwrites the online entries of the frames still in its
    memory at its next push (reading Q13; BASELINE configs[4] "overwrites those frames'
    K/V memory via vi_refine_commit").
The refiner runs in its own host thread (its results are "only created to be used by the
Online Inpainter"), so the online loop never waits for it; `synchronous=True` runs
each refine job inline after the online step that triggered it (the deterministic
schedule the parity test replays on the oracle).  Both contexts may live on one GPU (a
stream per GPU, BASELINE configs[4]) or on two (the paper's layout: the K/V
payload then crosses NVLink inside vi_refine_commit's device-to-device copy).
This module is host orchestration only: every step of the path runs in libvi.so.
"""
from __future__ import annotations

import queue
import threading
import time
from typing import Dict, Optional

import numpy as np
import torch

from . import vi


class RefinedRun:
    def __init__(self, cfg, weights: Dict[str, np.ndarray], window: int = 20, every: int = 5,
                 device_online: int = 0, device_refiner: Optional[int] = None, refiner: bool = True,
                 synchronous: bool = False, refined_span: Optional[int] = None, refined_rate: int = 0,
                 max_refined_refs: int = 0):
        """refined_span = s' (not None): the online memory also keeps Eq. 4's refined memory
        M-bar_{t-s'}^{t} U M-bar_{1,r'}^{t} (refined_rate r', max_refined_refs kept), and the
        refiner commits only the frames Eq. 4 can use (its window's frames still in the online
        span, within s' of its newest frame, or multiples of r')."""
        assert cfg.t_new == 1, "the online inpainter processes one frame at a time (Eq. 3/4)"
        self.cfg, self.window, self.every = cfg, window, every
        self.refiner_on, self.synchronous = refiner, synchronous
        self.sr, self.rr = refined_span, refined_rate
        ocfg = cfg
        if refined_span is not None:
            ocfg = cfg.replace(refined_mem=1, refined_span=refined_span, refined_rate=refined_rate,
                               max_refined_refs=max_refined_refs)
        # CUDA clamps the priority to the device's greatest (most negative) value
        self.online = vi.Context.from_synth(ocfg, device=device_online, stream_priority=-100)
        self.online.set_weights(weights)
        self.dev_ref = device_online if device_refiner is None else device_refiner
        self.ref = None
        if refiner:
            rcfg = cfg.replace(t_new=window, mem_frames=0)
            self.ref = vi.Context.from_synth(rcfg, device=self.dev_ref, max_new_frames=window)
            self.ref.set_weights(weights)
            shape = (cfg.layers, cfg.tokens, cfg.d_model)
            with torch.cuda.device(self.dev_ref):
                self.kbuf = torch.empty(shape, dtype=torch.bfloat16, device=f"cuda:{self.dev_ref}")
                self.vbuf = torch.empty_like(self.kbuf)
        self.stats = dict(windows=0, commits=0, not_resident=0, refine_s=0.0, lag_frames=[], watermark=-1)
        self._q: "queue.Queue" = queue.Queue()
        self._online_frame = -1

    # -- refiner -------------------------------------------------------------------
    def _refine(self, feats_ref: torch.Tensor, f: int, ref_out: torch.Tensor):
        """Re-inpaint frames [f - window + 1, f] jointly; commit their K/V to the online ctx."""
        t0 = time.perf_counter()
        lo = max(0, f - self.window + 1)
        n = f - lo + 1
        # fixed staging buffers: the step graph is keyed by its buffers (vi_run_step)
        with torch.cuda.device(self.dev_ref):
            self.ref_in[:n].copy_(feats_ref[lo:f + 1])
            torch.cuda.current_stream(self.dev_ref).synchronize()
        first = self.ref.run_step(self.ref_in[:n], n, ref_out[:n])
        self.ref.sync()
        for i in range(n):
            fid = lo + i
            if self.sr is not None and not (fid >= f - max(self.sr, self.cfg.mem_frames) or
                                            (self.rr > 0 and fid % self.rr == 0)):
                continue                             # Eq. 4 would not select it: not handed over
            if self.ref.read_kv(first + i, self.kbuf, self.vbuf) != vi.VI_OK:
                continue
            st = self.online.commit(fid, self.kbuf, self.vbuf)
            if st == vi.VI_OK:
                self.stats["commits"] += 1
            else:
                self.stats["not_resident"] += 1
        self.stats["windows"] += 1
        self.stats["refine_s"] += time.perf_counter() - t0
        self.stats["watermark"] = f
        self.stats["lag_frames"].append(self._online_frame - f)

    def _worker(self, feats_ref, ref_out):
        while True:
            f = self._q.get()
            if f is None:
                return
            self._refine(feats_ref, f, ref_out)

    # -- the live loop ----------------------------------------------------------------
    def run(self, feats: torch.Tensor, out: torch.Tensor, feats_ref: Optional[torch.Tensor] = None):
        """Inpaint feats [N, H, W, C] (device, bf16) frame by frame into out.  feats_ref: the
        same frames on the refiner's device (defaults to feats).  The loop is paced like a live
        stream (each frame completes before the next is taken).  Returns the online wall
        seconds, CUDA events on the online stream from the first frame's start to the last
        frame's end."""
        N = feats.shape[0]
        feats_ref = feats if feats_ref is None else feats_ref
        ref_out = None
        worker = None
        if self.ref is not None:
            ref_out = torch.empty((self.window,) + tuple(feats.shape[1:]), dtype=feats.dtype,
                                  device=feats_ref.device)
            self.ref_in = torch.empty_like(ref_out)
            if not self.synchronous:
                worker = threading.Thread(target=self._worker, args=(feats_ref, ref_out), daemon=True)
                worker.start()
        stream = torch.cuda.ExternalStream(self.online.stream(), device=feats.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stage_in = torch.empty_like(feats[:1])
        stage_out = torch.empty_like(out[:1])
        e0.record(stream)
        for f in range(N):
            with torch.cuda.stream(stream):          # ordered on the online stream
                stage_in.copy_(feats[f:f + 1])
            self.online.run_step(stage_in, 1, stage_out)
            with torch.cuda.stream(stream):
                out[f:f + 1].copy_(stage_out)
            # live pacing: frame f is shown (and its memory entries exist) before frame f+1
            # is taken, so commits see the online memory as a live stream would
            self.online.sync()
            self._online_frame = f
            if self.ref is not None and (f + 1) % self.every == 0:
                if self.synchronous:
                    self._refine(feats_ref, f, ref_out)
                else:
                    self._q.put(f)
        e1.record(stream)
        if worker is not None:
            self._q.put(None)
            worker.join()
        self.online.sync()
        return e0.elapsed_time(e1) / 1e3

    def close(self):
        self.online.close()
        if self.ref is not None:
            self.ref.close()
