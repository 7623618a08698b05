"""GPU parity of the Refined dual-model run (§3.5, Eq. 4; SURVEY §8(f)
NEXT-1): an online context (T = 1, memory span M) and a refining context (joint windows of
`window` past frames, M = 0) whose per-block K/V of those frames are read back
(vi_memory_read) and committed into the online memory (vi_refine_commit).

The oracle replays the same schedule with two OracleStreams: the refiner's K/V (fp64,
computed by the oracle itself) are committed into the online oracle, applied at its next
push.  Bars: the bf16 path's 2e-2 on every output frame, identical ring state (which
slots hold refined entries) and, with the refiner off, bitwise equality with the plain
Memory model (degradation to memory mode)."""
import numpy as np
import pytest
import torch

from oracle import vi_oracle as O
from vi_synth import CONFIGS, make_features, make_weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2403_16161_b200 import build
    build.build()


def _cfg():
    return CONFIGS["C3S"].replace(t_new=1, mem_frames=3, layers=2)


def _oracle_refined(cfg, w, feats, window, every):
    online = O.OracleStream(cfg, w)
    ref = O.OracleStream(cfg.replace(t_new=window, mem_frames=0), w)
    outs = []
    for f in range(feats.shape[0]):
        online.push(1)
        out, _ = online.step(feats[f:f + 1])
        outs.append(out[0])
        if (f + 1) % every == 0:
            lo = max(0, f - window + 1)
            n = f - lo + 1
            first, _ = ref.push(n)
            ref.step(feats[lo:f + 1])
            for i in range(n):
                K = np.stack([ref.frame_kv(l, first + i)[0] for l in range(cfg.layers)])
                V = np.stack([ref.frame_kv(l, first + i)[1] for l in range(cfg.layers)])
                online.commit(lo + i, K, V)
    return np.stack(outs), online


def test_refined_synchronous_schedule_matches_oracle():
    from paper_2403_16161_b200.refined import RefinedRun
    cfg = _cfg()
    w = make_weights(cfg, seed=0, variant="sensitive")
    N, window, every = 9, 4, 2
    feats = make_features(cfg, N, seed=0, masked="moving")
    ref_out, orc = _oracle_refined(cfg, w, feats, window, every)
    run = RefinedRun(cfg, w, window=window, every=every, synchronous=True)
    f = torch.from_numpy(feats).to(torch.bfloat16).cuda()
    out = torch.empty_like(f)
    run.run(f, out)
    got = out.float().cpu().numpy().astype(np.float64)
    for i in range(N):
        e = O.rel_err(got[i], ref_out[i])
        assert e <= 2e-2, f"frame {i}: rel_err {e:.3e}"
    assert run.online.state() == tuple(orc.mem.state())       # same refined slots
    assert run.stats["windows"] == N // every and run.stats["commits"] > 0
    run.close()


def test_refiner_off_is_the_memory_model():
    from paper_2403_16161_b200 import vi
    from paper_2403_16161_b200.refined import RefinedRun
    cfg = _cfg()
    w = make_weights(cfg, seed=1)
    feats = make_features(cfg, 6, seed=1, masked="moving")
    f = torch.from_numpy(feats).to(torch.bfloat16).cuda()
    out = torch.empty_like(f)
    run = RefinedRun(cfg, w, refiner=False)
    run.run(f, out)
    ctx = vi.Context.from_synth(cfg)
    ctx.set_weights(w)
    ref = torch.empty_like(f)
    for i in range(6):
        ctx.run_step(f[i:i + 1], 1, ref[i:i + 1])
    ctx.sync()
    assert torch.equal(out, ref)
    run.close()


def test_memory_read_roundtrip_and_protocol():
    """vi_memory_read returns exactly what vi_refine_commit wrote (host and device buffers)."""
    from paper_2403_16161_b200 import vi
    cfg = _cfg()
    ctx = vi.Context.from_synth(cfg)
    ctx.set_weights(make_weights(cfg, seed=2))
    f = torch.from_numpy(make_features(cfg, 3, seed=2)).to(torch.bfloat16).cuda()
    o = torch.empty_like(f)
    for i in range(3):
        ctx.run_step(f[i:i + 1], 1, o[i:i + 1])
    shape = (cfg.layers, cfg.tokens, cfg.d_model)
    k = torch.randn(shape).to(torch.bfloat16)
    v = torch.randn(shape).to(torch.bfloat16)
    assert ctx.commit(1, k, v) == vi.VI_OK
    ctx.run_step(f[0:1], 1, o[0:1])                                  # the push applies it
    kd, vd = torch.empty(shape, dtype=torch.bfloat16, device="cuda"), torch.empty(shape, dtype=torch.bfloat16,
                                                                                 device="cuda")
    assert ctx.read_kv(1, kd, vd) == vi.VI_OK
    assert torch.equal(kd.cpu(), k) and torch.equal(vd.cpu(), v)
    kh, vh = torch.empty(shape, dtype=torch.bfloat16), torch.empty(shape, dtype=torch.bfloat16)
    assert ctx.read_kv(1, kh, vh) == vi.VI_OK
    assert torch.equal(kh, k) and torch.equal(vh, v)
    assert ctx.read_kv(10, kh, vh) == vi.VI_E_PROTOCOL               # future frame
    ctx.run_step(f[0:1], 1, o[0:1])                                  # frame 4: frame 0 leaves (M = 3)
    assert ctx.read_kv(0, kh, vh) == vi.VI_NOT_RESIDENT


# ---------------------------------------------------------------- Eq. 4's refined memory M-bar

def _refined_stream(cfg, w, steps, commits, seed, tol):
    """Free-running oracle (+ bf16-storage emulation on the bf16 path) and GPU streams with
    refine commits of arbitrary K/V (commits[i] = frame ids committed before push i); every step
    compared stage by stage, ring state (slots, refined bits) and commit codes bit-exact."""
    import gpu_harness
    from test_gpu_parity import check_attention_kernel, compare_step
    from vi_synth import make_kv
    g = gpu_harness.GpuStream(cfg, w)
    o = O.OracleStream(cfg, w)
    e = O.emulate_bf16_storage(cfg, w) if cfg.dtype == "bf16" else None
    for i in range(steps):
        for fid in commits.get(i, ()):
            K, V = make_kv(cfg, seed + 100, fid, scale=0.5)        # bf16-representable on the bf16 path
            if cfg.dtype == "bf16":                                 # the payload is in the ctx dtype
                Kg, Vg = (torch.from_numpy(a).to(torch.bfloat16).contiguous() for a in (K, V))
            else:
                Kg, Vg = K, V
            codes = [g.ctx.commit(fid, Kg, Vg), o.commit(fid, K, V)]
            if e is not None:
                codes.append(e.commit(fid, K, V))
            assert len(set(codes)) == 1, (i, fid, codes)
        feats = make_features(cfg, 1, first_frame=i, seed=seed, masked="moving")
        o.push(1)
        _, ost = o.step(feats)
        est = None
        if e is not None:
            e.push(1)
            _, est = e.step(feats)
        _, gst = g.step(feats)
        assert g.ctx.state() == tuple(o.mem.state()), f"step {i}: ring state differs"
        compare_step(cfg, ost, gst, tol, tag=f"step {i}: ", est=est)
        if cfg.dtype == "bf16":
            fids = o.mem.window() + [o.mem.cur_first]
            check_attention_kernel(g, cfg, gst["layers"][-1], cfg.layers - 1, fids, tol, tag=f"step {i}: ")
    return g, o


# a refiner lagging the online stream: at frame i it hands over frames up to i - 3 (some still
# in the online span: overwritten in place; older ones land in the refined span or, multiples
# of r' = 3, in the refined references; the oldest are useless and rejected or dropped)
_COMMITS = {4: [0, 1], 6: [1, 2, 3], 8: [3, 4, 5], 9: [6], 11: [6, 7, 8], 12: [9], 13: [0, 9, 10]}


def test_refined_memory_bf16_matches_oracle():
    """Eq. 4 on the bf16 tensor-core path: online span 2, refined span s' = 2,
    refined references every r' = 3 frames (2 kept); 14 one-frame steps."""
    cfg = CONFIGS["C3S"].replace(layers=2, t_new=1, mem_frames=2, refined_mem=1, refined_span=2, refined_rate=3,
                                 max_refined_refs=2)
    w = make_weights(cfg, seed=40, variant="sensitive")
    g, o = _refined_stream(cfg, w, 14, _COMMITS, seed=40, tol=2e-2)
    assert g.ctx.refined_watermark() == o.mem.t == 10
    sid, ref, _ = g.ctx.state()
    assert sum(1 for s in sid[cfg.mem_frames + 1:] if s >= 0) >= 3     # refined regions in use


def test_refined_memory_fp32_matches_oracle():
    """The same schedule on the fp32 SIMT path (BASELINE configs[0] shape) at 1e-4."""
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=2, refined_mem=1, refined_span=2, refined_rate=3,
                                max_refined_refs=2)
    w = make_weights(cfg, seed=41, variant="sensitive")
    _refined_stream(cfg, w, 14, _COMMITS, seed=41, tol=1e-4)
