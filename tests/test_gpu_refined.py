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
