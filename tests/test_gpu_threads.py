"""Two contexts driven from two host threads at once on one GPU (the Refined model's online and
refining inpainters share a process; SPEC's refiner thread): each context's
outputs equal the same steps run alone, bitwise, and one context's profiling mode never
leaks into the other's launches (every launch argument comes from its own context)."""
import threading

import pytest
import torch

from vi_synth import CONFIGS, make_features, make_weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2403_16161_b200 import build
    build.build()


def _steps(ctx, cfg, feats, outs, prof=None):
    if prof is not None:
        ctx.profile(prof)
    for i in range(len(outs)):
        ctx.run_step(feats[i], cfg.t_new, outs[i])
    ctx.sync()


def test_two_contexts_two_threads_bitwise():
    from paper_2403_16161_b200 import vi
    cfgs = [CONFIGS["C3S"].replace(layers=2), CONFIGS["C3S"].replace(layers=2, t_new=1, mem_frames=4)]
    ws = [make_weights(c, seed=50 + i, variant="sensitive") for i, c in enumerate(cfgs)]
    steps = 6
    feats = [[torch.from_numpy(make_features(c, c.t_new, first_frame=i * c.t_new, seed=60 + k)).to(
        torch.bfloat16).cuda() for i in range(steps)] for k, c in enumerate(cfgs)]
    ref = []
    for k, c in enumerate(cfgs):                      # alone, one after the other
        ctx = vi.Context.from_synth(c)
        ctx.set_weights(ws[k])
        outs = [torch.empty_like(f) for f in feats[k]]
        _steps(ctx, c, feats[k], outs)
        ref.append(outs)
        ctx.close()
    ctxs = []
    for k, c in enumerate(cfgs):
        ctx = vi.Context.from_synth(c)
        ctx.set_weights(ws[k])
        ctxs.append(ctx)
    got = [[torch.empty_like(f) for f in feats[k]] for k in range(2)]
    errs = []

    def run(k):
        try:
            _steps(ctxs[k], cfgs[k], feats[k], got[k], prof=3 if k == 0 else 0)
        except Exception as e:       # surfaced below
            errs.append(e)
    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(2):
        for i in range(steps):
            assert torch.equal(got[k][i], ref[k][i]), f"context {k} step {i}"
    # context 0 timed its own GEMMs (profile mode 3); context 1 launched untimed
    p0, p1 = ctxs[0].profile_read(), ctxs[1].profile_read()
    assert p0["gemm"][1] > 0 and p1["gemm"][1] == 0
    for c in ctxs:
        c.close()
