"""GPU parity of the head-sharded memory step: G ranks, each with its
heads' Q/K/V projection, K/V memory and attention, all-gather of the head outputs, then the
replicated output projection / FFN.

One GPU stands in for G ranks the way B200_PROFILING.md allows: the G contexts run in one
process, their kernels never wait on one another, and the exchange is the library's
vi_tp_local_allgather (stream-ordered copies between the ranks' gathered buffers) between
each block's _attn and _ffn halves.  The NCCL path (the one `bench.py --tp` uses on N GPUs)
runs here over a 1-rank communicator.  Bars: the oracle's (BASELINE north_star, 2e-2 on
the bf16 path), and the replicated outputs of all ranks bitwise identical."""
import numpy as np
import pytest
import torch

from oracle import vi_oracle as O
from vi_synth import CONFIGS, make_features, make_kv, make_weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2403_16161_b200 import build
    build.build()


def _rel(got, ref):
    return O.rel_err(got.float().cpu().numpy().astype(np.float64), ref)


class TpGroup:
    """G head-sharded contexts of one process on cuda:0, driven block by block."""

    def __init__(self, cfg, w, G):
        from paper_2403_16161_b200 import vi
        self.vi, self.cfg, self.G = vi, cfg, G
        self.ctxs = [vi.Context.from_synth(cfg, tp_size=G, tp_rank=r) for r in range(G)]
        for c in self.ctxs:
            c.set_weights(w)
        self.x = [torch.zeros(cfg.t_new * cfg.tokens, cfg.d_model, dtype=torch.float32, device="cuda")
                  for _ in range(G)]

    def step(self, feats):
        cfg = self.cfg
        n = feats.shape[0]
        f = torch.from_numpy(feats).to(torch.bfloat16).cuda()
        pushed = [c.push(n) for c in self.ctxs]
        assert all(p == pushed[0] for p in pushed)
        xs = [x[: n * cfg.tokens] for x in self.x]
        for c, x in zip(self.ctxs, xs):
            c.soft_split(f, n, x, 1)
        for l in range(cfg.layers):
            for c, x in zip(self.ctxs, xs):
                c.memory_step_attn(l, x)
            self.vi.tp_local_allgather(self.ctxs)
            for c, x in zip(self.ctxs, xs):
                c.memory_step_ffn(l, x, x)
        outs = []
        for c, x in zip(self.ctxs, xs):
            out = torch.empty(n, cfg.feat_h, cfg.feat_w, cfg.feat_c, dtype=torch.bfloat16, device="cuda")
            c.soft_composite(x, n, out, 1)
            outs.append(out)
        for c in self.ctxs:
            c.sync()
        return outs, [x.clone() for x in xs]


def _run_group(cfg, w, G, ns, seed=0):
    from paper_2403_16161_b200 import vi
    grp = TpGroup(cfg, w, G)
    orc = O.OracleStream(cfg, w)
    emu = O.emulate_bf16_storage(cfg, w)       # logit-sensitive weights: bf16-storage bars
    full = vi.Context.from_synth(cfg)           # the unsharded context on the same frames
    full.set_weights(w)
    fid = 0
    for i, n in enumerate(ns):
        feats = make_features(cfg, n, first_frame=fid, seed=seed)
        fid += n
        orc.push(n)
        ref, ost = orc.step(feats)
        emu.push(n)
        ref_e, est = emu.step(feats)
        outs, xs = grp.step(feats)
        for r in range(1, G):   # replicated work is bitwise identical on every rank
            assert torch.equal(outs[r], outs[0]) and torch.equal(xs[r], xs[0]), f"step {i}: rank {r} differs"
        # bars (test_gpu_parity.compare_step): within 2e-2 + E of the oracle, E = the
        # bf16-storage emulation's distance to the oracle (GPU-free)
        for what, g, o, e in (("x", xs[0], ost["x"], est["x"]), ("out", outs[0], ref, ref_e)):
            gh = g.float().cpu().numpy().astype(np.float64)
            go, eo = O.rel_err(gh, o), O.rel_err(e, o)
            assert go <= 2e-2 + eo, f"G={G} step {i}: {what} {go:.3e} vs oracle > 2e-2 + E {eo:.3e}"
        # the gathered head outputs of the last block: against the unsharded context's (same
        # kernels, only the KV split differs) and against the oracle / emulation as above
        buf = torch.empty(n * cfg.tokens, cfg.d_model, dtype=torch.bfloat16, device="cuda")
        grp.ctxs[G - 1].debug_read("o", buf)
        fo = torch.empty(n * cfg.tokens, cfg.d_model, dtype=torch.bfloat16, device="cuda")
        f_feat = torch.from_numpy(feats).to(torch.bfloat16).cuda()
        full.run_step(f_feat, n, torch.empty_like(f_feat))
        full.debug_read("o", fo)
        ref_o, emu_o = ost["layers"][-1]["o"], est["layers"][-1]["o"]
        e_sh, e_full = _rel(buf, ref_o), _rel(fo, ref_o)
        assert _rel(buf, fo.float().cpu().numpy().astype(np.float64)) <= 1e-2, (e_sh, e_full)
        bar = 2e-2 + O.rel_err(emu_o, ref_o)
        assert e_sh <= bar, f"G={G} step {i}: o rel_err {e_sh:.3e} (unsharded {e_full:.3e}) > {bar:.3e}"
    return grp


@pytest.mark.parametrize("G", [2, 4, 8])
def test_head_sharded_group_matches_oracle(G):
    """C3S (4 heads, d 128, 180 tokens/frame, T=2, M=3): G=2 two heads per rank, G=4 one
    head per rank, G=8 one head and half of the query rows per rank."""
    cfg = CONFIGS["C3S"]
    _run_group(cfg, make_weights(cfg, seed=0, variant="sensitive"), G, ns=[2, 2, 2, 2])


def test_head_sharded_ragged_chunks_empty_query_part():
    """n=1 chunks leave the second query part of every head empty at G=8 (part rows are
    fixed by T_max): those ranks skip the attention but still join the exchange."""
    cfg = CONFIGS["C3S"].replace(layers=1)
    _run_group(cfg, make_weights(cfg, seed=1, variant="sensitive"), 8, ns=[2, 1, 2, 1, 1])


def test_head_sharded_memory_is_the_heads_columns():
    """Each rank's K/V memory holds exactly its heads' columns of the unsharded memory, and a
    refine commit (full [L,P,D] payload) lands as the rank's column slice."""
    from paper_2403_16161_b200 import vi
    cfg = CONFIGS["C3S"].replace(layers=1)
    w = make_weights(cfg, seed=2)
    G = 4
    grp = TpGroup(cfg, w, G)
    full = vi.Context.from_synth(cfg)
    full.set_weights(w)
    xf = torch.zeros(cfg.t_new * cfg.tokens, cfg.d_model, dtype=torch.float32, device="cuda")
    for i in range(2):
        feats = make_features(cfg, 2, first_frame=2 * i, seed=2)
        grp.step(feats)
        f = torch.from_numpy(feats).to(torch.bfloat16).cuda()
        full.push(2)
        full.soft_split(f, 2, xf, 1)
        full.memory_step(0, xf, xf)
    full.sync()
    d, P = cfg.head_dim, cfg.tokens
    kf = torch.empty(P, cfg.d_model, dtype=torch.bfloat16, device="cuda")
    vf = torch.empty_like(kf)
    full.debug_read("k", kf, 0, 1)
    full.debug_read("v", vf, 0, 1)
    for r, c in enumerate(grp.ctxs):
        kr = torch.empty(P, d, dtype=torch.bfloat16, device="cuda")
        vr = torch.empty_like(kr)
        c.debug_read("k", kr, 0, 1)
        c.debug_read("v", vr, 0, 1)
        # same bf16 GEMM over the rank's weight rows: identical to the unsharded columns
        assert torch.equal(kr, kf[:, r * d:(r + 1) * d]) and torch.equal(vr, vf[:, r * d:(r + 1) * d])
    k, v = make_kv(cfg, 7, 1)
    kb, vb = (torch.from_numpy(a).to(torch.bfloat16).contiguous() for a in (k, v))   # ctx dtype, host
    for c in grp.ctxs:
        assert c.commit(1, kb, vb) == vi.VI_OK
    grp.step(make_features(cfg, 2, first_frame=4, seed=2))   # the push applies the commits
    for r, c in enumerate(grp.ctxs):
        kr = torch.empty(P, d, dtype=torch.bfloat16, device="cuda")
        vr = torch.empty_like(kr)
        c.debug_read("k", kr, 0, 1)
        c.debug_read("v", vr, 0, 1)
        kk, vv = kb[0][:, r * d:(r + 1) * d], vb[0][:, r * d:(r + 1) * d]
        assert torch.equal(kr.cpu(), kk) and torch.equal(vr.cpu(), vv)


def test_nccl_one_rank_communicator_run_step():
    """The NCCL path: head-major gathered buffer + ncclAllGather inside the captured step
    graph, over a 1-rank communicator; equals the oracle and the unsharded context."""
    from paper_2403_16161_b200 import vi
    cfg = CONFIGS["C3S"]
    w = make_weights(cfg, seed=3, variant="sensitive")
    ctx = vi.Context.from_synth(cfg, tp_size=1, tp_rank=0, nccl_id=vi.tp_unique_id())
    ctx.set_weights(w)
    ref_ctx = vi.Context.from_synth(cfg)
    ref_ctx.set_weights(w)
    orc = O.OracleStream(cfg, w)
    for i in range(4):
        feats = make_features(cfg, 2, first_frame=2 * i, seed=3)
        orc.push(2)
        ref, _ = orc.step(feats)
        f = torch.from_numpy(feats).to(torch.bfloat16).cuda()
        out, out2 = torch.empty_like(f), torch.empty_like(f)
        ctx.run_step(f, 2, out)
        ref_ctx.run_step(f, 2, out2)
        ctx.sync()
        ref_ctx.sync()
        assert _rel(out, ref) <= 2e-2
        # same kernels, same K order in the output projection: identical to unsharded
        assert torch.equal(out, out2)


def test_split_phase_equals_memory_step_and_protocol():
    from paper_2403_16161_b200 import vi
    cfg = CONFIGS["C3S"].replace(layers=2)
    w = make_weights(cfg, seed=4)
    a, b = vi.Context.from_synth(cfg), vi.Context.from_synth(cfg)
    for c in (a, b):
        c.set_weights(w)
    feats = make_features(cfg, 2, seed=4)
    f = torch.from_numpy(feats).to(torch.bfloat16).cuda()
    xa = torch.empty(2 * cfg.tokens, cfg.d_model, dtype=torch.float32, device="cuda")
    xb = torch.empty_like(xa)
    for c, x in ((a, xa), (b, xb)):
        c.push(2)
        c.soft_split(f, 2, x, 1)
    for l in range(cfg.layers):
        a.memory_step(l, xa, xa)
        b.memory_step_attn(l, xb)
        with pytest.raises(vi.ViError) as e:
            b.memory_step_attn(l, xb)               # this layer's _ffn is pending
        assert e.value.status == vi.VI_E_PROTOCOL
        b.memory_step_ffn(l, xb, xb)
    a.sync()
    b.sync()
    assert torch.equal(xa, xb)
    # a sharded context without a communicator cannot run the fused step
    s = vi.Context.from_synth(cfg, tp_size=2, tp_rank=0)
    s.set_weights(w)
    s.push(2)
    with pytest.raises(vi.ViError) as e:
        s.memory_step(0, xa, xa)
    assert e.value.status == vi.VI_E_PROTOCOL
    with pytest.raises(vi.ViError) as e:
        s.memory_step_ffn(0, xa, xa)               # _ffn before _attn
    assert e.value.status == vi.VI_E_PROTOCOL


@pytest.mark.parametrize("G", [2, 4, 8])
def test_head_sharded_window_attention(G):
    """Window attention (BASELINE configs[3]: heads sharded across GPUs with an all-gather of
    the head outputs) on the reduced map: 10 x 18 tokens in 2 x 3 windows of 5 x 6.  G = 8 > H:
    each head's windows are split between a rank pair by window rows (part-local outputs,
    gathered back to token rows before the output projection)."""
    cfg = CONFIGS["C3S"].replace(win_h=5, win_w=6)
    _run_group(cfg, make_weights(cfg, seed=5, variant="sensitive"), G, ns=[2, 1, 2, 2])


def test_head_sharded_window_attention_c4_shape_g8():
    """BASELINE configs[3] ("heads sharded across 2/4/8 GPUs") at its full token shape (2 of
    its 16 blocks): 720 tokens in 16 windows of 5 x 9, 5 new frames over a 10-frame memory,
    8 ranks = 4 heads x 2 halves of the window rows."""
    cfg = CONFIGS["C4"].replace(layers=2)
    _run_group(cfg, make_weights(cfg, seed=6, variant="sensitive"), 8, ns=[5, 5, 5, 5])


def test_bench_tp_one_rank_json_line():
    """`bench.py --tp` (the strong-scaling head-sharded run: NCCL all-gather inside every block)
    launched as the driver launches N = 1: one JSON line with the contract's keys, scaling
    "strong", the NCCL parallelism named, and the kernels counted."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--tp", "--config", "C3T1", "--steps", "5",
                        "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert k in line, k
    assert line["scaling"] == "strong" and line["value"] > 0 and line["gpu_launches"] > 0
    assert "NCCL" in line["config"]["parallelism"]
