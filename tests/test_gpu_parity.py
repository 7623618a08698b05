"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on the same
seeded inputs.  Bars (BASELINE.json north_star; metric = reading Q18, oracle.rel_err):
  * soft-split indexing and ring bookkeeping: bit-exact;
  * fp32 SIMT path: rel_err <= 1e-4 on every stage and output;
  * bf16 tensor-core path: rel_err <= 2e-2 on every stage and output.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import vi_oracle as O
from vi_synth import CONFIGS, make_features, make_kv, make_weights, round_bf16, rng_for

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2403_16161_b200 import build
    build.build()


def H():
    import gpu_harness
    return gpu_harness


def assert_close(got, ref, tol, what):
    got = got.float().cpu().numpy() if isinstance(got, torch.Tensor) else got
    e = O.rel_err(got, ref)
    assert np.isfinite(got).all(), f"{what}: non-finite values"
    assert e <= tol, f"{what}: rel_err {e:.3e} > {tol}"
    return e


# Per-test worst error / bar ratios (headroom record): VI_PARITY_LOG=<file> appends one JSON
# line per compared stage group, so a GPU run documents how close every test is to its bar.
PARITY_LOG = os.environ.get("VI_PARITY_LOG")


def log_parity(tag, errs, bars, emu=None):
    if not PARITY_LOG:
        return
    worst = max(errs, key=lambda k: errs[k] / bars[k])
    rec = {"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], "tag": tag,
           "worst_stage": worst, "err": errs[worst], "bar": bars[worst], "ratio": errs[worst] / bars[worst],
           "stages": {k: round(v, 6) for k, v in errs.items()}}
    if emu:
        we = max(emu, key=emu.get)
        rec["vs_emulation"] = {"stage": we, "err": emu[we]}
    with open(PARITY_LOG, "a") as f:
        f.write(json.dumps(rec) + "\n")


def stage_pairs(cfg, ost, gst, est=None):
    """(name, gpu, oracle, emulation) for every compared stage of one step."""
    out = [("x0", gst["x0"], ost["x0"], est["x0"] if est else None)]
    for l, (ol, gl) in enumerate(zip(ost["layers"], gst["layers"])):
        el = est["layers"][l] if est else None
        names = (("q",) if "q" in gl else ()) + (("o", "u", "g") if cfg.ffn_kind == 1 else ("o", "g")) + ("x",)
        for k in names:
            out.append((f"{k}{l}", gl[k], ol[k], el[k] if el else None))
    out.append(("out", gst["out"], ost["out"], est["out"] if est else None))
    return out


def compare_step(cfg, ost, gst, tol, tag="", est=None):
    """Stage-by-stage parity against the fp64 oracle (BASELINE north_star bars; metric =
    reading Q18).  Without `est` (the metric config's N(0, 0.02) weights, the fp32 path)
    every stage and output is held to `tol` as it stands.

    With `est` = the same step through ``oracle.emulate_bf16_storage`` (the oracle with every
    tensor the design stores in bf16 -- h, Q, K, V, O, h2, g -- rounded there; GPU-free,
    computed in this test from the same inputs): the logit-sensitive weight variants, whose
    attention amplifies the storage rounding of Q/K (a logit s moves by ~|s| 2^-8), hold every
    stage to rel_err(gpu, oracle) <= tol + E with E = rel_err(emulation, oracle) -- the
    storage error at this logit scale plus the plain bar for the GPU's own arithmetic (triangle
    inequality), no constant fitted to a GPU measurement.  The GPU's distance
    to the emulation itself is logged, not asserted: the two round h / Q / K of slightly
    different fp32-vs-fp64 values, so ~2.5 % of the stored elements sit one ulp apart at a
    rounding boundary, and sharp logits amplify exactly that (tools/parity_diag.py).  The
    attention kernel's own arithmetic (bf16 P, exp2 approximations) is held to `tol`
    separately against fp64 attention of the GPU's own Q/K/V (check_attention_kernel)."""
    errs, bars, emu = {}, {}, {}
    if "tp" in gst:
        assert np.array_equal(gst["tp"].float().cpu().numpy().astype(np.float64), ost["tp"]), "soft split not bit-exact"
    for name, g, o, e in stage_pairs(cfg, ost, gst, est):
        g = g.float().cpu().numpy() if isinstance(g, torch.Tensor) else g
        assert np.isfinite(g).all(), f"{tag}{name}: non-finite values"
        if e is None:
            errs[name], bars[name] = O.rel_err(g, o), tol
        else:
            emu[name] = O.rel_err(g, e, den_ref=o)
            errs[name], bars[name] = O.rel_err(g, o), tol + O.rel_err(e, o)
        assert errs[name] <= bars[name], f"{tag}{name}: rel_err {errs[name]:.3e} > {bars[name]:.3e}"
    log_parity(tag, errs, bars, emu)
    return errs


def check_attention_kernel(g, cfg, gl, layer, fids, tol, tag=""):
    """The attention kernel's own arithmetic: the GPU's attention output of block `layer`
    against fp64 attention (oracle.attention) of the GPU's OWN stored Q and K/V memory rows
    (frames `fids`, read back through vi_debug_read) -- isolates the bf16 P, the exp2
    approximations and the split merges from everything upstream; held to the plain bar."""
    ks, vs = [], []
    slot_ids = list(g.ctx.state()[0])
    for fid in fids:
        k, v = g.kv(layer, slot_ids.index(fid))
        ks.append(k.float().cpu().numpy().astype(np.float64))
        vs.append(v.float().cpu().numpy().astype(np.float64))
    q = gl["q"].float().cpu().numpy().astype(np.float64)
    ref = O.attention(q, np.concatenate(ks), np.concatenate(vs), cfg.heads)
    e = O.rel_err(gl["o"].float().cpu().numpy(), ref)
    assert e <= tol, f"{tag}attention kernel vs fp64 attention of its own Q/K/V: {e:.3e} > {tol}"
    log_parity(tag + "attention-kernel", {"o_kernel": e}, {"o_kernel": tol})
    return e


def run_pair(cfg, w, steps, ns=None, seed=0, masked=False, emulate=False):
    """Free-running oracle and GPU streams over the same frames; compare every step.
    `emulate`: also run the bf16-storage emulation (logit-sensitive weight variants)."""
    g = H().GpuStream(cfg, w)
    o = O.OracleStream(cfg, w)
    e = O.emulate_bf16_storage(cfg, w) if emulate else None
    fid = 0
    worst = 0.0
    for i in range(steps):
        n = ns[i] if ns else cfg.t_new
        feats = make_features(cfg, n, first_frame=fid, seed=seed, masked=masked)
        fid += n
        f_o, ev_o = o.push(n)
        _, ost = o.step(feats)
        est = None
        if e is not None:
            e.push(n)
            _, est = e.step(feats)
        _, gst = g.step(feats)
        assert (gst["first"], gst["evicted"]) == (f_o, ev_o)
        assert g.ctx.state() == tuple(o.mem.state()), "ring state differs"
        errs = compare_step(cfg, ost, gst, TOL[cfg.dtype], tag=f"step {i}: ", est=est)
        if cfg.dtype == "bf16" and not cfg.win_h:
            fids = o.mem.window() + list(range(o.mem.cur_first, o.mem.next_id))
            check_attention_kernel(g, cfg, gst["layers"][-1], cfg.layers - 1, fids, TOL["bf16"], tag=f"step {i}: ")
        worst = max(worst, max(errs.values()))
    return g, o, worst


def full_shape_step(cfg, w, steps, seed, masked=False, emulate=False, n=None):
    """Run `steps` chunks of n frames through the oracle, the GPU (eager, stage by stage) and,
    for logit-sensitive weights, the bf16-storage emulation; compare the last step (memory
    full) stage by stage.  Returns the GPU stream."""
    n = n or cfg.t_new
    g = H().GpuStream(cfg, w)
    o = O.OracleStream(cfg, w)
    e = O.emulate_bf16_storage(cfg, w) if emulate else None
    for i in range(steps):
        feats = make_features(cfg, n, first_frame=n * i, seed=seed, masked=masked)
        last = i == steps - 1
        o.push(n)
        _, ost = o.step(feats)
        est = None
        if e is not None:
            e.push(n)
            _, est = e.step(feats)
        _, gst = g.step(feats, stages=last)
    compare_step(cfg, ost, gst, TOL[cfg.dtype], tag=f"step {steps - 1}: ", est=est)
    if cfg.dtype == "bf16" and not cfg.win_h:
        fids = o.mem.window() + list(range(o.mem.cur_first, o.mem.next_id))
        check_attention_kernel(g, cfg, gst["layers"][-1], cfg.layers - 1, fids, TOL["bf16"], tag=f"step {steps - 1}: ")
    return g


# ---------------------------------------------------------------- soft split / composite

@pytest.mark.parametrize("name", ["C1", "C3", "C2"])
def test_soft_split_bit_exact(name):
    from paper_2403_16161_b200 import vi
    cfg = CONFIGS[name]
    ctx = vi.Context.from_synth(cfg)
    n = cfg.t_new
    feats = make_features(cfg, n, seed=11)
    f = H().tdev(feats, cfg.dtype)
    out = torch.empty(n, cfg.tokens, cfg.patch_dim, dtype=H().tdtype(cfg), device="cuda")
    ctx.soft_split(f, n, out, 0)
    ctx.sync()
    ref = O.soft_split(feats, cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
    assert np.array_equal(out.float().cpu().numpy().astype(np.float64), ref)


@pytest.mark.parametrize("name", ["C1", "C3", "C2"])
def test_soft_composite_and_identity(name):
    from paper_2403_16161_b200 import vi
    cfg = CONFIGS[name]
    ctx = vi.Context.from_synth(cfg)
    n = cfg.t_new
    dt = H().tdtype(cfg)
    g = (cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
    yp = rng_for(3, "yp").standard_normal((n, cfg.tokens, cfg.patch_dim)).astype(np.float32)
    yp = round_bf16(yp) if cfg.dtype == "bf16" else yp
    out = torch.empty(n, cfg.feat_h, cfg.feat_w, cfg.feat_c, dtype=dt, device="cuda")
    ctx.soft_composite(H().tdev(yp, cfg.dtype), n, out, 0)
    ctx.sync()
    ref = O.soft_composite(yp, cfg.feat_h, cfg.feat_w, cfg.feat_c, *g)
    assert_close(out, ref, 2 ** -8 if cfg.dtype == "bf16" else 1e-6, "composite")
    # identity: composite(split(x)) == x bit-exactly (<= 9 exact copies, exact division)
    feats = make_features(cfg, n, seed=12)
    f = H().tdev(feats, cfg.dtype)
    tok = torch.empty(n, cfg.tokens, cfg.patch_dim, dtype=dt, device="cuda")
    ctx.soft_split(f, n, tok, 0)
    ctx.soft_composite(tok, n, out, 0)
    ctx.sync()
    if cfg.dtype == "bf16":
        assert torch.equal(out, f)
    else:
        np.testing.assert_allclose(out.cpu().numpy(), feats, rtol=2.5e-7, atol=0)


# ---------------------------------------------------------------- fp32 path (configs[0])

def test_c1_fp32_stream_per_stage():
    """BASELINE configs[0]: 1 block, 24 tokens/frame, 1 new frame + 3-frame memory,
    fp32 end to end; 7 steps wrap the 4-slot ring twice."""
    cfg = CONFIGS["C1"]
    w = make_weights(cfg, seed=0)
    _, _, worst = run_pair(cfg, w, steps=7)
    assert worst <= 1e-4


def test_c1_fp32_sensitive_two_layers():
    cfg = CONFIGS["C1"].replace(layers=2)
    w = make_weights(cfg, seed=1, variant="sensitive")
    run_pair(cfg, w, steps=5)


def test_c1_f3n_fp32():
    cfg = CONFIGS["C1"].replace(ffn_kind=1, ffn_hidden=49 * 4, layers=2)
    w = make_weights(cfg, seed=2, variant="sensitive")
    run_pair(cfg, w, steps=4)


def test_I1_causal_replay_through_abi():
    """T=1 steps from an empty memory == one block-causal joint pass (north_star check)."""
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=5)
    w = make_weights(cfg, seed=3, variant="sensitive")
    feats = make_features(cfg, 5, seed=3)
    joint = O.joint_forward(feats, w, cfg, mode="causal")
    g = H().GpuStream(cfg, w)
    for i in range(5):
        out, _ = g.step(feats[i:i + 1], stages=False)
        assert_close(out[0], joint["out"][i], 1e-4, f"I1 frame {i}")


def test_I2_refine_commit_through_abi():
    """Committing a bidirectional joint pass's K/V for t-M..t-1 makes the memory step on
    frame t reproduce that pass's frame-t output (vi_refine_commit path, Eq. 4)."""
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=3)
    w = make_weights(cfg, seed=4, variant="sensitive")
    feats = make_features(cfg, 4, seed=4)
    joint = O.joint_forward(feats, w, cfg, mode="full")
    g = H().GpuStream(cfg, w)
    for i in range(3):
        g.step(feats[i:i + 1], stages=False)
    for i in range(3):
        K = np.stack([joint["k"][l][i] for l in range(cfg.layers)]).astype(np.float32)
        V = np.stack([joint["v"][l][i] for l in range(cfg.layers)]).astype(np.float32)
        assert g.ctx.commit(i, K, V) == 0                       # host payload
    out, _ = g.step(feats[3:4], stages=False)
    _, ref, _ = g.ctx.state()
    assert sum(ref) == 3
    assert_close(out[0], joint["out"][3], 1e-4, "I2")


def test_commit_rows_land_in_slab_and_device_payload():
    cfg = CONFIGS["C1"].replace(mem_frames=3)
    w = make_weights(cfg, seed=5)
    g = H().GpuStream(cfg, w)
    for i in range(3):
        g.step(make_features(cfg, 1, first_frame=i, seed=5), stages=False)
    k, v = make_kv(cfg, 9, 1)
    kd, vd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    assert g.ctx.commit(1, kd, vd) == 0                            # device payload
    assert g.ctx.commit(2, kd, vd) == g.vi.VI_OK
    assert g.ctx.evict(2) == 0                                     # evicted before apply: dropped
    g.step(make_features(cfg, 1, first_frame=3, seed=5), stages=False)
    gk, gv = g.kv(0, 1 % g.ctx.S)
    assert torch.equal(gk.cpu(), torch.from_numpy(k[0])) and torch.equal(gv.cpu(), torch.from_numpy(v[0]))
    sid, ref, mask = g.ctx.state()
    assert ref[1] == 1 and sid[2] == -1


def test_kv_memory_rows_match_oracle():
    cfg = CONFIGS["C1"].replace(layers=2)
    w = make_weights(cfg, seed=6, variant="sensitive")
    g, o, _ = run_pair(cfg, w, steps=5)
    for fid in o.mem.window() + [o.mem.cur_first]:
        for l in range(cfg.layers):
            K, V = o.frame_kv(l, fid)
            gk, gv = g.kv(l, fid % g.ctx.S)
            assert_close(gk, K, 1e-4, f"K l{l} f{fid}")
            assert_close(gv, V, 1e-4, f"V l{l} f{fid}")


def test_protocol_errors():
    from paper_2403_16161_b200 import vi
    cfg = CONFIGS["C1"]
    g = H().GpuStream(cfg, make_weights(cfg))
    x = g.x
    with pytest.raises(vi.ViError) as e:
        g.ctx.memory_step(0, x, x)                  # no push yet
    assert e.value.status == vi.VI_E_PROTOCOL
    g.ctx.push(1)
    with pytest.raises(vi.ViError) as e:
        g.ctx.memory_step(1, x, x)                  # out of order
    assert e.value.status == vi.VI_E_PROTOCOL
    assert g.ctx.evict(0) == vi.VI_E_PROTOCOL        # current chunk, step not finished
    assert g.ctx.commit(5, np.zeros(1, np.float32), np.zeros(1, np.float32)) == vi.VI_E_PROTOCOL
    with pytest.raises(vi.ViError) as e:
        g.ctx.push(2)                               # n > max_new_frames
    assert e.value.status == vi.VI_E_ARG


# ---------------------------------------------------------------- bf16 tensor-core path

def test_c3s_bf16_stream_per_stage():
    """Reduced FuseFormer shape (2 blocks, 180 tokens/frame, T=2, M=3): several 128-row
    tiles with ragged tails, F3N, split-KV attention; 5 steps wrap the 5-slot ring."""
    cfg = CONFIGS["C3S"]
    w = make_weights(cfg, seed=0)
    _, _, worst = run_pair(cfg, w, steps=5)
    assert worst <= 2e-2


def test_c3s_bf16_sensitive_and_ragged_chunks():
    cfg = CONFIGS["C3S"].replace(t_new=3)
    w = make_weights(cfg, seed=1, variant="sensitive")
    run_pair(cfg, w, steps=5, ns=[3, 1, 2, 3, 1], emulate=True)


def test_c3s_bf16_sharp_logits_online_softmax():
    cfg = CONFIGS["C3S"].replace(layers=1)
    w = make_weights(cfg, seed=2, variant="sharp")
    run_pair(cfg, w, steps=4, emulate=True)


def test_c2_shape_headdim64_mlp():
    cfg = CONFIGS["C2"].replace(layers=1, mem_frames=2, t_new=2, feat_h=30, feat_w=54)
    w = make_weights(cfg, seed=3, variant="sensitive")
    run_pair(cfg, w, steps=3, emulate=True)


def test_bf16_kv_rows_and_determinism():
    cfg = CONFIGS["C3S"].replace(layers=1)
    w = make_weights(cfg, seed=4, variant="sensitive")
    g1, o, _ = run_pair(cfg, w, steps=3, emulate=True)
    for fid in o.mem.window() + list(range(o.mem.cur_first, o.mem.next_id)):
        K, V = o.frame_kv(0, fid)
        gk, gv = g1.kv(0, fid % g1.ctx.S)
        assert_close(gk, K, 2e-2, f"K f{fid}")
        assert_close(gv, V, 2e-2, f"V f{fid}")
    # two contexts on the same inputs are bitwise identical (no atomics)
    g1b, g2 = H().GpuStream(cfg, w), H().GpuStream(cfg, w)
    for i in range(3):
        feats = make_features(cfg, cfg.t_new, first_frame=i * cfg.t_new, seed=0)
        a, _ = g1b.step(feats, stages=False)
        b, _ = g2.step(feats, stages=False)
        assert torch.equal(a, b)


def test_run_step_host_buffers_equal_device_path():
    cfg = CONFIGS["C3S"].replace(layers=1)
    w = make_weights(cfg, seed=5)
    g = H().GpuStream(cfg, w)
    from paper_2403_16161_b200 import vi
    c2 = vi.Context.from_synth(cfg)
    c2.set_weights(w)
    for i in range(3):
        feats = make_features(cfg, cfg.t_new, first_frame=i * cfg.t_new, seed=7)
        ref, _ = g.step(feats, stages=False)
        host_in = torch.from_numpy(feats).to(torch.bfloat16).contiguous()
        host_out = torch.empty_like(host_in)
        c2.run_step(host_in, cfg.t_new, host_out)
        assert torch.equal(host_out, ref.cpu())


def test_c3_full_shape_step():
    """The metric config (BASELINE configs[2]) at full size: 3 steps of 5 frames fill the
    10-frame memory, the 4th step (3600 queries x 10800 keys) is compared stage by stage."""
    cfg = CONFIGS["C3"].replace(layers=2)
    g = full_shape_step(cfg, make_weights(cfg, seed=0), 4, seed=0)
    assert g.ctx.state()[2] == (1 << 15) - 1


def test_c3t1_full_shape_step():
    """The paper's own Eq. 3 mode at the metric shape (configs[2] with ONE new frame per step,
    P:121 "narrowing the prediction pipeline to only one frame"; C5's online model): 11 steps
    fill the 10-frame memory, the 11th (720 queries x 7920 keys, the small-chunk attention
    path) is compared stage by stage."""
    cfg = CONFIGS["C3T1"].replace(layers=2)
    g = full_shape_step(cfg, make_weights(cfg, seed=30), 11, seed=30)
    assert g.ctx.state()[2] == (1 << 11) - 1


def test_c3t1_full_shape_sensitive():
    """C3T1 with logit-sensitive weights (memory-dependent output): 1 block, 11 steps."""
    cfg = CONFIGS["C3T1"].replace(layers=1)
    full_shape_step(cfg, make_weights(cfg, seed=31, variant="sensitive"), 11, seed=31, emulate=True)


def test_c3_graph_replayed_8_block_step():
    """The step bench.py times: BASELINE configs[2] in full (8 blocks), vi_run_step replaying
    one captured CUDA graph per (ring state, buffers).  Its outputs are compared with the
    oracle after the memory is full, and are bitwise equal to the eager path (vi_soft_split /
    vi_memory_step x 8 / vi_soft_composite launched one by one)."""
    from paper_2403_16161_b200 import vi
    cfg = CONFIGS["C3"]
    w = make_weights(cfg, seed=32)
    ctx = vi.Context.from_synth(cfg)
    ctx.set_weights(w)
    eager = H().GpuStream(cfg, w)
    o = O.OracleStream(cfg, w)
    for i in range(4):
        feats = make_features(cfg, 5, first_frame=5 * i, seed=32)
        o.push(5)
        ref, _ = o.step(feats)
        f = torch.from_numpy(feats).to(torch.bfloat16).cuda()
        out = torch.empty_like(f)
        ctx.run_step(f, 5, out)
        ctx.sync()
        ge, _ = eager.step(feats, stages=False)
        assert torch.equal(out, ge), f"step {i}: graph replay differs from the eager launches"
        if i >= 2:                   # memory full from step 2 on (15 slots)
            assert_close(out, ref, 2e-2, f"step {i} out")
    assert ctx.state()[2] == (1 << 15) - 1
    # a replay of an already captured graph (same ring state and buffers) is deterministic too
    assert ctx.launches() > 0


def test_c3t1_run_step_equals_per_layer_calls():
    """One frame per step (C3T1, 3 blocks): vi_run_step's graph, in which the split-K
    reductions of the embedding and of FFN2 also write the next block's LN1, is bitwise equal
    to the public per-layer calls (vi_soft_split / vi_memory_step / vi_soft_composite, no LN1
    fusion across calls) on every step, and matches the oracle once the memory is full."""
    from paper_2403_16161_b200 import vi
    cfg = CONFIGS["C3T1"].replace(layers=3)
    w = make_weights(cfg, seed=35)
    ctx = vi.Context.from_synth(cfg)
    ctx.set_weights(w)
    eager = H().GpuStream(cfg, w)
    o = O.OracleStream(cfg, w)
    for i in range(12):
        feats = make_features(cfg, 1, first_frame=i, seed=35)
        f = torch.from_numpy(feats).to(torch.bfloat16).cuda()
        out = torch.empty_like(f)
        ctx.run_step(f, 1, out)
        ctx.sync()
        ge, _ = eager.step(feats, stages=False)
        assert torch.equal(out, ge), f"step {i}: vi_run_step differs from the per-layer calls"
        o.push(1)
        ref, _ = o.step(feats)
        if i >= 10:                  # memory full (10 frames + the new one)
            assert_close(out, ref, 2e-2, f"step {i} out")


def test_positional_embedding_bf16():
    """pos_embed = 1 (reading Q8: an additive [P, D] table at the split, never temporal): the
    oracle adds it in embed(); the GPU's embed GEMM epilogue adds it per token row."""
    cfg = CONFIGS["C3S"].replace(layers=1, pos_embed=1)
    w = make_weights(cfg, seed=33, variant="sensitive")
    assert w["pos"] is not None
    run_pair(cfg, w, steps=3, emulate=True)


def test_positional_embedding_fp32():
    cfg = CONFIGS["C1"].replace(pos_embed=1)
    w = make_weights(cfg, seed=34)
    run_pair(cfg, w, steps=4)


def _run_steps(cfg, w, steps, seed):
    from paper_2403_16161_b200 import vi
    ctx = vi.Context.from_synth(cfg)
    ctx.set_weights(w)
    outs = []
    for i in range(steps):
        f = torch.from_numpy(make_features(cfg, cfg.t_new, first_frame=i * cfg.t_new, seed=seed)).to(torch.bfloat16).cuda()
        out = torch.empty_like(f)
        ctx.run_step(f, cfg.t_new, out)
        ctx.sync()                     # device buffers: run_step only enqueues on the context's stream
        outs.append(out.float())
    ctx.close()
    return outs


@pytest.mark.parametrize("env", [{"VI_SK_UNIT_COST": "0"}, {"VI_SK_UNIT_COST": "400"},
                                 {"VI_SK_UNIT_COST": "96", "VI_SK_TAIL_W": "6"}, {"VI_SK_TAIL_W": "40"}])
def test_stream_k_partition_invariance(env, monkeypatch):
    """The stream-K attention at the C3 shape under other work splits (unit-start cost, tail
    weight): different CTA boundaries, pieces, owners and merge orders (a split that once hung
    is among them) give the default split's output up to merge rounding.  The default split is
    the one test_c3_full_shape_step pins to the oracle."""
    cfg = CONFIGS["C3"].replace(layers=1)
    w = make_weights(cfg, seed=21)
    ref = _run_steps(cfg, w, 4, seed=21)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got = _run_steps(cfg, w, 4, seed=21)
    for i in (2, 3):           # memory full: every unit spans 85 key tiles
        scale = ref[i].abs().max().item()
        err = (got[i] - ref[i]).abs().max().item() / scale
        assert err < 1e-2, f"step {i}: {err:.3g} under {env}"


@pytest.mark.parametrize("split", ["1", "3"])
def test_window_split_invariance(split, monkeypatch):
    """Window attention (C4 shape, 1 block) with 1 or 3 CTAs per (head, window, query pair)
    unit instead of the default 2: same output up to merge rounding."""
    cfg = CONFIGS["C4"].replace(layers=1)
    w = make_weights(cfg, seed=22)
    ref = _run_steps(cfg, w, 4, seed=22)
    monkeypatch.setenv("VI_WIN_SPLIT", split)
    got = _run_steps(cfg, w, 4, seed=22)
    scale = ref[3].abs().max().item()
    err = (got[3] - ref[3]).abs().max().item() / scale
    assert err < 1e-2, f"window split {split}: {err:.3g}"


def test_splitk_small_m_gemms_both_paths(monkeypatch):
    """One new frame per step (C3T1 shape, M = 720 rows): the output projection and FFN2 run
    as split-K partials + one deterministic reduction (fused with LN2 after the projection).
    The unsplit GEMMs (VI_SPLITK=0) give the same output up to accumulation order, and the
    split run is pinned to the oracle by test_c3t1_full_shape_step; here the unsplit one is."""
    cfg = CONFIGS["C3T1"].replace(layers=1)
    w = make_weights(cfg, seed=24)
    ref = _run_steps(cfg, w, 3, seed=24)
    again = _run_steps(cfg, w, 3, seed=24)
    for a, b in zip(ref, again):
        assert torch.equal(a, b), "split-K path is not deterministic"
    monkeypatch.setenv("VI_SPLITK", "0")
    got = _run_steps(cfg, w, 3, seed=24)
    for i in range(3):
        scale = ref[i].abs().max().item()
        err = (got[i] - ref[i]).abs().max().item() / scale
        assert err < 1e-2, f"step {i}: split vs unsplit {err:.3g}"
    full_shape_step(cfg, w, 11, seed=24)


def test_stream_k_headdim64_c3_shape():
    """Head dim 64 through the stream-K kernel (attn_sk2<64>): the C3 token grid (3600
    queries x 10800 keys, 60 units) with D = 256; the 4th step compared stage by stage."""
    cfg = CONFIGS["C3"].replace(layers=1, d_model=256)
    full_shape_step(cfg, make_weights(cfg, seed=23), 4, seed=23)


def test_c2_full_shape_step():
    """BASELINE configs[1] at full size (STTN-shaped: 8 blocks, 4 heads of d 64, D 256,
    5x9-cell patches of a 60x108x256 map -> 144 tokens/frame, MLP-GELU 1024, T=5, M=10):
    3 steps fill the memory, the 4th (720 queries x 2160 keys) is compared stage by stage,
    on masked frames."""
    cfg = CONFIGS["C2"]
    g = full_shape_step(cfg, make_weights(cfg, seed=0, variant="sensitive"), 4, seed=0, masked=True, emulate=True)
    assert g.ctx.state()[2] == (1 << 15) - 1


def test_reference_frames_bf16():
    """Eq. 3's reference frames M_{1,r}^{f-1} (reading Q12): span 2, a reference every 3rd
    frame, 2 reference slots; 10 one-frame steps move frames 0, 3, 6 into reference slots
    (0 leaves again at frame 9) -- ring state bit-exact, every stage within the bf16 bar."""
    cfg = CONFIGS["C3S"].replace(layers=2, t_new=1, mem_frames=2, ref_rate=3, max_refs=2)
    w = make_weights(cfg, seed=8, variant="sensitive")
    run_pair(cfg, w, steps=10, masked="moving", emulate=True)


def test_reference_frames_fp32_and_refine_commit():
    """The SIMT fp32 path with references, a refine commit of a reference frame and an explicit
    eviction of another one."""
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=2, ref_rate=2, max_refs=2)
    w = make_weights(cfg, seed=9, variant="sensitive")
    g = H().GpuStream(cfg, w)
    o = O.OracleStream(cfg, w)
    for i in range(9):
        feats = make_features(cfg, 1, first_frame=i, seed=9)
        if i == 6:      # frame 2 is a reference by now: commit it; evict reference 0... (0 left at 6)
            K, V = make_kv(cfg, 11, 2)
            assert g.ctx.commit(2, K, V) == o.commit(2, K, V) == 0
        if i == 8:
            assert g.ctx.evict(4) == o.evict(4) == 0
        assert g.ctx.push(1) == o.push(1)
        ref, _ = o.step(feats)
        out = torch.empty(1, cfg.feat_h, cfg.feat_w, cfg.feat_c, dtype=torch.float32, device="cuda")
        xg = g.x[: cfg.tokens]
        f = H().tdev(feats, cfg.dtype)
        g.ctx.soft_split(f, 1, xg, 1)
        for l in range(cfg.layers):
            g.ctx.memory_step(l, xg, xg)
        g.ctx.soft_composite(xg, 1, out, 1)
        g.ctx.sync()
        assert g.ctx.state() == tuple(o.mem.state()), f"step {i}"
        assert_close(out, ref, 1e-4, f"step {i} out")


# ---------------------------------------------------------------- window attention (configs[3])

def test_window_attention_c3s_ragged():
    """Window attention (E2FGVI-shaped) on the reduced map: 10 x 18 tokens in 5 x 6 windows
    (30 tokens, padded to 32 rows), ragged chunks, the memory wraps; every stage vs the oracle."""
    cfg = CONFIGS["C3S"].replace(t_new=3, win_h=5, win_w=6)
    w = make_weights(cfg, seed=12, variant="sensitive")
    run_pair(cfg, w, steps=5, ns=[3, 1, 2, 3, 2], emulate=True)


def test_window_attention_with_reference_frames():
    """Window attention over a memory with reference frames: a reference move copies the slot's
    rows inside every window's key region (window-major memory); 10 one-frame steps."""
    cfg = CONFIGS["C3S"].replace(layers=2, t_new=1, mem_frames=2, ref_rate=3, max_refs=2, win_h=5, win_w=6)
    w = make_weights(cfg, seed=14, variant="sensitive")
    run_pair(cfg, w, steps=10, masked="moving", emulate=True)


def test_window_attention_c4_full_shape_step():
    """BASELINE configs[3] shape (2 of its 16 blocks): 720 tokens/frame in 16 windows of 5 x 9,
    5 new frames over a 10-frame memory; the 4th step compared stage by stage."""
    cfg = CONFIGS["C4"].replace(layers=2)
    full_shape_step(cfg, make_weights(cfg, seed=13, variant="sensitive"), 4, seed=13, emulate=True)


def test_run_step_async_pipelined_equals_run_step():
    """vi_run_step_async (copies on a second stream, two staging slots) == vi_run_step, bitwise,
    over a sequence long enough to reuse both slots and wrap the ring."""
    cfg = CONFIGS["C3S"].replace(layers=1)
    w = make_weights(cfg, seed=14)
    from paper_2403_16161_b200 import vi
    a, b = vi.Context.from_synth(cfg), vi.Context.from_synth(cfg)
    for c in (a, b):
        c.set_weights(w)
    steps = 7
    host_in = [torch.from_numpy(make_features(cfg, cfg.t_new, first_frame=i * cfg.t_new, seed=14)).to(
        torch.bfloat16).contiguous().pin_memory() for i in range(steps)]
    outs_a = [torch.empty_like(h).pin_memory() for h in host_in]
    outs_b = [torch.empty_like(h) for h in host_in]
    for i in range(steps):
        a.run_step_async(host_in[i], cfg.t_new, outs_a[i])
        b.run_step(host_in[i], cfg.t_new, outs_b[i])
    a.sync()
    for i in range(steps):
        assert torch.equal(outs_a[i], outs_b[i]), f"step {i}"
    assert a.state() == b.state()
