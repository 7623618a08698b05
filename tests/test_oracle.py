"""Pins of the fp64 oracle against things other than itself (no GPU needed).

Each test names what it pins against: a torch library routine (fp64, CPU), a worked
example printed in SPEC.md / BASELINE.json (tests/golden/), a closed form, brute force,
or an exact invariant of the memory method (I1 causal replay, I2 refine equivalence).
"""
import json
import math
import os
import random

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

import oracle
from oracle import vi_oracle as O
from vi_synth import CONFIGS, make_features, make_weights, round_bf16, rng_for

GOLD = os.path.join(os.path.dirname(__file__), "golden")
torch.set_default_dtype(torch.float64)


def spec():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        return json.load(f)


def tiny(**kw):
    base = CONFIGS["C1"].replace(**kw)
    return base


# ---------------------------------------------------------------- soft split / composite

def _unfold_ref(F, kh, kw, sh, sw, ph, pw):
    """torch.nn.functional.unfold, reordered from (c, ky, kx) to (ky, kx, c)."""
    T, H, W, C = F.shape
    x = torch.from_numpy(np.ascontiguousarray(F.transpose(0, 3, 1, 2))).double()
    u = Fn.unfold(x, (kh, kw), padding=(ph, pw), stride=(sh, sw))      # [T, C*kh*kw, L]
    L = u.shape[-1]
    u = u.reshape(T, C, kh * kw, L).permute(0, 3, 2, 1).reshape(T, L, kh * kw * C)
    return u.numpy()


@pytest.mark.parametrize("name", ["C1", "C3S", "C2"])
def test_soft_split_matches_torch_unfold(name):
    cfg = CONFIGS[name]
    F = make_features(cfg.replace(feat_c=min(cfg.feat_c, 8)), 2, seed=3).astype(np.float64)
    g = (cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
    got = O.soft_split(F, *g)
    assert np.array_equal(got, _unfold_ref(F, *g))   # bit-exact: pure copies


def test_soft_split_brute_force_index_formula():
    rng = rng_for(1, "split-bf")
    F = rng.standard_normal((1, 5, 7, 3))
    got = O.soft_split(F, 3, 3, 2, 2, 1, 1)
    oh, ow = O.out_size(5, 3, 2, 1), O.out_size(7, 3, 2, 1)
    for tok in range(oh * ow):
        oy, ox = divmod(tok, ow)
        for j in range(27):
            ky, rem = divmod(j, 9)
            kx, c = divmod(rem, 3)
            y, x = oy * 2 - 1 + ky, ox * 2 - 1 + kx
            want = F[0, y, x, c] if (0 <= y < 5 and 0 <= x < 7) else 0.0
            assert got[0, tok, j] == want


def test_token_counts_spec_and_baseline():
    for c in spec()["token_count"]["cases"]:
        kh = c.get("kh", c.get("k")); kw = c.get("kw", c.get("k"))
        sh = c.get("sh", c.get("s")); sw = c.get("sw", c.get("s"))
        n = O.out_size(c["h"], kh, sh, c["p"]) * O.out_size(c["w"], kw, sw, c["p"])
        assert n == c["tokens"], c
    assert CONFIGS["C1"].tokens == 24 and CONFIGS["C3"].tokens == 720 and CONFIGS["C2"].tokens == 144


def test_coverage_spec_example_and_fold_of_ones():
    c = spec()["coverage"]
    cnt = O.coverage(c["h"], c["w"], c["k"], c["k"], c["s"], c["s"], c["p"], c["p"])
    assert cnt[0, 0] == c["corner"] and cnt[3, 3] == c["interior"]
    for name in ["C1", "C3", "C2"]:
        cfg = CONFIGS[name]
        ones = torch.ones(1, cfg.kh * cfg.kw, cfg.tokens)
        ref = Fn.fold(ones, (cfg.feat_h, cfg.feat_w), (cfg.kh, cfg.kw), padding=(cfg.ph, cfg.pw),
                      stride=(cfg.sh, cfg.sw))[0, 0].numpy()
        cov = O.coverage(cfg.feat_h, cfg.feat_w, cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
        assert np.array_equal(cov, ref.astype(np.int64))
        assert cov.min() >= 1


@pytest.mark.parametrize("name", ["C1", "C3S"])
def test_soft_composite_matches_torch_fold(name):
    cfg = CONFIGS[name]
    C = 5
    rng = rng_for(2, "comp")
    Yp = rng.standard_normal((2, cfg.tokens, cfg.kh * cfg.kw * C))
    got = O.soft_composite(Yp, cfg.feat_h, cfg.feat_w, C, cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
    y = torch.from_numpy(Yp).reshape(2, cfg.tokens, cfg.kh * cfg.kw, C).permute(0, 3, 2, 1)
    y = y.reshape(2, C * cfg.kh * cfg.kw, cfg.tokens)
    kw = dict(output_size=(cfg.feat_h, cfg.feat_w), kernel_size=(cfg.kh, cfg.kw),
              padding=(cfg.ph, cfg.pw), stride=(cfg.sh, cfg.sw))
    ref = (Fn.fold(y, **kw) / Fn.fold(torch.ones_like(y), **kw)).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-14, atol=1e-14)


def test_split_then_composite_is_identity():
    """SPEC S:229 / BJ north_star: identity projections give back the input.
    Exact for bf16-representable values (<= 9 copies sum exactly), <= 2 ulp otherwise."""
    cfg = CONFIGS["C3S"]
    g = (cfg.kh, cfg.kw, cfg.sh, cfg.sw, cfg.ph, cfg.pw)
    F = make_features(cfg.replace(feat_c=16), 2, seed=5)           # bf16-representable
    back = O.soft_composite(O.soft_split(F, *g), cfg.feat_h, cfg.feat_w, 16, *g)
    assert np.array_equal(back, F.astype(np.float64))
    G = rng_for(5, "id64").standard_normal(F.shape)
    back = O.soft_composite(O.soft_split(G, *g), cfg.feat_h, cfg.feat_w, 16, *g)
    np.testing.assert_allclose(back, G, rtol=4.5e-16, atol=0)


def test_uncovered_cell_is_config_error():
    Yp = np.zeros((1, 1, 4))
    with pytest.raises(ValueError):
        O.soft_composite(Yp, 3, 3, 1, 2, 2, 3, 3, 0, 0)   # 2x2 window, stride 3: cells uncovered


# ---------------------------------------------------------------- numeric primitives

def test_matmul_spec_example():
    m = spec()["matmul"]
    got = O.linear(np.array(m["a"], float), np.array(m["b"], float).T, None)
    assert np.array_equal(got, np.array(m["out"], float))


def test_softmax_spec_examples():
    for c in spec()["softmax"]["cases"]:
        x = np.array([math.log(2) if v == "ln2" else v for v in c["in"]], float)
        want = np.array([eval(v) if isinstance(v, str) else v for v in c["out"]], float)
        np.testing.assert_allclose(O.softmax_rows(x[None])[0], want, rtol=1e-15)
    S = rng_for(0, "sm").standard_normal((50, 300)) * 30
    assert np.abs(O.softmax_rows(S).sum(-1) - 1).max() < 1e-12


def test_layer_norm_spec_examples_and_torch():
    for c in spec()["layer_norm"]["cases"]:
        x = np.array(c["in"], float)
        g = np.full_like(x, c.get("gain", 1.0))
        b = np.array(c["bias"], float) if "bias" in c else np.zeros_like(x)
        np.testing.assert_allclose(O.layer_norm(x[None], g, b)[0], c["out"], atol=c.get("atol", 1e-12))
    rng = rng_for(0, "ln")
    x, g, b = rng.standard_normal((7, 64)) * 3 + 1, rng.standard_normal(64), rng.standard_normal(64)
    ref = Fn.layer_norm(torch.from_numpy(x), (64,), torch.from_numpy(g), torch.from_numpy(b), eps=1e-5)
    np.testing.assert_allclose(O.layer_norm(x, g, b), ref.numpy(), rtol=1e-12, atol=1e-12)
    y = O.layer_norm(x, np.ones(64), np.zeros(64))
    assert np.abs(y.mean(-1)).max() < 1e-12 and np.abs(y.var(-1) * (1 + 1e-5 / x.var(-1)) - 1).max() < 1e-9


def test_gelu_matches_torch_exact_erf():
    x = np.linspace(-8, 8, 2001)
    np.testing.assert_allclose(O.gelu(x), Fn.gelu(torch.from_numpy(x)).numpy(), rtol=1e-13, atol=1e-15)
    assert O.gelu(np.array([0.0]))[0] == 0.0


def _attn_brute(Q, K, V, heads):
    nq, D = Q.shape
    d = D // heads
    out = np.zeros((nq, D))
    for h in range(heads):
        for i in range(nq):
            s = [sum(Q[i, h * d + t] * K[j, h * d + t] for t in range(d)) / math.sqrt(d) for j in range(len(K))]
            m = max(s)
            e = [math.exp(v - m) for v in s]
            z = sum(e)
            for t in range(d):
                out[i, h * d + t] = sum(e[j] / z * V[j, h * d + t] for j in range(len(K)))
    return out


def test_attention_brute_force_and_torch_sdpa():
    rng = rng_for(0, "attn")
    Q, K, V = rng.standard_normal((4, 8)), rng.standard_normal((7, 8)), rng.standard_normal((7, 8))
    got = O.attention(Q, K, V, heads=2)
    np.testing.assert_allclose(got, _attn_brute(Q, K, V, 2), rtol=1e-13, atol=1e-14)
    Q, K, V = rng.standard_normal((30, 64)), rng.standard_normal((90, 64)), rng.standard_normal((90, 64))
    got = O.attention(Q, K, V, heads=4, row_chunk=7)
    t = lambda a: torch.from_numpy(a).reshape(a.shape[0], 4, 16).transpose(0, 1)
    ref = Fn.scaled_dot_product_attention(t(Q), t(K), t(V)).transpose(0, 1).reshape(30, 64)
    np.testing.assert_allclose(got, ref.numpy(), rtol=1e-12, atol=1e-13)


def test_attention_single_key_and_permutation_invariance():
    rng = rng_for(1, "attn2")
    Q, K, V = rng.standard_normal((5, 8)), rng.standard_normal((1, 8)), rng.standard_normal((1, 8))
    np.testing.assert_allclose(O.attention(Q, K, V, 2), np.repeat(V, 5, 0), rtol=1e-15)
    K, V = rng.standard_normal((40, 8)), rng.standard_normal((40, 8))
    perm = rng.permutation(40)
    np.testing.assert_allclose(O.attention(Q, K, V, 2), O.attention(Q, K[perm], V[perm], 2), rtol=1e-12)
    o, lse = O.attention(Q, K, V, 2, return_lse=True)
    S = Q[:, :4] @ K[:, :4].T / 2.0
    np.testing.assert_allclose(lse[0], np.log(np.exp(S).sum(-1)), rtol=1e-13)


def test_mac_count_closed_forms():
    m = spec()["score_macs"]
    j, s = m["joint"], m["single_query"]
    assert O.mac_counts(j["P"], 0, j["n"], j["D"]) == j["macs"]
    assert O.mac_counts(s["P"], s["C"], 1, s["D"]) == s["macs"]
    assert O.mac_counts(24, 3, 1, 64) == 147456


# ---------------------------------------------------------------- block vs torch modules

def _torch_block(x_chunk, x_all_ln_src, w, l, cfg, kv_inputs):
    """Pre-norm block assembled from torch.nn modules (fp64): MultiheadAttention with the
    oracle's in/out projections, then LN2 + Linear-GELU-Linear (MLP) with residuals."""
    D = cfg.d_model
    mha = torch.nn.MultiheadAttention(D, cfg.heads, bias=True, batch_first=True)
    with torch.no_grad():
        mha.in_proj_weight.copy_(torch.from_numpy(w["wqkv"][l].astype(np.float64)))
        mha.in_proj_bias.copy_(torch.from_numpy(w["bqkv"][l].astype(np.float64)))
        mha.out_proj.weight.copy_(torch.from_numpy(w["wo"][l].astype(np.float64)))
        mha.out_proj.bias.copy_(torch.from_numpy(w["bo"][l].astype(np.float64)))
    ln = lambda x, g, b: Fn.layer_norm(x, (D,), torch.from_numpy(g[l].astype(np.float64)),
                                        torch.from_numpy(b[l].astype(np.float64)), eps=1e-5)
    xq = torch.from_numpy(x_chunk)
    kv = ln(torch.from_numpy(kv_inputs), w["ln1_g"], w["ln1_b"])
    a, _ = mha(ln(xq, w["ln1_g"], w["ln1_b"])[None], kv[None], kv[None], need_weights=False)
    x1 = xq + a[0]
    h2 = ln(x1, w["ln2_g"], w["ln2_b"])
    u = Fn.linear(h2, torch.from_numpy(w["w1"][l].astype(np.float64)), torch.from_numpy(w["b1"][l].astype(np.float64)))
    y = Fn.linear(Fn.gelu(u), torch.from_numpy(w["w2"][l].astype(np.float64)), torch.from_numpy(w["b2"][l].astype(np.float64)))
    return (x1 + y).detach().numpy()


def test_block_memory_matches_torch_modules():
    cfg = CONFIGS["C1"]
    w = make_weights(cfg, seed=0, variant="sensitive")
    rng = rng_for(0, "blk")
    x_mem = rng.standard_normal((3 * cfg.tokens, cfg.d_model))
    x_new = rng.standard_normal((cfg.tokens, cfg.d_model))
    mem = []
    for j in range(3):
        _, _, K, V = O.qkv(x_mem[j * 24:(j + 1) * 24], w, 0, cfg)
        mem.append((K, V))
    got, _ = O.block_memory(x_new, mem, w, 0, cfg, 1)
    ref = _torch_block(x_new, None, w, 0, cfg, np.concatenate([x_mem, x_new]))
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-11)


def test_encoder_layer_equivalence_first_frame():
    """Empty memory => the block is a plain pre-norm ViT encoder layer."""
    cfg = CONFIGS["C1"]
    w = make_weights(cfg, seed=1, variant="sensitive")
    layer = torch.nn.TransformerEncoderLayer(cfg.d_model, cfg.heads, cfg.ffn_hidden, dropout=0.0,
                                             activation="gelu", layer_norm_eps=1e-5, batch_first=True,
                                             norm_first=True)
    sd = {"self_attn.in_proj_weight": w["wqkv"][0], "self_attn.in_proj_bias": w["bqkv"][0],
          "self_attn.out_proj.weight": w["wo"][0], "self_attn.out_proj.bias": w["bo"][0],
          "linear1.weight": w["w1"][0], "linear1.bias": w["b1"][0], "linear2.weight": w["w2"][0],
          "linear2.bias": w["b2"][0], "norm1.weight": w["ln1_g"][0], "norm1.bias": w["ln1_b"][0],
          "norm2.weight": w["ln2_g"][0], "norm2.bias": w["ln2_b"][0]}
    layer.load_state_dict({k: torch.from_numpy(v.astype(np.float64)) for k, v in sd.items()})
    layer.eval()
    x = rng_for(2, "enc").standard_normal((cfg.tokens, cfg.d_model))
    got, _ = O.block_memory(x, [], w, 0, cfg, 1)
    with torch.no_grad():
        ref = layer(torch.from_numpy(x)[None])[0].numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-11)


def test_f3n_matches_torch_fold_unfold():
    cfg = CONFIGS["C3S"].replace(ffn_hidden=49 * 3)
    rng = rng_for(3, "f3n")
    u = rng.standard_normal((2, cfg.tokens, 49 * 3))
    got = O.f3n_mix(u, cfg)
    t = torch.from_numpy(u).reshape(2, cfg.tokens, 49, 3).permute(0, 3, 2, 1).reshape(2, 3 * 49, cfg.tokens)
    kw = dict(kernel_size=(7, 7), padding=(3, 3), stride=(3, 3))
    f = Fn.fold(t, (cfg.feat_h, cfg.feat_w), **kw) / Fn.fold(torch.ones_like(t), (cfg.feat_h, cfg.feat_w), **kw)
    r = Fn.unfold(f, **kw).reshape(2, 3, 49, cfg.tokens).permute(0, 3, 2, 1).reshape(2, cfg.tokens, 147)
    np.testing.assert_allclose(got, r.numpy(), rtol=1e-13, atol=1e-14)


def test_f3n_without_overlap_is_plain_mlp():
    """k = s, p = 0: fold o unfold is the identity, so the Fusion-FFN reduces to an MLP."""
    cfg = CONFIGS["C1"].replace(kh=3, kw=3, sh=3, sw=3, ph=0, pw=0, ffn_kind=1, ffn_hidden=9 * 4)
    w = make_weights(cfg, seed=4, variant="sensitive")
    h2 = rng_for(4, "h2").standard_normal((2 * cfg.tokens, cfg.d_model))
    _, g1 = O.ffn(h2, w, 0, cfg, 2)
    _, g0 = O.ffn(h2, w, 0, cfg.replace(ffn_kind=0), 2)
    np.testing.assert_allclose(g1, g0, rtol=1e-15, atol=0)


# ---------------------------------------------------------------- memory invariants

def _stream(cfg, w, feats, n_steps, T):
    s = O.OracleStream(cfg, w)
    outs = []
    for i in range(n_steps):
        s.push(T)
        o, _ = s.step(feats[i * T:(i + 1) * T])
        outs.append(o)
    return s, np.concatenate(outs)


@pytest.mark.parametrize("ffn_kind", [0, 1])
def test_I1_causal_replay_equals_block_causal_joint_pass(ffn_kind):
    """Memory filled from frames 0..t-1 by T=1 steps == one joint pass over 0..t with a
    frame-level causal mask (BASELINE north_star; SPEC S:324 replay oracle)."""
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=6, ffn_kind=ffn_kind,
                                ffn_hidden=(49 * 2 if ffn_kind else 128))
    w = make_weights(cfg, seed=0, variant="sensitive")
    feats = make_features(cfg, 5, seed=0)
    _, outs = _stream(cfg, w, feats, 5, 1)
    joint = O.joint_forward(feats, w, cfg, mode="causal")
    np.testing.assert_allclose(outs, joint["out"], rtol=1e-11, atol=1e-12)


def test_I1_detects_ignored_memory():
    cfg = CONFIGS["C1"].replace(mem_frames=6)
    w = make_weights(cfg, seed=0, variant="sensitive")
    feats = make_features(cfg, 3, seed=0)
    joint = O.joint_forward(feats, w, cfg, mode="causal")
    solo = O.joint_forward(feats[2:3], w, cfg, mode="causal")
    assert O.rel_err(solo["out"][0], joint["out"][2]) > 1e-2


def test_I2_refine_commit_equivalence():
    """Commit the K/V that a bidirectional joint pass over t-M..t gives for t-M..t-1; a
    memory step on frame t then reproduces the joint pass's frame-t output (Eq. 4 reading)."""
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=3)
    w = make_weights(cfg, seed=1, variant="sensitive")
    feats = make_features(cfg, 4, seed=1)
    joint = O.joint_forward(feats, w, cfg, mode="full")
    s = O.OracleStream(cfg, w)
    for i in range(3):
        s.push(1); s.step(feats[i:i + 1])
    for i in range(3):
        K = np.stack([joint["k"][l][i] for l in range(cfg.layers)])
        V = np.stack([joint["v"][l][i] for l in range(cfg.layers)])
        assert s.commit(i, K, V) == O.VI_OK
    s.push(1)
    out, _ = s.step(feats[3:4])
    np.testing.assert_allclose(out[0], joint["out"][3], rtol=1e-11, atol=1e-12)
    s2 = O.OracleStream(cfg, w)                               # control: no commit
    for i in range(4):
        s2.push(1); o2, _ = s2.step(feats[i:i + 1])
    assert O.rel_err(o2[0], joint["out"][3]) > 1e-3


def test_first_frame_equals_single_frame_joint():
    cfg = CONFIGS["C1"].replace(layers=2)
    w = make_weights(cfg, seed=2, variant="sensitive")
    feats = make_features(cfg, 1, seed=2)
    s = O.OracleStream(cfg, w)
    s.push(1)
    out, _ = s.step(feats)
    np.testing.assert_allclose(out, O.joint_forward(feats, w, cfg, "full")["out"], rtol=1e-12, atol=1e-13)


def test_chunk_equals_joint_over_chunk_plus_memory():
    """T=2 chunks, bidirectional inside the chunk (reading Q9): the chunk's rows equal a
    joint pass where each chunk sees itself + everything before it."""
    cfg = CONFIGS["C1"].replace(layers=2, t_new=2, mem_frames=8)
    w = make_weights(cfg, seed=3, variant="sensitive")
    feats = make_features(cfg, 4, seed=3)
    _, outs = _stream(cfg, w, feats, 2, 2)
    # joint reference with a chunk-causal mask built by hand from the torch-free oracle pieces
    n, P = 4, cfg.tokens
    Tp, X = O.embed(feats, w, cfg)
    ch = np.repeat(np.arange(n) // 2, P)
    allowed = ch[None, :] <= ch[:, None]
    for l in range(cfg.layers):
        _, Q, K, V = O.qkv(X, w, l, cfg)
        X = X + O.linear(O.attention(Q, K, V, cfg.heads, allowed=allowed), w["wo"][l], w["bo"][l])
        _, g = O.ffn(O.layer_norm(X, w["ln2_g"][l], w["ln2_b"][l]), w, l, cfg, n)
        X = X + O.linear(g, w["w2"][l], w["b2"][l])
    _, ref = O.compose(X, w, cfg, n)
    np.testing.assert_allclose(outs, ref, rtol=1e-11, atol=1e-12)


def test_window_eviction_limits_context():
    """With span M, frame f sees exactly frames f-M..f-1 (Eq. 3)."""
    cfg = CONFIGS["C1"].replace(mem_frames=2)
    w = make_weights(cfg, seed=5, variant="sensitive")
    feats = make_features(cfg, 5, seed=5)
    s, outs = _stream(cfg, w, feats, 5, 1)
    assert s.mem.window() == [2, 3]
    # changing frame 0 must not change frame 4's output: frame 4 sees 2, 3 whose cached
    # inputs depend on 0 only through 1 ... so instead check frame 3 with frame 0 changed
    f2 = feats.copy(); f2[0] = make_features(cfg, 1, first_frame=99, seed=5)[0]
    _, outs2 = _stream(cfg, w, f2, 5, 1)
    assert not np.allclose(outs2[1], outs[1])   # frame 1 sees 0
    assert not np.allclose(outs2[2], outs[2])   # frame 2 sees 0 directly


def test_causality_future_frames_do_not_change_past():
    cfg = CONFIGS["C1"].replace(mem_frames=3)
    w = make_weights(cfg, seed=6)
    feats = make_features(cfg, 4, seed=6)
    _, a = _stream(cfg, w, feats, 4, 1)
    f2 = feats.copy(); f2[3] += 1.0
    _, b = _stream(cfg, w, f2, 4, 1)
    assert np.array_equal(a[:3], b[:3]) and not np.array_equal(a[3], b[3])


# ---------------------------------------------------------------- ring bookkeeping

def test_ring_goldens():
    with open(os.path.join(GOLD, "ring_trace.json")) as f:
        g = json.load(f)
    m = O.OracleMemory(g["M"], g["T_max"])
    S = g["M"] + g["T_max"]
    for op in g["ops"]:
        if op["op"] == "push":
            first, ev = m.push(op["n"])
            assert first == op["first"] and ev == op["evicted"], op
            _, ref, mask = m.state()
            assert mask == int(op["mask"], 16), (op, hex(mask))
            if "refined_slots" in op:
                assert [i for i in range(S) if ref[i]] == op["refined_slots"]
        elif op["op"] == "commit":
            assert m.commit(op["id"], None) == op["status"], op
            if "slot" in op:
                assert op["id"] % S == op["slot"]
        else:
            assert m.evict(op["id"]) == op["status"], op
            if op["status"] == 0:
                assert m.state()[0][op["slot"]] == -1


def test_ring_slot_model_never_collides_random_traces():
    rnd = random.Random(0)
    for trial in range(300):
        M, T = rnd.randint(0, 12), rnd.randint(1, 6)
        m = O.OracleMemory(M, T)
        for _ in range(40):
            r = rnd.random()
            if r < 0.6:
                m.push(rnd.randint(1, T))
            elif r < 0.8 and m.next_id:
                m.evict(rnd.randint(0, m.next_id))
            elif m.next_id:
                m.commit(rnd.randint(0, m.next_id), None)
            slot_id, _, mask = m.state()          # asserts no two residents share a slot
            assert bin(mask).count("1") == len(m.resident) <= M + T
            assert all(j >= m.cur_first - M for j in m.resident)


def test_protocol_errors():
    m = O.OracleMemory(3, 1)
    assert m.evict(0) == O.VI_E_PROTOCOL          # nothing pushed yet: future frame
    m.push(1)
    assert m.commit(0, None) == O.VI_E_PROTOCOL   # current frame
    m.push(1)
    assert m.commit(0, None) == O.VI_OK
    assert m.evict(5) == O.VI_E_PROTOCOL
    assert m.evict(-1) == O.VI_E_ARG
    with pytest.raises(ValueError):
        m.push(2)


def test_rel_err_metric():
    ref = np.array([1.0, -1.0, 0.0, 1e-9])
    assert O.rel_err(ref, ref) == 0.0
    got = ref + np.array([0, 0, 0.01, 0])
    rms = math.sqrt(np.mean(ref ** 2))
    assert abs(O.rel_err(got, ref) - 0.01 / rms) < 1e-15


def test_round_bf16_is_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 3.4e38], np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(round_bf16(x), ref)


def test_rel_err_with_emulation_denominator_triangle():
    """rel_err(g, e; den_ref=o) + rel_err(e, o) bounds rel_err(g, o) (the parity tests' bar)."""
    rng = np.random.default_rng(5)
    o = rng.standard_normal(1000)
    e = o + 1e-3 * rng.standard_normal(1000)
    g = e + 1e-3 * rng.standard_normal(1000)
    assert O.rel_err(g, o) <= O.rel_err(g, e, den_ref=o) + O.rel_err(e, o) + 1e-15
    assert O.rel_err(g, e, den_ref=e) == O.rel_err(g, e)


def test_bf16_round_matches_torch_and_ties():
    """The emulation's bf16 rounding (fp64 -> fp32 -> bf16, RNE) against torch's cast and hand
    values: 1 + 2^-8 is a tie (rounds to even 1), 1 + 3 2^-8 a tie rounding up to 1 + 2^-6."""
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 0.1, -7.77e-3, 1e30], np.float64)
    ref = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.bf16_round(x), ref)
    assert O.bf16_round(np.array([1.0 + 2 ** -8]))[0] == 1.0
    assert O.bf16_round(np.array([1.0 + 3 * 2 ** -8]))[0] == 1.0 + 2 ** -6
    big = np.random.default_rng(1).standard_normal(4096) * 3
    assert np.array_equal(O.bf16_round(big), torch.from_numpy(big.astype(np.float32)).to(torch.bfloat16).double().numpy())


def test_bf16_storage_emulation_rounds_the_stored_tensors():
    """emulate_bf16_storage: LN1's output h is the oracle's rounded to bf16, Q/K/V are the exact
    projection of that h rounded to bf16, O and g are bf16 values; the embedding (x0) is
    unchanged; the result differs from the oracle only by that storage rounding."""
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=2)
    w = make_weights(cfg, seed=3, variant="sharp")
    o, e = O.OracleStream(cfg, w), O.emulate_bf16_storage(cfg, w)
    feats = make_features(cfg, 1, seed=3)
    o.push(1); e.push(1)
    _, so = o.step(feats)
    _, se = e.step(feats)
    assert np.array_equal(so["x0"], se["x0"])
    l0o, l0e = so["layers"][0], se["layers"][0]
    assert np.array_equal(l0e["h1"], O.bf16_round(l0o["h1"]))          # LN1 output (GEMM operand)
    Q, K, V = (O.bf16_round(O.linear(l0e["h1"], w["wqkv"][0], w["bqkv"][0])[:, i * 64:(i + 1) * 64]) for i in range(3))
    for k, ref in (("q", Q), ("k", K), ("v", V)):
        assert np.array_equal(l0e[k], ref)                         # rounded after the exact projection
        assert not np.array_equal(l0e[k], l0o[k])
    assert np.array_equal(l0e["o"], O.bf16_round(l0e["o"]))
    assert np.array_equal(l0e["g"], O.bf16_round(l0e["g"]))
    assert 0 < O.rel_err(se["out"], so["out"]) < 0.2
    # and the K/V a later step attends to are the rounded ones (re-projected from cached inputs)
    f2 = make_features(cfg, 1, first_frame=1, seed=3)
    o.push(1); e.push(1)
    o.step(f2); e.step(f2)
    Ke, Ve = e.frame_kv(1, 0)
    assert np.array_equal(Ke, O.bf16_round(Ke)) and np.array_equal(Ve, O.bf16_round(Ve))


# ---------------------------------------------------------------- reference frames (Eq. 3 M_{1,r})

def _select_memory(f, s, r, R):
    """SPEC select_memory, written out: neighbours [max(0, f-s), f-1]; references =
    multiples of r in [0, f-1] minus the neighbours -- of which the memory keeps the R most
    recent (DESIGN reading Q12)."""
    nb = set(range(max(0, f - s), f))
    refs = sorted(j for j in range(0, f) if r > 0 and j % r == 0 and j not in nb)
    return nb, set(refs[-R:] if R > 0 else [])


def test_reference_golden_spec_select_memory():
    """select_memory(18, 5, 10) -> neighbours {13..17}, references {0, 10}."""
    m = O.OracleMemory(5, 1, ref_rate=10, max_refs=4)
    for f in range(19):
        m.push(1)
        m.mark_stepped()
    assert m.window() == [0, 10, 13, 14, 15, 16, 17]
    nb, refs = _select_memory(18, 5, 10, 4)
    assert set(m.window()) == nb | refs


def test_reference_window_matches_spec_sets_and_cap():
    for s, r, R in ((3, 4, 2), (5, 10, 4), (2, 3, 1), (4, 2, 3)):
        m = O.OracleMemory(s, 1, ref_rate=r, max_refs=R)
        for f in range(40):
            m.push(1)
            nb, refs = _select_memory(f, s, r, R)
            assert set(m.window()) == nb | refs, (s, r, R, f)
            m.mark_stepped()


def test_reference_memory_step_equals_masked_joint_pass():
    """Exact memoisation with references: T=1 memory steps with span s and references every r
    frames (R kept) == one joint pass where frame i's queries see exactly select_memory(i) and
    itself (the recurrence of Eq. 3 with M_{f-s}^{f-1} U M_{1,r}^{f-1})."""
    s, r, R, n = 2, 3, 2, 9
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=s, ref_rate=r, max_refs=R)
    w = make_weights(cfg, seed=7, variant="sensitive")
    feats = make_features(cfg, n, seed=7)
    mask = np.zeros((n, n), bool)
    for i in range(n):
        nb, refs = _select_memory(i, s, r, R)
        for j in nb | refs | {i}:
            mask[i, j] = True
    joint = O.joint_forward(feats, w, cfg, mode="mask", frame_mask=mask)
    st = O.OracleStream(cfg, w)
    for i in range(n):
        st.push(1)
        out, _ = st.step(feats[i:i + 1])
        np.testing.assert_allclose(out[0], joint["out"][i], rtol=1e-9, atol=1e-11)
    # the references matter: without them frame 8 (refs {0, 3}) differs
    plain = O.joint_forward(feats, w, cfg, mode="mask",
                            frame_mask=np.array([[j <= i and j >= i - s for j in range(n)] for i in range(n)]))
    assert np.abs(plain["out"][8] - joint["out"][8]).max() > 1e-6


# ---------------------------------------------------------------- Eq. 4's refined memory M-bar

def _select_refined(f, t, s, s2, r2, R2):
    """SPEC select_refined, written out: online neighbours [max(0,f-s), f-1];
    refined neighbours [max(0,t-s'), t] minus the online ones (store precedence: a frame is
    held once); refined references = multiples of r' in [0, t] minus both, of which the
    memory keeps the R' newest (reading Q22).  t < 0: no refined frame yet (select_memory)."""
    online = set(range(max(0, f - s), f))
    if t < 0:
        return online, set(), set()
    refined = set(range(max(0, t - s2), t + 1)) - online
    refs = sorted(j for j in range(t + 1) if r2 > 0 and j % r2 == 0 and j not in online and j not in refined)
    return online, refined, set(refs[-R2:] if R2 > 0 else [])


def test_refined_golden_spec_select_refined():
    """SPEC S:473 / Fig. 3 caption: f=18, t=14, s=s'=3, r'=10 -> online {15,16,17},
    refined {11..14}, refined references {0, 10}."""
    online, refined, refs = _select_refined(18, 14, 3, 3, 10, 4)
    assert (online, refined, refs) == ({15, 16, 17}, {11, 12, 13, 14}, {0, 10})
    m = O.OracleMemory(3, 1, refined_span=3, refined_rate=10, max_refined_refs=2)
    for f in range(18):
        m.push(1)
        m.mark_stepped()
    for j in range(15):
        m.commit(j, None)
    m.push(1)
    assert m.window() == sorted(online | refined | refs) and m.t == 14
    assert (m.rspan, set(m.rrefs)) == (refined, refs)


def test_refined_window_matches_spec_sets_random():
    """The set model's memory equals SPEC select_refined's sets for random (s, s', r', R') and
    refiner schedules (the refiner commits every frame up to its lagging watermark t)."""
    rnd = random.Random(77)
    for trial in range(200):
        s, s2, r2, R2 = rnd.randint(0, 5), rnd.randint(0, 5), rnd.randint(0, 6), rnd.randint(1, 3)
        lag, every = rnd.randint(1, 6), rnd.randint(1, 4)
        m = O.OracleMemory(s, 1, refined_span=s2, refined_rate=r2, max_refined_refs=R2)
        t = -1
        for f in range(40):
            if f % every == 0 and f - lag > t and f - lag >= 0:
                t = f - lag
                for j in range(t + 1):
                    m.commit(j, None)
            m.push(1)
            online, refined, refs = _select_refined(f, t, s, s2, r2, R2)
            assert m.window() == sorted(online | refined | refs), (trial, f, t)
            assert m.t == t
            m.mark_stepped()


def test_refined_memory_without_commits_is_the_memory_model():
    """Degradation: no refine commit -> exactly Eq. 3's memory."""
    a = O.OracleMemory(4, 2)
    b = O.OracleMemory(4, 2, refined_span=3, refined_rate=5, max_refined_refs=2)
    for n in (2, 1, 2, 2, 1, 2, 2):
        assert a.push(n) == b.push(n)
        assert a.window() == b.window()
        a.mark_stepped(); b.mark_stepped()


def test_refined_memory_step_equals_masked_joint_pass():
    """Exact memoisation with Eq. 4's refined memory (invariant I3): an identity refiner (it
    commits every frame's own per-block K/V once the frame is t = f - 2 old, every 3 frames)
    makes T=1 memory steps with online span s, refined span s' and refined references every r'
    frames equal one joint pass in which frame i's queries see exactly select_refined(i, t)
    and itself (Eq. 4)."""
    s, s2, r2, R2, n, lag, every = 1, 2, 3, 2, 13, 2, 3
    cfg = CONFIGS["C1"].replace(layers=2, mem_frames=s, refined_mem=1, refined_span=s2, refined_rate=r2,
                                max_refined_refs=R2)
    w = make_weights(cfg, seed=17, variant="sensitive")
    feats = make_features(cfg, n, seed=17)
    st = O.OracleStream(cfg, w)
    kv = {}
    mask = np.zeros((n, n), bool)
    t = -1
    outs = []
    for i in range(n):
        if i % every == 0 and i - lag > t and i - lag >= 0:
            t = i - lag
            for j in range(t + 1):
                K = np.stack([kv[(l, j)][0] for l in range(cfg.layers)])
                V = np.stack([kv[(l, j)][1] for l in range(cfg.layers)])
                st.commit(j, K, V)
        st.push(1)
        online, refined, refs = _select_refined(i, t, s, s2, r2, R2)
        assert st.mem.window() == sorted(online | refined | refs)
        for j in online | refined | refs | {i}:
            mask[i, j] = True
        out, _ = st.step(feats[i:i + 1])
        outs.append(out[0])
        for l in range(cfg.layers):
            kv[(l, i)] = st.frame_kv(l, i)
    joint = O.joint_forward(feats, w, cfg, mode="mask", frame_mask=mask)
    for i in range(n):
        np.testing.assert_allclose(outs[i], joint["out"][i], rtol=1e-9, atol=1e-11)
    # the refined memory matters: Eq. 3 with the same span alone differs at the last frame
    plain = O.joint_forward(feats, w, cfg, mode="mask",
                            frame_mask=np.array([[i - s <= j <= i for j in range(n)] for i in range(n)]))
    assert np.abs(plain["out"][n - 1] - joint["out"][n - 1]).max() > 1e-6


# ---------------------------------------------------------------- window attention (BASELINE configs[3])

def test_window_ids_partition_the_grid():
    cfg = CONFIGS["C4"]
    win = O.token_windows(cfg)
    assert np.bincount(win).tolist() == [45] * 16                  # 4 x 4 windows of 5 x 9 tokens
    oy, ox = np.divmod(np.arange(cfg.tokens), cfg.ow)
    for w in range(16):                                            # each window is a 5 x 9 rectangle
        ys, xs = oy[win == w], ox[win == w]
        assert ys.max() - ys.min() == 4 and xs.max() - xs.min() == 8


def test_window_attention_equals_per_window_attention():
    """The masked block == attention run separately on each window's tokens (all frames of the
    memory and the chunk), O scattered back."""
    cfg = CONFIGS["C3S"].replace(layers=1, win_h=5, win_w=6)        # 10 x 18 grid -> 2 x 3 windows
    w = make_weights(cfg, seed=3, variant="sensitive")
    rng = rng_for(3, "win")
    P, D, n = cfg.tokens, cfg.d_model, 2
    x = rng.standard_normal((n * P, D))
    mem = []
    for j in range(3):
        _, _, K, V = O.qkv(rng.standard_normal((P, D)), w, 0, cfg)
        mem.append((K, V))
    _, st = O.block_memory(x, mem, w, 0, cfg, n)
    _, Q, Kc, Vc = O.qkv(x, w, 0, cfg)
    K = np.concatenate([k for k, _ in mem] + [Kc]); V = np.concatenate([v for _, v in mem] + [Vc])
    win = O.token_windows(cfg)
    ref = np.zeros_like(st["o"])
    for wid in range(win.max() + 1):
        qi = np.nonzero(np.tile(win, n) == wid)[0]
        ki = np.nonzero(np.tile(win, len(mem) + n) == wid)[0]
        ref[qi] = O.attention(Q[qi], K[ki], V[ki], cfg.heads)
    np.testing.assert_allclose(st["o"], ref, rtol=1e-12, atol=1e-13)


def test_window_of_the_whole_grid_is_global_attention():
    cfg = CONFIGS["C3S"].replace(layers=1)
    whole = cfg.replace(win_h=cfg.oh, win_w=cfg.ow)
    w = make_weights(cfg, seed=4, variant="sensitive")
    rng = rng_for(4, "win")
    x = rng.standard_normal((cfg.tokens, cfg.d_model))
    _, _, K, V = O.qkv(rng.standard_normal((cfg.tokens, cfg.d_model)), w, 0, cfg)
    a, _ = O.block_memory(x, [(K, V)], w, 0, cfg, 1)
    b, _ = O.block_memory(x, [(K, V)], w, 0, whole, 1)
    np.testing.assert_array_equal(a, b)
