"""C-ABI checks that need no GPU: libvi.so loads, exports every symbol include/vi.h
declares, and its integer ring bookkeeping matches the oracle's set model bit-exactly."""
import json
import os
import random
import re
import subprocess

import pytest

from oracle import vi_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def V():
    from paper_2403_16161_b200 import build
    build.build()
    from paper_2403_16161_b200 import vi
    return vi


def header_symbols():
    src = open(os.path.join(ROOT, "include", "vi.h")).read()
    return sorted(set(re.findall(r"^\s*(?:vi_status|const char\*|int64_t|int|void\*)\s+(vi_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol(V):
    syms = header_symbols()
    assert len(syms) >= 25, syms
    out = subprocess.run(["nm", "-D", "--defined-only", V.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (vi_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(V.EXPORTS) == set(syms)
    assert "sm_100a" in V.version()


def test_library_is_sm100a_tensor_core_code(V):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", V.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # TMA tensor loads
    assert "LDTM" in sass             # tcgen05.ld (TMEM -> registers)
    assert "HMMA" not in sass.replace("UTCHMMA", "")   # no legacy mma.sync path


def test_ring_goldens_through_abi(V):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "ring_trace.json")))
    r = V.Ring(g["M"], g["T_max"])
    S = g["M"] + g["T_max"]
    for op in g["ops"]:
        if op["op"] == "push":
            first, ev = r.push(op["n"])
            assert (first, ev) == (op["first"], op["evicted"])
            _, ref, mask = r.state()
            assert mask == int(op["mask"], 16)
            if "refined_slots" in op:
                assert [i for i in range(S) if ref[i]] == op["refined_slots"]
        elif op["op"] == "commit":
            assert r.commit(op["id"]) == op["status"]
        else:
            assert r.evict(op["id"]) == op["status"]


def test_ring_matches_oracle_set_model_random_traces(V):
    rnd = random.Random(1234)
    for trial in range(400):
        M, T = rnd.randint(0, 20), rnd.randint(1, 8)
        r, m = V.Ring(M, T), O.OracleMemory(M, T)
        for step in range(60):
            x = rnd.random()
            if x < 0.45:
                n = rnd.randint(1, T)
                assert r.push(n) == m.push(n)
            elif x < 0.6:
                r.mark_stepped(); m.mark_stepped()
            elif x < 0.8:
                fid = rnd.randint(-1, m.next_id + 1)
                assert r.evict(fid) == m.evict(fid), (trial, step, fid)
            else:
                fid = rnd.randint(-1, m.next_id + 1)
                assert r.commit(fid) == m.commit(fid, None), (trial, step, fid)
            assert r.state() == tuple(list(x) if isinstance(x, list) else x for x in m.state())


def test_ring_rejects_bad_arguments(V):
    with pytest.raises(V.ViError):
        V.Ring(60, 5)                  # S > 64
    r = V.Ring(3, 2)
    with pytest.raises(V.ViError):
        r.push(3)
    with pytest.raises(V.ViError):
        r.push(0)


def test_create_without_gpu_fails_loudly(V):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(V.ViError) as e:
        V.Context(layers=1)
    assert e.value.status == V.VI_E_CUDA


def test_create_validates_config_before_touching_the_gpu(V):
    with pytest.raises(V.ViError) as e:
        V.Context(tokens_per_frame=719)
    assert e.value.status == V.VI_E_CONFIG
    with pytest.raises(V.ViError) as e:
        V.Context(mem_frames=60)
    assert e.value.status == V.VI_E_CONFIG
    with pytest.raises(V.ViError) as e:
        V.Context(sh=9, kh=7, feat_h=60, tokens_per_frame=7 * 36)   # stride > kernel: uncovered cells
    assert e.value.status == V.VI_E_CONFIG


def test_ring_with_references_matches_oracle_random_traces(V):
    """Reference slots (Eq. 3 M_{1,r}, reading Q12): slot table, refined bits, moves and
    evictions bit-exact against the oracle's set model, including explicit evictions and
    commits of reference frames."""
    rnd = random.Random(99)
    for trial in range(300):
        M, T = rnd.randint(0, 8), rnd.randint(1, 4)
        rr, R = rnd.randint(1, 6), rnd.randint(1, 4)
        r, m = V.Ring(M, T, rr, R), O.OracleMemory(M, T, ref_rate=rr, max_refs=R)
        for step in range(60):
            x = rnd.random()
            if x < 0.45:
                n = rnd.randint(1, T)
                assert r.push(n) == m.push(n), (trial, step)
            elif x < 0.6:
                r.mark_stepped(); m.mark_stepped()
            elif x < 0.75:
                fid = rnd.randint(-1, m.next_id + 1)
                assert r.evict(fid) == m.evict(fid), (trial, step, fid)
            else:
                fid = rnd.randint(-1, m.next_id + 1)
                assert r.commit(fid) == m.commit(fid, None), (trial, step, fid)
            assert r.state() == tuple(list(x) if isinstance(x, list) else x for x in m.state()), (trial, step)


def test_ring_reference_golden_spec(V):
    """SPEC S:464 select_memory(18, 5, 10): at frame 18 the memory holds 13..17 and the
    references 0 and 10."""
    r = V.Ring(5, 1, 10, 2)
    for f in range(19):
        r.push(1)
        r.mark_stepped()
    sid, _, _ = r.state()
    assert sorted(x for x in sid if x >= 0) == [0, 10, 13, 14, 15, 16, 17, 18]
    assert sid[6:] in ([0, 10], [10, 0])          # the two reference slots follow the 6 span slots


# ---------------------------------------------------------------- Eq. 4's refined memory M-bar

def test_ring_refined_matches_oracle_random_traces(V):
    """Eq. 4's refined memory (reading Q22): slot table, refined bits, watermark, commit codes
    and evictions bit-exact against the oracle's set model over random traces of pushes,
    explicit evictions and refine commits (resident, landing in the refined span or the
    refined references, or useless), with and without Eq. 3 references alongside."""
    rnd = random.Random(4242)
    for trial in range(400):
        M, T = rnd.randint(0, 6), rnd.randint(1, 3)
        sr, rrt, RR = rnd.randint(0, 5), rnd.randint(0, 5), rnd.randint(0, 3)
        rr, R = (rnd.randint(1, 5), rnd.randint(1, 3)) if rnd.random() < 0.3 else (0, 0)
        r = V.Ring(M, T, rr, R, refined_span=sr, refined_rate=rrt, max_refined_refs=RR)
        m = O.OracleMemory(M, T, ref_rate=rr, max_refs=R, refined_span=sr, refined_rate=rrt, max_refined_refs=RR)
        for step in range(70):
            x = rnd.random()
            if x < 0.35:
                n = rnd.randint(1, T)
                assert r.push(n) == m.push(n), (trial, step)
                r.mark_stepped(); m.mark_stepped()
            elif x < 0.45:
                fid = rnd.randint(-1, m.next_id + 1)
                assert r.evict(fid) == m.evict(fid), (trial, step, fid)
            else:
                fid = rnd.randint(max(-1, m.next_id - 3 * (M + sr + 2)), m.next_id + 1)
                assert r.commit(fid) == m.commit(fid, None), (trial, step, fid)
            assert r.state() == tuple(m.state()), (trial, step)
            assert r.watermark == m.t


def test_ring_refined_golden_spec_select_refined(V):
    """SPEC S:473 (Fig. 3 caption): select_refined(f=18, t=14, s=s'=3, r'=10) -> online
    {15, 16, 17}, refined {11..14}, refined references {0, 10}.  The online inpainter has shown
    frames 0..17 (span 3); the refiner has committed its results for frames 0..14 (t = 14);
    at frame 18's push the memory holds exactly those sets."""
    r = V.Ring(3, 1, refined_span=3, refined_rate=10, max_refined_refs=2)
    m = O.OracleMemory(3, 1, refined_span=3, refined_rate=10, max_refined_refs=2)
    for f in range(18):
        for x in (r, m):
            x.push(1)
            x.mark_stepped()
    codes = [r.commit(j) for j in range(15)]
    assert codes == [m.commit(j, None) for j in range(15)]
    assert all(c == V.VI_OK for c in codes)
    r.push(1); m.push(1)
    sid, ref, _ = r.state()
    S = 3 + 1
    online = sorted(x for x in sid[:S] if 0 <= x < 18)
    refined_span = sorted(x for x in sid[S:S + 4] if x >= 0)
    refined_refs = sorted(x for x in sid[S + 4:] if x >= 0)
    assert (online, refined_span, refined_refs) == ([15, 16, 17], [11, 12, 13, 14], [0, 10])
    assert r.watermark == 14 and m.window() == [0, 10, 11, 12, 13, 14, 15, 16, 17]
    assert all(ref[i] for i in range(len(sid)) if sid[i] in (0, 10, 11, 12, 13, 14))
    assert r.state() == tuple(m.state())
