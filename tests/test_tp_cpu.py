"""Head-sharding host logic without a GPU.

* vi_tp_layout (the partition every sharded context uses, CUDA-free): the (head, query-row)
  units of the G ranks tile the attention exactly once, and each rank's chunk of the
  head-major gathered buffer holds exactly its units.
* Two gloo ranks (world_size 2) run the sharded decomposition end to end on CPU: each
  computes its heads' attention (oracle arithmetic) into its chunk laid out by
  vi_tp_layout, the chunks are all-gathered with torch.distributed, and the assembled
  concat_h(O_h) W_o equals the unsharded block's on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


@pytest.fixture(scope="module")
def V():
    from paper_2403_16161_b200 import build
    build.build()
    from paper_2403_16161_b200 import vi
    return vi


@pytest.mark.parametrize("H,G", [(4, 1), (4, 2), (4, 4), (4, 8), (4, 16), (8, 2), (2, 6), (1, 3)])
def test_layout_tiles_heads_and_rows(V, H, G):
    d, rows_max = 8, 37          # odd row count: the last query part is short
    owner = -np.ones((H, rows_max), dtype=int)
    L0 = V.tp_layout(H, d, rows_max, G, 0)
    head_rows = L0["head_rows"]
    cell_rank = -np.ones((H, head_rows), dtype=int)   # rank owning each gathered-buffer row
    for r in range(G):
        L = V.tp_layout(H, d, rows_max, G, r)
        assert L["chunk_elems"] * G == H * head_rows * d      # equal chunks cover the buffer
        assert L["head_rows"] == head_rows
        rows = range(L["row0"], min(L["row0"] + L["part_rows"], rows_max))
        for h in range(L["head0"], L["head0"] + L["nheads"]):
            for i in rows:
                assert owner[h, i] == -1, (h, i)
                owner[h, i] = r
        # elements [r*chunk, (r+1)*chunk) of the head-major [H][head_rows][d] buffer
        flat = np.arange(r * L["chunk_elems"], (r + 1) * L["chunk_elems"]) // d
        hh, ii = flat // head_rows, flat % head_rows
        cell_rank[hh, ii] = r
        assert set(zip(hh.tolist(), ii.tolist())) >= {(h, i) for h in range(L["head0"], L["head0"] + L["nheads"])
                                                    for i in rows}
    assert (owner >= 0).all()
    assert (cell_rank[:, :rows_max] == owner).all()


@pytest.mark.parametrize("H,G", [(4, 3), (4, 6), (3, 2), (4, 0)])
def test_layout_rejects_uneven_splits(V, H, G):
    with pytest.raises(V.ViError) as e:
        V.tp_layout(H, 8, 16, G, 0)
    assert e.value.status == V.VI_E_CONFIG


def test_unique_id_is_128_bytes(V):
    a, b = V.tp_unique_id(), V.tp_unique_id()
    assert len(a) == 128 and a != b


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist

    from oracle import vi_oracle as O
    from paper_2403_16161_b200 import streams, vi
    from vi_synth import rng_for
    streams.init("gloo", streams.DistInfo.from_env())
    uid = streams.broadcast_bytes(vi.tp_unique_id() if rank == 0 else None)   # what bench.py --tp does
    H, d, nq, nk = 4, 16, 45, 70
    D = H * d
    rng = rng_for(0, "tp-cpu")
    Q, K, Vv = (rng.standard_normal((m, D)) for m in (nq, nk, nk))
    Wo = rng.standard_normal((D, D)) * 0.1
    res = {}
    for G in (2, 4, 8):            # G logical ranks over the 2 processes
        buf = np.zeros(0)
        mine = range(rank, G, world)
        L0 = vi.tp_layout(H, d, nq, G, 0)
        chunks = {}
        for r in mine:
            L = vi.tp_layout(H, d, nq, G, r)
            ch = np.zeros((L["chunk_elems"],), np.float64)
            hs, rows = range(L["head0"], L["head0"] + L["nheads"]), range(L["row0"], min(L["row0"] + L["part_rows"], nq))
            if len(rows):
                cols = np.concatenate([np.arange(h * d, (h + 1) * d) for h in hs])
                Oh = O.attention(Q[list(rows)][:, cols], K[:, cols], Vv[:, cols], L["nheads"])
                view = ch.reshape(L["nheads"], -1, d)       # [heads][rows of the part][d]
                for j in range(L["nheads"]):
                    view[j, :len(rows)] = Oh[:, j * d:(j + 1) * d]
            chunks[r] = ch
        # all-gather: every rank's chunk to every process (rank order)
        gathered = [None] * world
        dist.all_gather_object(gathered, chunks)
        allc = {}
        for g in gathered:
            allc.update(g)
        buf = np.concatenate([allc[r] for r in range(G)]).reshape(H, L0["head_rows"], d)
        O_cat = np.concatenate([buf[h, :nq] for h in range(H)], axis=1)   # concat_h(O_h) [nq, D]
        ref = O.attention(Q, K, Vv, H)
        res[G] = (float(np.max(np.abs(O_cat - ref))), float(np.max(np.abs(O_cat @ Wo.T - ref @ Wo.T))))
    out[rank] = (res, uid)
    dist.destroy_process_group()


def test_two_gloo_ranks_sharded_attention_gather_equals_unsharded():
    ctx = mp.get_context("spawn")
    world, port = 2, _free_port()
    out = ctx.Manager().dict()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    assert len(out[0][1]) == 128 and out[0][1] == out[1][1]        # one NCCL id for the group
    for rank in range(world):
        for G, (e_o, e_proj) in out[rank][0].items():
            assert e_o < 1e-12 and e_proj < 1e-12, (rank, G, e_o, e_proj)
