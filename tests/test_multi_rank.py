"""N > 1 host path on CPU: two gloo ranks (world_size 2) exercising the stream split,
the max-over-ranks timing rule and per-rank independent ring bookkeeping."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2403_16161_b200 import streams
    from paper_2403_16161_b200 import build
    build.build()
    from paper_2403_16161_b200 import vi
    info = streams.DistInfo.from_env()
    streams.init("gloo", info)
    ids = streams.stream_ids(info.rank, info.world, 8)
    # each rank times a different amount; the job time is the max over ranks
    local_time = 1.0 + info.rank
    tmax, = streams.max_over_ranks([local_time])
    # each rank's stream has its own ring: bookkeeping is rank-local
    r = vi.Ring(10, 5)
    for _ in range(3 + info.rank):
        r.push(5)
    _, _, mask = r.state()
    streams.barrier()
    out[rank] = (ids, tmax, mask, streams.aggregate_fps(5 * 10, info.world, tmax))
    torch.distributed.destroy_process_group()


def test_two_gloo_ranks_split_streams_and_reduce_time():
    ctx = mp.get_context("spawn")
    world, port = 2, _free_port()
    manager = ctx.Manager()
    out = manager.dict()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ids0, t0, m0, fps0 = out[0]
    ids1, t1, m1, fps1 = out[1]
    assert sorted(ids0 + ids1) == list(range(8)) and not set(ids0) & set(ids1)
    assert t0 == t1 == 2.0                      # max over ranks
    assert fps0 == fps1 == 2 * 50 / 2.0          # whole-job throughput
    assert m0 == 0x7fff and m1 == 0x7fff         # 3 / 4 pushes of 5 frames: ring full on both


def test_single_rank_helpers():
    from paper_2403_16161_b200 import streams
    assert streams.stream_ids(0, 1, 3) == [0, 1, 2]
    assert streams.max_over_ranks([1.5, 2.5]) == [1.5, 2.5]
    assert streams.stream_seed(3) != streams.stream_seed(4)
