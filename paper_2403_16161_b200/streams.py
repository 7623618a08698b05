"""Multi-GPU host logic (one process per GPU).

Two ways the memory step shards:
* independent live streams split across GPUs: the streams share nothing (each has its own
  ring memory), so N GPUs serve N streams with no data-path collective (weak scaling);
* one stream with its attention heads split across GPUs: libvi.so joins an NCCL
  communicator (its unique id broadcast here) and all-gathers the head outputs inside
  every block (strong scaling of one stream's step).
Cross-rank traffic here is only the timing reduction (max over ranks), barriers and the
id broadcast.  Works with the NCCL backend on GPUs and with gloo on CPU (tests).
"""
from __future__ import annotations

import dataclasses
import os
from typing import List, Sequence

import torch
import torch.distributed as dist


@dataclasses.dataclass(frozen=True)
class DistInfo:
    rank: int
    world: int
    local_rank: int

    @staticmethod
    def from_env() -> "DistInfo":
        return DistInfo(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                        int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, info: DistInfo, device: torch.device = None) -> None:
    """Join the process group when more than one rank runs (MASTER_ADDR/PORT from env)."""
    if info.world > 1 and not dist.is_initialized():
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, rank=info.rank, world_size=info.world, **kw)


def stream_ids(rank: int, world: int, n_streams: int) -> List[int]:
    """Live streams served by `rank`: round-robin, every stream on exactly one rank."""
    return list(range(rank, n_streams, world))


def stream_seed(stream_id: int, base: int = 0) -> int:
    """Each live stream draws its own synthetic frames (independent problems)."""
    return base * 1_000_003 + stream_id


def max_over_ranks(values: Sequence[float], device: torch.device = None) -> List[float]:
    """Element-wise max over ranks (the benchmark's timing rule); identity at world 1."""
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def broadcast_bytes(payload, device: torch.device = None) -> bytes:
    """Rank 0's bytes on every rank (the NCCL unique id of a head-sharded group)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return payload
    obj = [payload]
    dist.broadcast_object_list(obj, src=0, device=device)
    return obj[0]


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def aggregate_fps(frames_per_rank: int, world: int, max_seconds: float) -> float:
    """Whole-job throughput: every rank processed frames_per_rank frames; the job took the
    slowest rank's time."""
    return world * frames_per_rank / max_seconds
