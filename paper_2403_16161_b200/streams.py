"""Multi-GPU host logic: independent live streams split across GPUs (one process per GPU).

The memory step of different live streams shares nothing (each stream has its own ring
memory), so N GPUs serve N x streams with no data-path collective (weak scaling); the
only cross-rank traffic is the timing reduction of the benchmark (max over ranks) and
barriers.  Works with the NCCL backend on GPUs and with gloo on CPU (tests).
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


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def aggregate_fps(frames_per_rank: int, world: int, max_seconds: float) -> float:
    """Whole-job throughput: every rank processed frames_per_rank frames; the job took the
    slowest rank's time."""
    return world * frames_per_rank / max_seconds
