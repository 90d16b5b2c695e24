"""Frame-level data parallelism: frames are independent, so rank r of W
processes the contiguous range [r*F/W, (r+1)*F/W) with no data-path collective; the only
exchange is one gather of fixed-size detection records to rank 0 (NCCL over NVLink on
GPUs, gloo in the CPU tests).

Record layout per frame (int32): [delay x K | doppler x K | power bits x K | count].
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(frames: int, rank: int, world: int) -> tuple[int, int]:
    return rank * frames // world, (rank + 1) * frames // world


def pack(delay: torch.Tensor, doppler: torch.Tensor, power: torch.Tensor, counts: torch.Tensor,
         out: torch.Tensor | None = None) -> torch.Tensor:
    """(F, K) int32, (F, K) int32, (F, K) float32, (F,) int32 -> (F, 3K + 1) int32."""
    k = delay.shape[1]
    if out is None:
        out = torch.empty(delay.shape[0], 3 * k + 1, dtype=torch.int32, device=delay.device)
    out[:, :k] = delay
    out[:, k:2 * k] = doppler
    out[:, 2 * k:3 * k] = power.contiguous().view(torch.int32)
    out[:, 3 * k] = counts
    return out


def unpack(rec: torch.Tensor, k: int):
    return (rec[:, :k], rec[:, k:2 * k], rec[:, 2 * k:3 * k].contiguous().view(torch.float32), rec[:, 3 * k])


class DetectionGather:
    """Pre-allocated gather of every rank's packed records to rank 0 (one dist.gather of
    equal-size padded shards; ~3K+1 int32 per frame, i.e. < 1 MB for cfg4).  Only rank 0
    receives the records."""

    def __init__(self, frames: int, k: int, rank: int, world: int, device: torch.device):
        self.frames, self.k, self.rank, self.world = frames, k, rank, world
        self.sizes = [b - a for a, b in (shard_range(frames, r, world) for r in range(world))]
        self.rows = max(self.sizes)
        self.local = torch.zeros(self.rows, 3 * k + 1, dtype=torch.int32, device=device)
        self.bufs = [torch.empty_like(self.local) for _ in range(world)] if rank == 0 else None

    def __call__(self, delay, doppler, power, counts) -> torch.Tensor | None:
        n = delay.shape[0]
        pack(delay, doppler, power, counts, out=self.local[:n])
        if self.world == 1:
            return self.local[:n]
        dist.gather(self.local, gather_list=self.bufs, dst=0)
        if self.rank != 0:
            return None
        return torch.cat([b[:s] for b, s in zip(self.bufs, self.sizes)])
