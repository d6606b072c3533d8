"""Multi-GPU plumbing for `bench.py --gpus N`: one process per GPU, N
independent replicas of the array (the online stage does not shard in this
round), so there is no data-path collective. Only the barrier
around the timed region and the max/sum over ranks go through
torch.distributed (NCCL on GPUs, gloo on CPU for the tests).
"""
from __future__ import annotations

import os


class Ranks:
    def __init__(self, backend: str | None = None, device: int | None = None):
        self.rank = int(os.environ.get("RANK", 0))
        self.local_rank = int(os.environ.get("LOCAL_RANK", 0))
        self.world = int(os.environ.get("WORLD_SIZE", 1))
        self.dist = None
        self.device = device
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            self.backend = backend
            if backend == "nccl":
                torch.cuda.set_device(self.local_rank if device is None else device)
                dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
            else:
                dist.init_process_group(backend)
            self.dist = dist

    def _tensor(self, x):
        import torch
        dev = f"cuda:{torch.cuda.current_device()}" if self.backend == "nccl" else "cpu"
        return torch.tensor([float(x)], dtype=torch.float64, device=dev)

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, x: float) -> float:
        """Max over ranks (multi-GPU times are the slowest rank's)."""
        if self.dist is None:
            return float(x)
        t = self._tensor(x)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.dist is None:
            return float(x)
        t = self._tensor(x)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()
            self.dist = None


def aggregate_throughput(blocks_per_rank: int, world: int, max_ms_per_step: float) -> float:
    """Whole-job blocks/s of N replicas timed by the slowest rank (weak scaling)."""
    return world * blocks_per_rank / (max_ms_per_step / 1e3)
