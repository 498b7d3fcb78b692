"""Data-parallel GNP training over batch samples.

The reference trains one batch per step. Its worker threads each take a
subset of columns, and `accumulate` sums their gradients in column order
(`src/gnn.cpp:369-388,426-440`). Here the columns of a global batch of B are
split evenly over the ranks of a process group, one process per GPU:

  1. each rank runs forward + L1 loss + backward on its B/N columns
     (`gnpc_train_backward_only` / `gnpc_train_backward_synthetic`). That gives
     the gradient of its local mean loss in the trainer's flat f64 device
     buffer.
  2. one all-reduce (SUM) of that buffer, then a 1/N scale. The mean of the
     local means is the global (1/B)Σ_k gradient, since the shards are equal.
     This is the only data-path collective.
  3. every rank applies the identical Adam step (`gnpc_train_apply_grads`).
     Parameters stay replicated bit-for-bit.

The driver is written against a small engine protocol so the same host logic
runs on the GPU trainer (NCCL) and, in the CPU tests, on an oracle-backed
engine (gloo).
"""
from __future__ import annotations

from dataclasses import dataclass


def shard_columns(global_batch: int, rank: int, world: int) -> slice:
    """Contiguous column block of a global batch owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} is not divisible by {world} ranks")
    per = global_batch // world
    return slice(rank * per, (rank + 1) * per)


@dataclass
class _CudaArray:
    """Zero-copy view of a device buffer for torch.as_tensor."""

    ptr: int
    count: int

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.count,), "typestr": "<f8", "data": (self.ptr, False), "version": 3}


class TrainerEngine:
    """Engine over the C-ABI trainer (capi.Trainer); gradients stay on device."""

    def __init__(self, trainer):
        import torch

        self.t = trainer
        ptr, cnt = trainer.grad_buffer()
        self.grad = torch.as_tensor(_CudaArray(ptr, cnt), device="cuda")

    def backward(self, x, b) -> float:
        # (n, Bl) logical arrays -> the C ABI's column-major n x Bl
        import numpy as np

        return self.t.backward_only(np.asfortranarray(x).ravel(order="F"),
                                    np.asfortranarray(b).ravel(order="F"))

    def backward_synthetic(self, seed: int) -> float:
        return self.t.backward_synthetic(seed)

    def grad_tensor(self):
        return self.grad

    def apply_grads(self) -> None:
        import torch

        torch.cuda.current_stream().synchronize()  # the all-reduce ran on torch's stream
        self.t.apply_grads()


class DataParallelTrainer:
    """One data-parallel step = local backward, gradient all-reduce, Adam."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist

        self.e = engine
        self.group = group
        self.dist = dist
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def _reduce(self, local_loss: float) -> float:
        import torch

        g = self.e.grad_tensor()
        if self.world > 1:
            self.dist.all_reduce(g, op=self.dist.ReduceOp.SUM, group=self.group)
            g.div_(self.world)
            lt = torch.tensor([local_loss], dtype=torch.float64, device=g.device)
            self.dist.all_reduce(lt, op=self.dist.ReduceOp.SUM, group=self.group)
            return float(lt.item()) / self.world
        return local_loss

    def step(self, x_global, b_global) -> float:
        """x_global, b_global: (n, B) arrays of the GLOBAL batch (every rank
        holds the same copy); this rank trains on its column shard."""
        cols = shard_columns(x_global.shape[1], self.rank, self.world)
        loss = self._reduce(self.e.backward(x_global[:, cols], b_global[:, cols]))
        self.e.apply_grads()
        return loss

    def step_shard(self, x_shard, b_shard) -> float:
        """The rank's own (n, B/N) shard (data already partitioned)."""
        loss = self._reduce(self.e.backward(x_shard, b_shard))
        self.e.apply_grads()
        return loss

    def step_synthetic(self, seed: int) -> float:
        """Device-generated pairs; rank r draws from stream seed + r."""
        loss = self._reduce(self.e.backward_synthetic(seed + self.rank))
        self.e.apply_grads()
        return loss
