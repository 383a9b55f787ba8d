"""Round sharding across GPUs: one process per GPU, per-round merge.

SURVEY.md §8(e).  A global round of R inputs (global ids ``it0 .. it0+R-1``)
is split into contiguous slices, rank r owning round indices
``[R*r//W, R*(r+1)//W)``.  Every rank holds the same corpus, campaign map and
findings, so the only exchanges are per round and tiny:

==========================  =========  ===========================================
what                        op         why
==========================  =========  ===========================================
int-arg pick totals [C]     all-gather rotation counts of later slices start after
                                       the picks of earlier ones (mutation.py:371-386)
stop / fatal index          MIN        first stopping input truncates the round
first hitter per edge [E],  MIN        novelty = "first hitter of an edge unseen at
first input per key [K]                the round start" (the OR of the coverage
                                       bitmaps, expressed as a MIN: hit <=> != none)
edge / key / entered counts SUM        campaign map and FindingsLog hit counts
admitted, allocs per rank   all-gather corpus append order, alloc-id prefixes
admitted children records   all-gather replicated corpus (rare)
new finding reports         object     FindingsLog entries (rare)
==========================  =========  ===========================================

With the global round size fixed, results do not depend on the GPU count.
NCCL has no bitwise OR; MIN over first-hitter ids subsumes it.  With the
``nccl`` backend the collectives run in place on the round's CUDA stream;
with ``gloo`` (CPU tests, or several ranks sharing one GPU) they are staged
through host memory.  World size 1 makes every collective the identity.
"""

from __future__ import annotations

import torch


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Round indices ``[lo, hi)`` of ``rank`` in a round of ``n`` inputs."""
    return n * rank // world, n * (rank + 1) // world


def owner_of(index: int, n: int, world: int) -> int:
    """Rank whose slice holds round index ``index``."""
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        if lo <= index < hi:
            return r
    raise ValueError(f"round index {index} outside a round of {n}")


class RoundComm:
    """Per-round collectives of a sharded campaign (torch.distributed)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = str(dist.get_backend(group))
        else:
            self.rank, self.world, self.backend = 0, 1, "none"
        self.staged = self.backend != "nccl"
        self.calls = 0

    def bounds(self, n: int) -> tuple[int, int]:
        return shard_bounds(n, self.rank, self.world)

    def _run(self, t: torch.Tensor, fn):
        if self.staged and t.is_cuda:
            h = t.cpu()
            fn(h)
            t.copy_(h)
        else:
            fn(t)

    def all_reduce(self, t: torch.Tensor, op: str, stream=None) -> None:
        """In-place MIN / SUM / MAX over ranks of ``t`` (stream-ordered on ``stream``)."""
        if self.world == 1 or t.numel() == 0:
            return
        self.calls += 1
        rop = {"min": self.dist.ReduceOp.MIN, "sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX}[op]
        with torch.cuda.stream(stream) if stream is not None else _null():
            self._run(t, lambda x: self.dist.all_reduce(x, op=rop, group=self.group))

    def all_gather(self, t: torch.Tensor, stream=None) -> torch.Tensor:
        """``[world, *t.shape]``: every rank's ``t`` in rank order."""
        if self.world == 1:
            return t.unsqueeze(0)
        self.calls += 1
        with torch.cuda.stream(stream) if stream is not None else _null():
            src = t.cpu() if (self.staged and t.is_cuda) else t.contiguous()
            out = torch.empty((self.world,) + tuple(src.shape), dtype=src.dtype, device=src.device)
            self.dist.all_gather(list(out.unbind(0)), src, group=self.group)
            return out.to(t.device, non_blocking=False) if out.device != t.device else out

    def all_gather_object(self, obj) -> list:
        if self.world == 1:
            return [obj]
        self.calls += 1
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
