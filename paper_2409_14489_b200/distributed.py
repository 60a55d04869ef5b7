"""Multi-GPU CB-ESSFM: shard/halo planner execution and the final gather.

One process per GPU (torch.distributed, NCCL backend on B200s). The
overlap-save schedule of a batch of waveforms is partitioned by
``planner.plan_shards``: whole waveforms per rank when there are at least as
many waveforms as ranks, otherwise contiguous block ranges of a waveform
(time shards). A time shard uploads only its circular input slice -- its
output span plus an N_ov/2 halo on each side, exactly the samples its blocks
read (dbp.py:473-475) -- so ranks never communicate inside the step loop.
The only collective is the final gather of the kept samples to rank 0
(SURVEY.md 8(e)).

``compute`` is injectable: the product passes the GPU launcher
(:func:`gpu_compute`); the CPU tests pass the numpy oracle, so the
partitioning and gather logic is exercised with gloo on world_size 2.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .planner import BlockSchedule, Shard, gather_slice, plan_shards


@dataclass(frozen=True)
class ShardWork:
    """What one rank computes: waveforms [w0, w1), blocks [b0, b1), the
    circular input slice (origin, length) and the output span [o0, o1)."""

    shard: Shard
    in_origin: int
    in_length: int
    out_begin: int
    out_end: int

    @property
    def empty(self) -> bool:
        return self.shard.is_empty()


def shard_work(n: int, block_size: int, overlap: int, batch: int, world: int,
               rank: int) -> ShardWork:
    sched = BlockSchedule(n, block_size, overlap)
    s = plan_shards(batch, sched.n_blocks, world)[rank]
    if s.is_empty():
        return ShardWork(s, 0, 0, 0, 0)
    b0, b1 = s.blocks
    if (b0, b1) == (0, sched.n_blocks):
        origin, length = 0, n                      # whole waveform, no slicing
    else:
        origin, length = sched.input_range(b0, b1)
    o0, o1 = sched.output_range(b0, b1)
    return ShardWork(s, origin, length, o0, o1)


def gpu_compute(engine, device=None):
    """Compute callable running the fused kernel of a DbpEngine on a halo'd
    host slice: returns the kept samples [Bw, 2, o1 - o0] as numpy."""
    import torch

    from .engine import launch

    def run(x_slice: np.ndarray, work: ShardWork, n: int) -> np.ndarray:
        dev = engine.device if device is None else device
        x = torch.from_numpy(x_slice).to(dev).to(engine.torch_dtype)
        out = torch.zeros((x.shape[0], 2, work.out_end - work.out_begin),
                          dtype=engine.torch_dtype, device=dev)
        launch(engine.plan, x, out, n=n, block_range=work.shard.blocks,
               in_origin=work.in_origin, out_origin=work.out_begin)
        return out.to(torch.complex128).cpu().numpy()

    return run


def run_distributed(x: np.ndarray, block_size: int, overlap: int, compute,
                    group=None, device=None) -> np.ndarray | None:
    """Shard a [B, 2, n] batch over the process group, run ``compute`` on
    each rank's halo'd slice, and gather the kept samples on rank 0.

    Every rank passes the same host batch (or at least the samples its
    shard reads). Returns the assembled [B, 2, n] complex128 array on rank
    0 and None elsewhere."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    batch, _, n = x.shape
    work = shard_work(n, block_size, overlap, batch, world, rank)
    w0, w1 = work.shard.waveforms
    if work.empty:
        piece = np.zeros((0, 2, 0), dtype=np.complex128)
    else:
        xs = x[w0:w1] if work.in_length == n and work.in_origin == 0 else \
            gather_slice(x[w0:w1], work.in_origin, work.in_length)
        piece = np.ascontiguousarray(compute(xs, work, n), dtype=np.complex128)

    # final gather (the only collective): pad every piece to the largest
    # shard and all_gather_into_tensor (NCCL-friendly), rank 0 assembles
    sizes = [shard_work(n, block_size, overlap, batch, world, r) for r in range(world)]
    max_elems = max((s.shard.waveforms[1] - s.shard.waveforms[0]) * 2 *
                    (s.out_end - s.out_begin) for s in sizes)
    max_elems = max(max_elems, 1)
    dev = torch.device("cpu") if device is None else device
    # exchanged as float64 pairs: gloo has no complex reductions/gathers
    buf = torch.zeros(2 * max_elems, dtype=torch.float64, device=dev)
    flat = torch.from_numpy(piece.reshape(-1).view(np.float64))
    buf[:flat.numel()] = flat.to(dev)
    gathered = torch.empty(world * 2 * max_elems, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(gathered, buf, group=group)
    if rank != 0:
        return None
    g = gathered.cpu().numpy().view(np.complex128).reshape(world, max_elems)
    out = np.zeros((batch, 2, n), dtype=np.complex128)
    for r, s in enumerate(sizes):
        if s.empty:
            continue
        a0, a1 = s.shard.waveforms
        span = s.out_end - s.out_begin
        out[a0:a1, :, s.out_begin:s.out_end] = \
            g[r, :(a1 - a0) * 2 * span].reshape(a1 - a0, 2, span)
    return out
