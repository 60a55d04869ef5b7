"""Multi-GPU CB-ESSFM: shard/halo planner execution and the final gather.

One process per GPU (torch.distributed, NCCL backend on B200s). The
overlap-save schedule of a batch of waveforms is partitioned by
``planner.plan_shards``: whole waveforms per rank when there are at least as
many waveforms as ranks, otherwise contiguous block ranges of a waveform
(time shards). A time shard uploads only its circular input slice -- its
output span plus an N_ov/2 halo on each side, exactly the samples its blocks
read (dbp.py:473-475) -- so ranks never communicate inside the step loop.
The only collective is the final gather of the kept samples to rank 0
(SURVEY.md 8(e)), done on the device in the compute dtype.

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


def circular_slice(x, origin: int, length: int):
    """x[..., (origin + arange(length)) mod n] for a torch tensor, on x's
    device (the halo'd input a time shard reads; planner.gather_slice is
    the numpy twin)."""
    import torch
    n = x.shape[-1]
    if origin == 0 and length == n:
        return x
    idx = (torch.arange(length, device=x.device) + origin) % n
    return x.index_select(-1, idx)


def gpu_compute(engine):
    """Compute callable running the fused kernel of a DbpEngine on a
    halo'd slice: takes a [Bw, 2, L] tensor (host or device), returns the
    kept samples [Bw, 2, o1 - o0] as a DEVICE tensor in the engine's dtype
    (no host round trip, no upcast)."""
    import torch

    from .engine import launch

    def run(x_slice, work: ShardWork, n: int):
        x = torch.as_tensor(x_slice).to(engine.device, engine.torch_dtype)
        out = torch.empty((x.shape[0], 2, work.out_end - work.out_begin),
                          dtype=engine.torch_dtype, device=engine.device)
        with torch.cuda.device(engine.device):
            launch(engine.plan, x, out, n=n, block_range=work.shard.blocks,
                   in_origin=work.in_origin, out_origin=work.out_begin)
        return out

    run.dtype = engine.torch_dtype
    run.device = engine.device
    return run


def run_distributed(x, block_size: int, overlap: int, compute, group=None):
    """Shard a [B, 2, n] batch over the process group, run ``compute`` on
    each rank's halo'd slice, and gather the kept samples on rank 0.

    ``x`` is a torch tensor (HBM or host) or a numpy array; every rank
    passes the same batch (or at least the samples its shard reads).
    ``compute(slice, work, n)`` returns the rank's kept samples as a torch
    tensor; its ``dtype`` / ``device`` attributes (set by
    :func:`gpu_compute`) fix the gather's dtype and device, otherwise x's
    are used. The gather is one ``dist.gather`` of the pieces viewed as
    real pairs, padded to the largest shard: on NCCL it stays in HBM in the
    compute dtype. Returns the assembled [B, 2, n] tensor on rank 0 and None
    elsewhere."""
    import torch
    import torch.distributed as dist

    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    batch, _, n = x.shape
    dtype = getattr(compute, "dtype", x.dtype)
    device = getattr(compute, "device", x.device)
    work = shard_work(n, block_size, overlap, batch, world, rank)
    w0, w1 = work.shard.waveforms
    if work.empty:
        piece = torch.zeros((0, 2, 0), dtype=dtype, device=device)
    else:
        xs = circular_slice(x[w0:w1], work.in_origin, work.in_length)
        piece = compute(xs, work, n).to(device, dtype)

    # final gather (the only collective): every piece padded to the largest
    # shard, real-pair view (gloo has no complex collectives), rank 0 assembles
    sizes = [shard_work(n, block_size, overlap, batch, world, r) for r in range(world)]
    max_elems = max(1, max((s.shard.waveforms[1] - s.shard.waveforms[0]) * 2 *
                           (s.out_end - s.out_begin) for s in sizes))
    rdt = torch.view_as_real(torch.zeros(1, dtype=dtype)).dtype
    buf = torch.zeros(2 * max_elems, dtype=rdt, device=device)
    if piece.numel():
        buf[:2 * piece.numel()] = torch.view_as_real(piece.contiguous()).reshape(-1)
    glist = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, glist, dst=0, group=group)
    if rank != 0:
        return None
    out = torch.zeros((batch, 2, n), dtype=dtype, device=device)
    for r, s in enumerate(sizes):
        if s.empty:
            continue
        a0, a1 = s.shard.waveforms
        span = s.out_end - s.out_begin
        vals = torch.view_as_complex(glist[r][:2 * (a1 - a0) * 2 * span].view(-1, 2))
        out[a0:a1, :, s.out_begin:s.out_end] = vals.view(a1 - a0, 2, span)
    return out
