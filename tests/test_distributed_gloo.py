"""Multi-process (world_size 2, gloo, CPU) coverage of the shard/halo
planner and the final gather (paper_2409_14489_b200/distributed.py). The
per-shard compute is the numpy oracle run on exactly the halo'd slice a rank
would upload, so the sharded result must equal the unsharded one bit for
bit."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import golden
from oracle import cbessfm_oracle as orc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_compute(cfg, rate, coeffs):
    def run(x_slice, work, n):
        import torch
        x_slice = x_slice.numpy()
        outs = []
        for wf in x_slice:
            full = np.zeros((2, n), dtype=complex)
            idx = (work.in_origin + np.arange(x_slice.shape[-1])) % n
            full[:, idx] = wf
            b0, b1 = work.shard.blocks
            res = orc.run_cb_blocks(full, cfg, rate, coeffs, b0, b1)
            outs.append(res[:, work.out_begin:work.out_end])
        return torch.from_numpy(np.stack(outs))
    return run


def _worker(rank, world, port, name, batch, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2409_14489_b200.distributed import run_distributed
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = golden(name)
        base = np.vstack([g.wave.x, g.wave.y])
        x = np.stack([np.roll(base, 97 * b, axis=-1) for b in range(batch)])
        out = run_distributed(x, g.cfg.block_size, g.cfg.overlap,
                              _oracle_compute(g.cfg, g.wave.sample_rate, g.coeffs))
        if rank == 0:
            out = out.numpy()
            ref = np.stack([orc.run_cb_blocks(xb, g.cfg, g.wave.sample_rate, g.coeffs)
                            for xb in x])
            q.put(("ok", bool(np.array_equal(out, ref)),
                   float(np.max(np.abs(out - ref)))))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e), 0.0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,batch", [("cfg2_nsb5", 1),      # time shards
                                        ("cfg1_nsb3_st2", 1),  # time shards, many blocks
                                        ("cfg1_nsb2_frac", 3)])  # waveform shards
def test_two_rank_shards_reassemble_exactly(name, batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, batch, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    status, same, err = q.get(timeout=10)
    assert status == "ok", same
    assert same, f"max abs deviation {err}"
