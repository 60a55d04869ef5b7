import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
from conftest import golden, rel_rms
from oracle import cbessfm_oracle as orc
import paper_2409_14489_b200 as pb
from paper_2409_14489_b200.synth import gaussian_wdm
g = golden("cfg2_nsb5"); rate = g.wave.sample_rate
field = gaussian_wdm(1 << 20, rate, seed=7)
ref = orc.run_cb_blocks(field, g.cfg, rate, g.coeffs)
x = torch.from_numpy(field[None]).cuda().to(torch.complex64)
sched = pb.BlockSchedule(1 << 20, g.cfg.block_size, g.cfg.overlap)
keep = g.cfg.block_size - g.cfg.overlap
for kernel in ("fat", "cluster"):
    os.environ["CBESSFM_KERNEL"] = kernel
    for rng in ((0, 3), (0, 143)):
        out = torch.zeros_like(x)
        pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate, out=out, block_range=rng)
        got = out[0].to(torch.complex128).cpu().numpy()
        a, b = rng[0] * keep, min(rng[1] * keep, 1 << 20)
        e = rel_rms(got[:, a:b], ref[:, a:b])
        # per-block errors
        errs = [rel_rms(got[:, k*keep:min((k+1)*keep, 1<<20)], ref[:, k*keep:min((k+1)*keep,1<<20)]) for k in range(*rng)]
        bad = [k for k, ee in zip(range(*rng), errs) if ee > 1e-5]
        print(kernel, rng, f"{e:.3e}", "bad blocks:", bad[:20], len(bad))
