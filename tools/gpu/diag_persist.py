"""Run-to-run determinism of the configs[4] c128 launch: the persistent
cluster kernel against one cluster per block (CBESSFM_PERSIST=0), compared
bit for bit per overlap-save block. Prints the mismatching (waveform, block)
pairs and what the bad spans look like."""
import json
import os
import sys
import warnings
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2409_14489_b200 as pb  # noqa: E402
from paper_2409_14489_b200.synth import gaussian_wdm_device  # noqa: E402
from conftest import golden  # noqa: E402

batch = int(os.environ.get("DIAG_BATCH", "64"))
reps = int(os.environ.get("DIAG_REPS", "4"))
g = golden("cfg2_nsb5")
rate, n = 512e9, 1 << 23
cuda = torch.device("cuda:0")
x = torch.empty((batch, 2, n), dtype=torch.complex128, device=cuda)
for w in range(batch):
    gaussian_wdm_device(n, rate, 1000 + w, cuda, out=x[w])
keep = g.cfg.block_size - g.cfg.overlap


def run(persist):
    if persist is None:
        os.environ.pop("CBESSFM_PERSIST", None)
    else:
        os.environ["CBESSFM_PERSIST"] = persist
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        out = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate)
    torch.cuda.synchronize()
    return out


def report(tag, out, ref):
    a = torch.view_as_real(out).view(torch.int64)
    b = torch.view_as_real(ref).view(torch.int64)
    bad = (a != b).any(dim=-1).any(dim=1)          # [batch, n]
    nbad = int(bad.sum())
    print(f"{tag}: {nbad} differing samples", flush=True)
    if not nbad:
        return
    idx = bad.nonzero()
    blocks = {}
    for w, t in idx.cpu().numpy()[:: max(1, len(idx) // 200000)]:
        blocks.setdefault((int(w), int(t) // keep), 0)
        blocks[(int(w), int(t) // keep)] += 1
    print(f"  {len(blocks)} blocks: {sorted(blocks)[:40]}")
    for (w, bl) in sorted(blocks)[:6]:
        s = slice(bl * keep, min(n, (bl + 1) * keep))
        o, r = out[w, :, s], ref[w, :, s]
        d = (o - r).abs()
        frac = float((d > 0).double().mean())
        print(f"  wv {w} block {bl}: differing frac {frac:.3f}, |out| rms {float(o.abs().pow(2).mean().sqrt()):.3e}, "
              f"|ref| rms {float(r.abs().pow(2).mean().sqrt()):.3e}, max |d| {float(d.max()):.3e}, "
              f"finite {bool(torch.isfinite(torch.view_as_real(o)).all())}")
        # where inside the block do the differences sit (polyphase rank = t % 5)?
        dd = (d > 0).any(dim=0).cpu().numpy()
        t = np.arange(s.start, s.stop)[dd] - (bl * keep - (g.cfg.overlap // 2))
        print(f"    ranks hit (t % 5): {np.bincount(t % 5, minlength=5).tolist()}, first/last t {t.min()} {t.max()}")


ref = run("0")
for r in range(reps):
    ref2 = run("0")
    report(f"one cluster per block, rerun {r}", ref2, ref)
    del ref2
for xf in os.environ.get("DIAG_XFLAGS", "0").split(","):
    os.environ["CBESSFM_XFLAGS"] = xf
    for r in range(reps):
        out = run(None)
        report(f"persistent xflags={xf} run {r}", out, ref)
        del out
