"""Run-to-run determinism of the configs[4] c64 launch (one-block kernel) and of the
pipelined host path on one waveform: N launches compared bit for bit with the first."""
import os
import sys
import warnings
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2409_14489_b200 as pb  # noqa: E402
from paper_2409_14489_b200.synth import gaussian_wdm_device  # noqa: E402
from conftest import golden  # noqa: E402

reps = int(os.environ.get("DIAG_REPS", "20"))
g = golden("cfg2_nsb5")
rate, n, batch = 512e9, 1 << 23, 64
cuda = torch.device("cuda:0")
x = torch.empty((batch, 2, n), dtype=torch.complex64, device=cuda)
for w in range(batch):
    gaussian_wdm_device(n, rate, 1000 + w, cuda, out=x[w])


def run():
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        out = pb.run_dbp_tensor(x, g.cfg, g.coeffs, rate)
    torch.cuda.synchronize()
    return out


ref = run()
bad = 0
for r in range(reps):
    out = run()
    nb = int((torch.view_as_real(out).view(torch.int32) != torch.view_as_real(ref).view(torch.int32)).sum())
    bad += nb > 0
    if nb:
        print(f"c64 launch {r}: {nb} words differ", flush=True)
    del out
print(f"c64 one-block kernel: {reps - bad}/{reps} launches bit-identical to the first")

# the host pipeline (cluster kernel, chunked) on one c128 and one c64 waveform
for dt in ("c128", "c64"):
    eng = pb.DbpEngine(g.cfg, g.coeffs, rate, dtype=dt, device=0)
    hx = x[:1].to(eng.torch_dtype).cpu().pin_memory()
    outs = []
    bad = 0
    for r in range(reps):
        ho = torch.empty_like(hx).pin_memory()
        eng.run_host(hx, ho, chunks=[1, 2, 4, 8][r % 4])
        torch.cuda.synchronize()
        if r == 0:
            first = ho.clone()
        else:
            bad += not torch.equal(ho, first)
    print(f"{dt} run_host (1/2/4/8 chunks): {reps - bad}/{reps} bit-identical to the first")
