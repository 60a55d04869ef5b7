"""Smallest invocation of every kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases: fat (FP32 one-block-per-CTA, P = 5, N' = 2048), cluster64 / cluster128
(P-CTA cluster kernel, P = 5), cluster9 (P = 9, non-portable cluster, c128),
ip (in-place-pass c128 kernel, P = 5), wide128 / wide64 (wide-subband
path, N' = 8192 c128 / 16384 c64), nlpr (cbessfm_nlpr), ssfm
(cooperative four-step propagator), rx (receiver symbols + SNR), coeff
(coefficient grid transform). Each case runs one launch (two blocks for the
block kernels) and checks the output is finite."""
import os
import sys
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import torch

import paper_2409_14489_b200 as pb
from conftest import golden


def _block_kernel(kernel, dtype, name="cfg2_nsb5", blocks=(0, 2)):
    os.environ["CBESSFM_KERNEL"] = kernel
    g = golden(name)
    ct = torch.complex64 if dtype == "c64" else torch.complex128
    x = torch.from_numpy(np.vstack([g.wave.x, g.wave.y])[None]).cuda().to(ct)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        # only the launched blocks' kept span is written: start from zeros
        out = pb.run_dbp_tensor(x, g.cfg, g.coeffs, g.wave.sample_rate, block_range=blocks,
                                out=torch.zeros_like(x))
    torch.cuda.synchronize()
    plan = pb.get_plan(g.cfg, g.wave.sample_rate, g.coeffs, dtype)
    return plan.info().kernel_name, out


def case_fat():
    return _block_kernel("fat", "c64")


def case_cluster64():
    return _block_kernel("cluster", "c64")


def case_cluster128():
    return _block_kernel("cluster", "c128")


def case_cluster9():
    return _block_kernel("cluster", "c128", name="cfg1_nsb9_st3")


def case_ip():
    return _block_kernel("ip", "c128")


def case_wide128():
    # wide-subband path (csrc/cbessfm_wide.cu), N' = 8192 at c128
    return _block_kernel("cluster", "c128", name="wide_nsb2", blocks=(0, 2))


def case_wide64():
    # wide-subband path, N' = 16384 at c64
    return _block_kernel("cluster", "c64", name="wide_nsb1", blocks=(0, 2))


def case_nlpr():
    from conftest import GOLDEN, load_coeffs
    d = np.load(GOLDEN / "nlpr_kat.npz")
    c = load_coeffs(d)
    subs = [pb.DualPolWaveform(d["sx"][i], d["sy"][i], 32e9) for i in range(2)]
    out = pb.nlpr_step(subs, pb.build_mimo_transfer(c, 256), 1.0, 1e-3)
    return "cbessfm_nlpr", torch.from_numpy(np.stack([o.x for o in out]))


def case_ssfm():
    from paper_2409_14489_b200 import channel as ch
    from paper_2409_14489_b200.config import LinkConfig
    from paper_2409_14489_b200.synth import gaussian_wdm
    lk = LinkConfig(num_spans=1, span_length_km=80.0, gamma_w_km=1.3)
    steps = ch.span_step_sizes(lk, ch.SimSettings(step_km=20.0), 1e-3)
    x = torch.from_numpy(gaussian_wdm(1 << 12, 512e9, seed=1)[None]).cuda()
    ch.propagate_tensor(x, lk, steps, 512e9)
    torch.cuda.synchronize()
    return "cbessfm_ssfm", x


def case_rx():
    from paper_2409_14489_b200 import receiver as rxm
    from paper_2409_14489_b200.synth import gaussian_wdm

    class Wdm:
        baud_rate, rolloff, launch_power_w = 64e9, 0.05, 10 ** 0.1 * 1e-3
        num_channels, spacing = 5, 100e9
        channel_freqs = (np.arange(5) - 2.0) * 100e9
    x = torch.from_numpy(gaussian_wdm(1 << 14, 512e9, seed=4)).cuda().contiguous()
    sym = rxm.channel_symbols_tensor(x, 512e9, Wdm, Wdm.channel_freqs, 100e9)
    torch.cuda.synchronize()
    return "cbessfm_rx", sym


def case_coeff():
    from paper_2409_14489_b200 import coefficients as co
    geom = co.StepGeometry.spans(1, 80.0)
    c = co.analytic_coefficients(geom, 100e9, 7, 102.4e9, 1e-3, check_convergence=False)
    return "cbessfm_coeff", torch.from_numpy(np.asarray(c))


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    args = sys.argv[1:]
    save = None
    if "--save" in args:
        i = args.index("--save")
        save = args[i + 1]
        del args[i:i + 2]
    names = args or list(CASES)
    outs = {}
    for name in names:
        kname, out = CASES[name]()
        t = out if isinstance(out, torch.Tensor) else torch.as_tensor(out)
        finite = bool(torch.isfinite(torch.view_as_real(t) if t.is_complex() else t).all())
        print(f"{name}: {kname} finite={finite}", flush=True)
        outs[name] = t.detach().cpu().numpy()
        assert finite, name
    if save:
        np.savez(save, **outs)
