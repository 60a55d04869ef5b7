"""Checked build: the stand-in for compute-sanitizer (closed on this GPU
pool). libcbessfm_checked.so is the same code compiled with -DCB_CHECKED:
every kernel first fills its dynamic shared memory with a NaN pattern, and
global / shared / cluster indices are bounds-checked with a trap
(csrc/cbessfm_kernel.cuh CB_POISON_SMEM, CB_CHECK). Every kernel family's
smallest case (tools/sanitize_cases.py) must run without a trap, produce
finite output and match the unchecked build bit for bit: a read of a slot
no pass wrote, or read before its writer's barrier (a race), would carry
the poison into the result.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

LIB = ROOT / "paper_2409_14489_b200" / "libcbessfm_checked.so"
CASES = ["fat", "cluster64", "cluster128", "cluster9", "ip", "wide128", "wide64", "nlpr", "ssfm",
         "rx", "coeff"]


def _checked_lib():
    if not LIB.exists():
        res = subprocess.run([sys.executable, str(ROOT / "paper_2409_14489_b200" / "build.py"),
                              "--variant", "checked", "--define", "CB_CHECKED"],
                             cwd=ROOT, capture_output=True, text=True, timeout=1800)
        assert res.returncode == 0, res.stderr[-3000:]
    return LIB


def _run(lib, out, cases):
    env = dict(os.environ)
    env.pop("CBESSFM_KERNEL", None)
    if lib is not None:
        env["CBESSFM_LIB"] = str(lib)
    res = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_cases.py"), *cases,
                          "--save", str(out)], cwd=ROOT, capture_output=True, text=True,
                         timeout=1800, env=env)
    assert res.returncode == 0, (res.stdout[-2000:], res.stderr[-3000:])
    return np.load(out)


def test_checked_build_matches_bit_for_bit(cuda, tmp_path):
    lib = _checked_lib()
    plain = _run(None, tmp_path / "plain.npz", CASES)
    checked = _run(lib, tmp_path / "checked.npz", CASES)
    for c in CASES:
        a, b = plain[c], checked[c]
        assert np.all(np.isfinite(b.view(np.float64) if b.dtype.kind == "c" else b)), c
        assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8)), c


def test_repeated_concurrent_launches_are_deterministic(cuda):
    # a race shows up as run-to-run differences: the same batch, launched on
    # three streams at once with other work in flight, must give identical bits
    import torch
    from conftest import golden
    import paper_2409_14489_b200 as pb
    g = golden("cfg2_nsb5")
    for dtype, ct in (("c128", torch.complex128), ("c64", torch.complex64)):
        x = torch.from_numpy(np.vstack([g.wave.x, g.wave.y])[None]).to(cuda).to(ct)
        x = x.expand(6, 2, x.shape[-1]).contiguous()
        eng = pb.DbpEngine(g.cfg, g.coeffs, g.wave.sample_rate, dtype=dtype)
        ref = eng.run_device(x)
        torch.cuda.synchronize()
        streams = [torch.cuda.Stream() for _ in range(3)]
        outs = []
        for s in streams:
            with torch.cuda.stream(s):
                outs.append(eng.run_device(x, stream=s))
        torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o, ref)
        for w in range(1, 6):
            assert torch.equal(ref[w], ref[0])
