"""rel L2 of every golden DBP case against the reference output, c64 and
c128, through the library CBESSFM_LIB points at (precision A/B of kernel
variants): python tools/c64_errors.py"""
import sys
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np

from conftest import golden, rel_rms
import paper_2409_14489_b200 as pb

CASES = ("cfg1_nsb1", "cfg1_nsb2_frac", "cfg1_nsb3_st2", "cfg1_nsb9_st3", "cfg2_nsb5",
         "cfg4_nsb5_st1", "cfg4_nsb5_st10", "cfg4_nsb5_st50")
for name in CASES:
    g = golden(name)
    row = []
    for dtype in ("c64", "c128"):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            out = pb.run_dbp(g.wave, g.cfg, g.coeffs, dtype=dtype)
        row.append(f"{dtype} {rel_rms(np.vstack([out.x, out.y]), g.out):.3e}")
    print(f"{name:16s} " + "  ".join(row), flush=True)
