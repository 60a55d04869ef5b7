import sys, warnings, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from conftest import CASES, golden, rel_rms
import paper_2409_14489_b200 as pb
for name in CASES:
    g = golden(name)
    for dt in ("c128", "c64"):
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                o = pb.run_dbp(g.wave, g.cfg, g.coeffs, dtype=dt)
            torch.cuda.synchronize()
            print(name, dt, "%.3e" % rel_rms(np.vstack([o.x, o.y]), g.out), flush=True)
        except Exception as e:
            print(name, dt, "ERR", repr(e)[:300], flush=True)
