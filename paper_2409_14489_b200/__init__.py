"""B200-native CB-ESSFM digital backpropagation (arXiv 2409.14489 hot path).

Drop-in for the reference package's DBP entry point and config objects
(fiberdbp/__init__.py:9-31, the subset on the hot path):

    run_dbp(w, cfg, coeffs=None, counter=None)      dbp.py:437-478

plus run_dbp_sets (many CoefficientSets on one waveform in one launch, the
evaluations optimize_coefficients makes one run_dbp call at a time).

The coupled-band split-step pipeline runs as one fused sm_100a kernel per
launch (csrc/), reached through the C ABI in include/cbessfm.h; the host
planner (planner.py) builds the FP64 tables and the block/shard schedule.
"""

from .complexity import (CostCounter, CostReport, cb_essfm_cost,
                         count_runtime_multiplies, essfm_time_domain_cost)
from .config import (VARIANTS, CoefficientSet, DbpConfig, DualPolWaveform,
                     LinkConfig)
from .engine import (DbpEngine, MimoTransfer, SetEvaluator, build_mimo_transfer,
                     channel_memory_samples, get_plan, gvd_step, launch,
                     nlpr_step, run_dbp, run_dbp_sets, run_dbp_sets_tensor,
                     run_dbp_tensor)
from .planner import (BlockSchedule, EngineTables, Shard, build_tables,
                      plan_shards)

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")]
