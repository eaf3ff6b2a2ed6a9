"""Per-iteration J / N / D of C4 (CSPA) per relation."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402
cfg = W.CONFIGS["c4_cspa"]
edbs = cfg["gen"]()
e = al.engine("cspa")
for k, v in edbs.items():
    e.load_edb(k, al.tuple_array(2, v))
e.run()
for r in ("ValueFlow", "MemoryAlias", "ValueAlias"):
    log = np.array(e.iter_log(r), dtype=np.float64)
    print(r, "iters", len(log), "sum J %.3g" % log[:, 1].sum(), "sum N %.3g" % log[:, 2].sum(),
          "max J %.3g" % log[:, 1].max(), "max N %.3g" % log[:, 2].max(), "sum D %.3g" % log[:, 3].sum())
print(e.stats().phase_seconds)
