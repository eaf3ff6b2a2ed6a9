"""Dumps C2's per-iteration log (Δ in, J, N, D, |full|) to
gpurun_out/c2_iter_log.npy for the per-iteration cost analysis
(python scripts/iter_log_dump.py)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

edges = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
e = al.engine("reach")
e.load_edb("Edge", al.tuple_array(2, edges))
e.run()
log = np.array([list(r) for r in e.iter_log("Reach")], dtype=np.int64)
np.save("gpurun_out/c2_iter_log.npy", log)
print("iterations", len(log), "shape", log.shape)
