import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2311_02206_b200 import arraylog as al
from paper_2311_02206_b200 import workloads as W
e = al.engine("reach"); e.load_edb("Edge", al.tuple_array(2, W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1))); e.run()
log = np.array(e.iter_log("Reach"), dtype=np.float64)
d, j = log[:, 0], log[:, 1]
for th in (1e3, 1e4, 5e4, 1e5, 3e5, 1e6):
    m = d < th
    print(f"delta < {th:9.0f}: {m.sum():4d} iterations, J share {j[m].sum()/j.sum():.4f}")
print("first/last deltas", d[:3], d[-5:], "argmax", d.argmax())
