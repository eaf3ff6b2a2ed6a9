import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2311_02206_b200 import arraylog as al
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 24
a = np.random.default_rng(1).integers(0, 1 << 23, size=(n, 2), dtype=np.uint64)
al.canonicalize(al.tuple_array(2, a))
