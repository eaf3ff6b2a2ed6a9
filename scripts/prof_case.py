"""One fixpoint run of a named case for ncu captures
(python scripts/prof_case.py chain|c2|c2dl|c2log|<workloads.CONFIGS name>|cspa:<n>)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "chain"
if case in W.CONFIGS or case.startswith("cspa:"):
    if case.startswith("cspa:"):
        prog = "cspa"
        edbs = dict(zip(("assign", "dereference"), W.cspa_local(int(float(case[5:])), 362_000, 1_140_000, 256, 1)))
    else:
        prog, edbs = W.CONFIGS[case]["program"], W.CONFIGS[case]["gen"]()
    e = al.engine(prog)
    for k, v in edbs.items():
        e.load_edb(k, al.tuple_array(2, np.ascontiguousarray(v)))
    e.run()
    print("iterations", e.stats().iterations, {r: e.relation_count(r) for r in e.idb_relations()})
    sys.exit(0)
if case == "chain":
    edges = np.stack([np.arange(2999), np.arange(1, 3000)], 1).astype(np.uint64)
else:
    edges = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
e = al.engine("reach")
e.load_edb("Edge", al.tuple_array(2, edges))
e.run()
print("iterations", e.stats().iterations, "|Reach|", e.relation_count("Reach"))
if case == "c2dl":  # plus the host download (byte-offset packing on the device)
    rows = e.relation("Reach").data
    print("downloaded", rows.shape)
if case == "c2log":
    log = e.iter_log("Reach")
    big = sorted(range(len(log)), key=lambda i: -log[i][1])[:10]
    for i in sorted(big):
        print(i, log[i])
    js = np.array([r[1] for r in log])
    print("J quantiles", np.percentile(js, [10, 50, 90, 99, 100]))
