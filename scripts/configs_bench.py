"""Bench-style JSON lines for the other BASELINE configs on one B200 (EDB
resident in HBM, device time with CUDA events, best of 3 after warm-up):
python scripts/configs_bench.py > profiles/r1_configs.jsonl"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

_s = torch.cuda.Stream()  # a real stream: the events below are recorded where the engine runs
torch.cuda.set_stream(_s)
ctx = al.Context(0, _s.cuda_stream)
names = sys.argv[1:] or ["c1_tc_rand", "c3_sg_tree", "c3_sg_tree_w1000", "c3_sg_tree_w4000", "c4_cspa", "c5_tc_dag"]
for name in names:
    cfg = W.CONFIGS[name]
    edbs = cfg["gen"]()
    dev = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int64)).cuda() for k, v in edbs.items()}
    times, stats = [], None
    for rep in range(4):
        e = al.engine(cfg["program"], ctx=ctx)
        for k, v in edbs.items():
            e.load_edb_device(k, dev[k].data_ptr(), len(v))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(_s)
        e.run()
        b.record(_s)
        torch.cuda.synchronize()
        if rep:
            times.append(a.elapsed_time(b))
        s = e.raw_stats()
        stats = (s.iterations, s.join_tuples, {n: e.relation_count(n) for n in e.idb_relations()})
        e.close()
    ms = min(times)
    it, jt, sizes = stats
    print(json.dumps({"workload": name, "desc": cfg["desc"], "program": cfg["program"],
                      "edb_rows": {k: int(len(v)) for k, v in edbs.items()}, "time_to_fixpoint_s": ms / 1e3,
                      "join_tuples": int(jt), "join_tuples_per_s": jt / (ms / 1e3), "iterations": int(it),
                      "idb_sizes": sizes, "device": "1x B200", "timing": "CUDA events, best of 3 after warm-up",
                      "data": "synthetic (paper_2311_02206_b200/workloads.py)"}), flush=True)
