"""C4 calibration sweep: cspa_local(n, 362000, 1140000, module) at several
variable counts n, one B200, EDB resident.  Prints IDB sizes (VF / VA / MA),
iterations, join tuples and device time per n, to pick the n whose outputs
are closest to httpd's (VF 1.36e6, VA 2.34e8, MA 8.89e7; PAPER.md:603 via
SURVEY §8d).  Each n runs in its own process under a timeout so a density
past the explosion point cannot take the box down:

    python scripts/cspa_calibrate.py 1.5 1.4 1.3 [--module 256]
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def one(n: int, module: int) -> None:
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    from paper_2311_02206_b200 import arraylog as al
    from paper_2311_02206_b200 import workloads as W

    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = al.Context(0, s.cuda_stream)
    a, d = W.cspa_local(n, 362_000, 1_140_000, module, 1)
    dev = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int64)).cuda() for k, v in
           (("assign", a), ("dereference", d))}
    times = []
    for rep in range(2):
        e = al.engine("cspa", ctx=ctx)
        for k, v in dev.items():
            e.load_edb_device(k, v.data_ptr(), v.numel() // 2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        e.run()
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        st = e.raw_stats()
        sizes = {r: e.relation_count(r) for r in e.idb_relations()}
        e.close()
    print(json.dumps({"n": n, "module": module, "idb_sizes": sizes, "iterations": int(st.iterations),
                      "join_tuples": int(st.join_tuples), "time_s": times}), flush=True)


def main():
    args = [x for x in sys.argv[1:] if not x.startswith("--")]
    module = 256
    if "--module" in sys.argv:
        module = int(sys.argv[sys.argv.index("--module") + 1])
        args.remove(str(module))
    if "--one" in sys.argv:
        one(int(args[0]), module)
        return
    for x in args:
        n = int(float(x) * 1e6)
        try:
            r = subprocess.run([sys.executable, __file__, "--one", str(n), "--module", str(module)],
                               capture_output=True, text=True, timeout=180)
            line = (r.stdout.strip().splitlines() or [""])[-1]
            print(line if line.startswith("{") else json.dumps({"n": n, "error": r.stderr.strip()[-300:]}), flush=True)
        except subprocess.TimeoutExpired:
            print(json.dumps({"n": n, "error": "timeout 180 s"}), flush=True)


if __name__ == "__main__":
    main()
