"""Writes tests/golden/scale_digests.json: the full-scale records of the
benchmark configs (C2, C3 W=1000, C5), produced on a B200 by
tests/test_gpu_scale.scale_records after its checks passed:

  * rows strictly increasing, Σ Δ-history = |F|, ΣJ = Σ indeg(m) (TC);
  * resident device loop == host-driven loop == native partitioned driver
    over P loopback ranks (count, digest, iterations, ΣJ, Δ-history hash).

The CPU reference engine cannot run these sizes (hours, more
than the host's RAM); bounded samples of the same generators are compared
with it byte for byte in tests/test_gpu_scale.py.

    python tests/golden/make_scale_golden.py [config ...]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from tests.test_gpu_scale import GOLD, SCALE, scale_records  # noqa: E402


def main():
    names = sys.argv[1:] or sorted(SCALE)
    gold = json.loads(GOLD.read_text()) if GOLD.exists() else {}
    for name in names:
        recs = scale_records(name)
        base = recs["resident"]
        bad = {k: r for k, r in recs.items() if r != base}
        if bad:
            raise SystemExit(f"{name}: modes disagree: {bad} vs {base}")
        gold[name] = {"record": base, "checked": sorted(recs)}
        print(name, json.dumps(gold[name]), flush=True)
    GOLD.write_text(json.dumps(gold, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
