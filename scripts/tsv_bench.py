"""Fact-file ingestion and TSV output: device (tsv.cu) vs the reference's
io.hpp (oracle/_ref, one host thread), on the C2 edge file and on C2's
Reach output (python scripts/tsv_bench.py)."""
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from oracle.bindings import RefOracle  # noqa: E402
from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

ref = RefOracle()
tmp = Path(tempfile.mkdtemp())
edges = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
t = al.tuple_array(2, edges)
p = tmp / "edge.tsv"
al.to_tsv(t)  # warm-up
t0 = time.perf_counter()
text = al.to_tsv(t)  # raw (non-canonical) rows are formatted as given
p.write_text(text)
t1 = time.perf_counter()
print(f"edge file: {len(edges)} rows, {len(text)/1e6:.1f} MB written in {t1-t0:.3f} s (device to_tsv + file write)")
for rep in range(2):
    t0 = time.perf_counter()
    r = al.read_facts(p, 2)
    t1 = time.perf_counter()
    print(f"device read_facts: {r.count()} canonical rows in {(t1-t0)*1e3:.1f} ms ({len(text)/(t1-t0)/1e9:.2f} GB/s of text)")
t0 = time.perf_counter()
rc, rr = ref.read_facts(p, 2)
t1 = time.perf_counter()
print(f"reference read_facts: {len(rr)} rows in {(t1-t0)*1e3:.1f} ms; equal: {np.array_equal(rr, r.data)}")
e = al.engine("reach")
e.load_edb_tsv("Edge", p)
e.run()
n = e.relation_count("Reach")
for rep in range(2):
    t0 = time.perf_counter()
    out = e.relation_tsv("Reach")
    t1 = time.perf_counter()
    print(f"device relation_tsv(Reach): {n} rows -> {len(out)/1e9:.2f} GB in {t1-t0:.3f} s ({len(out)/(t1-t0)/1e9:.2f} GB/s)")
sample = e.relation("Reach").data[:2_000_000]
t0 = time.perf_counter()
rb = ref.to_tsv(sample, 2)
t1 = time.perf_counter()
print(f"reference to_tsv on a 2M-row sample: {(t1-t0)*1e3:.1f} ms -> extrapolated {(t1-t0)*n/2e6:.1f} s for {n} rows; "
      f"sample bytes equal: {rb == out[:len(rb)]}")
