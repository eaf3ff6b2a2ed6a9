"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch)
into per-kernel-class shares: profiles/<tag>_launches.md and the measured
DRAM traffic per launch that bench.py reports as roofline.traffic
(profiles/ncu_traffic.json).  python scripts/summarize_launches.py
gpurun_out/launches.csv <tag>"""
import collections
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CLASSES = [  # kernel-name substring -> bench/profiler class (ctx.h KClass)
    ("onesweep_kernel", "sort_pass"), ("onesweep_pipe_kernel", "sort_pass"), ("radix_hist", "sort_hist"),
    ("radix_bases", "sort_hist"),
    ("loop_probe_kernel", "join_probe"), ("join_probe_kernel", "join_probe"), ("loop_count_kernel", "join_probe"),
    ("loop_expand_insert", "join_insert"), ("loop_insert_keys", "join_insert"), ("loop_expand_route", "exchange"),
    ("loop_route_keys", "exchange"), ("loop_peer_sync", "loop_ctl"),
    ("loop_scan_kernel", "select"), ("scan_tiles", "select"), ("apply_offsets", "select"), ("select_kernel", "select"),
    ("loop_materialize_insert", "join_insert"), ("loop_select_insert", "join_insert"),
    ("loop_materialize_temp", "join_materialize"), ("join_materialize_kernel", "join_materialize"),
    ("merge_disjoint", "diff_merge"), ("diff_merge", "diff_merge"), ("diff_flags", "difference"),
    ("index_insert", "index_build"), ("table_", "index_build"),
    ("loop_gate", "loop_ctl"), ("loop_end", "loop_ctl"), ("loop_select_cand", "loop_ctl"),
]


def cls_of(name):
    for sub, c in CLASSES:
        if sub in name:
            return c
    return "other"


def main():
    path, tag = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    per = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        v = float(d["Metric Value"].replace(",", "") or 0)
        unit = d.get("Metric Unit", "")
        if d["Metric Name"].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        if d["Metric Name"] == "gpu__time_duration.sum":
            v *= {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6}.get(unit, 1)
        per[d["ID"]]["name"] = d["Kernel Name"]
        per[d["ID"]][d["Metric Name"]] = v
    agg = collections.defaultdict(lambda: {"launches": 0, "ns": 0.0, "dram": 0.0, "kernels": set()})
    for k in per.values():
        c = cls_of(k["name"])
        a = agg[c]
        a["launches"] += 1
        a["ns"] += k.get("gpu__time_duration.sum", 0)
        a["dram"] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        a["kernels"].add(k["name"].split("(")[0].replace("gd::<unnamed>::", "").replace("void ", "")[:60])
    total = sum(a["ns"] for a in agg.values())
    lines = [f"# ncu launch list summary ({tag})", "",
             f"Source: `{path}` ({len(per)} launches, cold-cache and serialised by ncu: compare shares, "
             "not absolute times).", "",
             "| class | launches | total ms | share | DRAM GB | DRAM GB per launch | kernels |", "|---|---|---|---|---|---|---|"]
    for c, a in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        lines.append(f"| {c} | {a['launches']} | {a['ns'] / 1e6:.2f} | {100 * a['ns'] / total:.1f}% | "
                     f"{a['dram'] / 1e9:.2f} | {a['dram'] / a['launches'] / 1e9:.4f} | {', '.join(sorted(a['kernels']))} |")
    out = ROOT / "profiles" / f"{tag}_launches.md"
    out.write_text("\n".join(lines) + "\n")
    tp = ROOT / "profiles" / "ncu_traffic.json"
    traffic = json.loads(tp.read_text()) if tp.exists() else {}
    for c, a in agg.items():
        traffic[c] = {"dram_bytes": a["dram"] / a["launches"], "launches": a["launches"],
                      "source": f"profiles/{tag}_launches.md (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                "mean per launch)"}
    tp.write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
