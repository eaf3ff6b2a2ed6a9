"""Key metrics + top stall reasons of ncu --set full reports -> JSON
(python scripts/ncu_summary.py out.json name=report.ncu-rep ...)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "launch__occupancy_limit_registers"]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = dict(zip(h, v))
        u = dict(zip(h, units))
        rec = {k: (d.get(k, "") + (" " + u[k] if u.get(k) else "")).strip() for k in KEYS}
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k]) for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and d[k] not in ("", "0")}
        tot = sum(st.values()) or 1
        rec["top_stalls_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(st.items(), key=lambda x: -x[1])[:6]}
        res.append(rec)
    return res


if __name__ == "__main__":
    out = {}
    for arg in sys.argv[2:]:
        name, path = arg.split("=", 1)
        out[name] = summarize(path)
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])
