"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches <launches.csv>          per-kernel share of device time
  python tools/ncu_summary.py full <prof.ncu-rep>               key counters of a --set full capture
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "")
            scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1.0)
            rows.append((r["Kernel Name"], v * scale))
    tot = sum(t for _, t in rows) or 1.0
    agg = defaultdict(lambda: [0, 0.0])
    for k, t in rows:
        name = k.split("(")[0]
        agg[name][0] += 1
        agg[name][1] += t
    out = [f"launches: {len(rows)}, total device time {tot/1e3:.3f} ms (ncu: serialized, cold-cache)", "",
           "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{name[:90]}` | {n} | {t:.1f} | {t/tot:.1%} | {t/n:.2f} |")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "l1tex__t_bytes.sum", "dram__bytes_read.sum.per_second"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rdr = list(csv.reader(io.StringIO(txt)))
    if len(rdr) < 3:
        return "no data"
    hdr = rdr[0]
    units = rdr[1]
    out = []
    for row in rdr[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        out.append(f"### {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                out.append(f"- {k}: {d[k]} {u.get(k, '')}")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
