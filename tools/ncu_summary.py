"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches <launches.csv>          per-kernel share of device time
  python tools/ncu_summary.py full <prof.ncu-rep>               key counters of a --set full capture
  python tools/ncu_summary.py traffic <prof.ncu-rep> <alpha> [B] per-launch DRAM traffic JSON of a
      tools/prof_replay.py capture (REPS=1: launches qkv, o, fc1, fc2) beside the algorithmic bytes
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
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                     "second": 1e6, "s": 1e6}.get(unit, 1.0)
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


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
          "msecond": 1e3, "%": 1.0}


def traffic(path, alpha, B=1):
    """JSON for bench.ncu_traffic(): dram read/write bytes per launch of the replay capture."""
    import json
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2403_01164_b200 import hg
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rdr = list(csv.reader(io.StringIO(txt)))
    hdr, units = rdr[0], rdr[1]
    H, F = 7168, 28672
    shapes = [("qkv", 3 * H, H), ("o", H, H), ("fc1", F, H), ("fc2", H, F)]
    per = {}
    for (name, N, K), row in zip(shapes, rdr[2:]):
        d, u = dict(zip(hdr, row)), dict(zip(hdr, units))
        val = lambda k: float(d[k].replace(",", "")) * _SCALE.get(u.get(k, ""), 1.0)  # noqa: E731
        p = hg.hg_plan(hg.make_rates(1, 1, 1), N, K, B, 0, hg.FIXED, alpha, 128, 32 << 20)
        per[name] = {"duration_us": round(val("gpu__time_duration.sum"), 3),
                     "dram_read_MB": val("dram__bytes_read.sum") / 1e6,
                     "dram_write_MB": val("dram__bytes_write.sum") / 1e6,
                     "dram_pct_peak": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                     "algorithmic_MB": 2 * K * (p.n_res + p.n_str) / 1e6}
    return json.dumps({"source": f"ncu --set full of tools/prof_replay.py (hg_gemv_replay, alpha={alpha}, B={B}, "
                                 "32 MiB chunks)", "per_launch": per}, indent=1)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "traffic":
        print(traffic(path, float(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 1))
    else:
        print(launches(path) if mode == "launches" else full(path))
