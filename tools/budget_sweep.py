"""Throughput vs GPU memory budget (Fig. 8 analogue; NEXT(3) of SURVEY 8(f)).

For each HBM budget the module scheduler (Sec. 4.5, hg_schedule) makes the highest-gain weights
GPU-resident, the rest of the OPT-30B stack is split by alpha between the host link and the CPU
lane, and bench.py's timed protocol runs.  One process: the 59 GB of pinned weights are built
once.  Prints one JSON line per budget (bench.py's fields) and a summary table.

  python tools/budget_sweep.py [--budgets 0,15,30,45,60] [bench.py options]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budgets", default="0,15,30,45,60")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--model", default="opt-30b", choices=sorted(bench.MODELS))
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--chunk-mb", type=int, default=32)
    ap.add_argument("--ring-mb", type=int, default=4096)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--no-breakdown", dest="breakdown", action="store_false")
    ap.add_argument("--no-abench", dest="abench", action="store_false")
    ap.add_argument("--abench-gamma", type=float, default=0.06)
    ap.add_argument("--out", default=None)
    ap.add_argument("--pageable", action="store_true")
    args = ap.parse_args()
    bench.set_model(args.model)
    if args.layers is None:
        args.layers = bench.LAYERS
    args.warmup = max(args.warmup, 3)
    st = bench.prepare(args)
    rows = []
    for b in [float(v) for v in args.budgets.split(",")]:
        line = bench.run_point(st, args, b)
        rows.append(line)
        print(json.dumps(line), flush=True)
    print("| HBM budget GB | resident GB | alpha | ms/token | e2e ms/token | path roofline ms | frac |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        pr = r["path_roofline"]
        res_gb = r["scheduler"]["placed_GB"] if r["scheduler"] else 0.0
        print(f"| {r['config']['hbm_budget_GB']:g} | {res_gb:.1f} | {r['config']['alpha']:.3f} | {r['value']:.2f} | "
              f"{r['e2e']['value']:.2f} | {pr['t_roof_ms_at_plan_alpha']:.2f} | {pr['frac_of_roof_at_plan']:.3f} |")
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)
    st["ctx"].close()


if __name__ == "__main__":
    main()
