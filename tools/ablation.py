"""Ablation of the B200 pipeline (Table 3 analogue; NEXT(4) of SURVEY 8(f)).

One process (weights built once).  Each variant gets a fresh context with its switches and runs
bench.py's timed protocol on the OPT-30B stack, batch 1, r = 0 unless stated:

  all                   Eq. (5) alpha refined by the alpha benchmark, device-tag chunk pipeline,
                        zero-copy join, mirrored glue                              (the bench default)
  no alpha benchmark    Eq. (5) alpha from the measured rates only                 (P:365 row)
  no hybrid: GPU only   alpha = 1: every host row streamed (the naive strategy, Fig. 5a)
  no hybrid: CPU only   alpha = 0: every host row on the CPU lane
  no mirrored glue      GPU-only glue: the CPU lane waits for x to cross the link (reading R24 off)
  host events           handshake = 0: one GEMV launch per chunk, host events (pre-tag pipeline)
  zero-copy streaming   stream_mode = 1: the GEMV's TMA bulk copies read the pinned host rows over
                        PCIe themselves (no copy engine, no ring, no tags, no cross-linear prefetch)
  one chunk per linear  1 GiB chunks: the GEMV of a linear starts after its whole slice arrived
                        (the pinned-but-blocking strategy of Fig. 5b, with pre-pinned weights)
  + module scheduler    HBM budget 10 GB placed by hg_schedule (Sec. 4.5)          (P:366 row)

  python tools/ablation.py [--out file.json]
"""
import argparse
import copy
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

VARIANTS = [
    ("all", {}, {}),
    ("no alpha benchmark", {"abench": False}, {}),
    ("no hybrid: GPU only (alpha=1)", {"alpha": 1.0}, {}),
    ("no hybrid: CPU only (alpha=0)", {"alpha": 0.0}, {}),
    ("no mirrored glue", {}, {"mirror_glue": 0}),
    ("host events, GEMV per chunk", {}, {"handshake": 0}),
    ("zero-copy streaming (SM TMA reads over PCIe)", {}, {"stream_mode": 1}),
    ("one chunk per linear (no chunk pipelining)", {"chunk_mb": 1024}, {}),
    ("+ module scheduler, 10 GB HBM", {"budget": 10.0}, {}),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--model", default="opt-30b", choices=sorted(bench.MODELS))
    ap.add_argument("--only", default=None, help="comma-separated variant indices")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    bench.set_model(a.model)
    args = argparse.Namespace(steps=a.steps, warmup=max(3, a.warmup), batch=1, layers=bench.LAYERS, alpha=None,
                              chunk_mb=32, ring_mb=4096, threads=0, breakdown=True, abench=True,
                              abench_gamma=0.06, hbm_budget_gb=0.0, pageable=False, resident=0.0)
    st = bench.prepare(args)
    hg = st["hg"]
    base_ctx = st["ctx"]
    rows = []
    sel = [int(i) for i in a.only.split(",")] if a.only else range(len(VARIANTS))
    for idx in sel:
        name, over, cfg = VARIANTS[idx]
        va = copy.copy(args)
        budget = over.get("budget", 0.0)
        for k, v in over.items():
            if k != "budget":
                setattr(va, k, v)
        ctx = hg.Context(st["local"], cpu_threads=st["threads"], cpu_first=-1, chunk_bytes=va.chunk_mb << 20,
                         ring_bytes=args.ring_mb << 20, max_k=bench.F, max_n=bench.F, wrap_prefetch=1,
                         collect_stats=0, **cfg)
        st["ctx"] = ctx
        line = bench.run_point(st, va, budget)
        ctx.close()
        rows.append({"variant": name, "line": line})
        print(json.dumps({"variant": name, "value": line["value"], "e2e": line["e2e"]["value"],
                          "alpha": line["config"]["alpha"], "lanes": line["lanes"]}), flush=True)
    st["ctx"] = base_ctx
    ref = rows[0]["line"]["value"] if rows and rows[0]["variant"] == "all" else None
    print("| variant | ms/token | relative throughput | alpha | CPU busy | link busy |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        L = r["line"]
        lanes = L["lanes"] or {}
        bf = lanes.get("busy_frac", {})
        rel = f"{100 * ref / L['value']:.1f}%" if ref else "-"
        print(f"| {r['variant']} | {L['value']:.2f} | {rel} | {L['config']['alpha']:.3f} | {bf.get('cpu', '-')} | "
              f"{bf.get('link', '-')} |")
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)
    base_ctx.close()


if __name__ == "__main__":
    main()
