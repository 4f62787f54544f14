"""Ablation of the B200 pipeline (Table 3 analogue; NEXT(4) of SURVEY 8(f)).

One process (weights built once).  Each variant gets a fresh context with its switches and runs
bench.py's timed protocol on the OPT-30B stack, batch 1, r = 0 unless stated.

--pageable: the paper's setting -- host weights are NOT page-locked, every streamed row is pinned on
the way (Sec. 4.2-4.3).  The rows follow Table 3:
  all                              hybrid (Fig. 5c): pin lane ahead across linears || link || CPU lane,
                                   alpha from Eq. (9) refined by the alpha benchmark
  no hybrid: pinned-blocking       Fig. 5b: each linear's rows pinned first on the CPU lane's threads,
                                   blocking the CPU lane and the link, then transferred
  no hybrid: naive                 Fig. 5a: no pin lane; copies straight from un-pinned memory (the
                                   driver stages them) beside the CPU lane
  no async parameter manager       hybrid with a 2-slot staging ring: pinning just in time, no run-ahead
  no alpha benchmark               Eq. (9) alpha from the measured rates only
(default) pinned once at load -- the B200 design (reading R7):
  all                   Eq. (5) alpha refined by the alpha benchmark, device-tag chunk pipeline,
                        zero-copy join, mirrored glue                              (the bench default)
  no alpha benchmark    Eq. (5) alpha from the measured rates only                 (P:365 row)
  GPU only / CPU only   alpha = 1 / alpha = 0 (the split itself, not Table 3's "no hybrid" row)
  no mirrored glue      GPU-only glue: the CPU lane waits for x to cross the link (reading R24 off)
  host events           handshake = 0: one GEMV launch per chunk, host events (pre-tag pipeline)
  zero-copy streaming   stream_mode = 1: the GEMV's TMA bulk copies read the pinned host rows over
                        PCIe themselves (no copy engine, no ring, no tags, no cross-linear prefetch)
  one chunk per linear  1 GiB chunks: the GEMV of a linear starts after its whole slice arrived
  + module scheduler    HBM budget 10 GB placed by hg_schedule (Sec. 4.5)          (P:366 row)

  python tools/ablation.py [--pageable] [--out file.json]
"""
import argparse
import copy
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

VARIANTS_PAGEABLE = [
    ("all (hybrid, Fig. 5c)", {"strategy": "hybrid"}, {}),
    ("no hybrid: pinned-blocking (Fig. 5b)", {"strategy": "blocking"}, {}),
    ("no hybrid: naive (Fig. 5a)", {"strategy": "naive"}, {}),
    # the same strategies at the hybrid's alpha (the per-module ordering of S:399)
    ("pinned-blocking at the hybrid's alpha", {"strategy": "blocking", "alpha": "from_all"}, {}),
    ("naive at the hybrid's alpha", {"strategy": "naive", "alpha": "from_all"}, {}),
    ("no async parameter manager (2-slot staging)", {"strategy": "hybrid", "staging_mb": 64}, {}),
    ("no alpha benchmark", {"strategy": "hybrid", "abench": False}, {}),
    # staging-ring size (P:246 bounds the pinned memory to "one pinned parameter per group")
    ("hybrid, 128 MiB staging", {"strategy": "hybrid", "staging_mb": 128}, {}),
    ("hybrid, 256 MiB staging", {"strategy": "hybrid", "staging_mb": 256}, {}),
    ("hybrid, 2 GiB staging", {"strategy": "hybrid", "staging_mb": 2048}, {}),
]

VARIANTS = [
    ("all", {}, {}),
    ("no alpha benchmark", {"abench": False}, {}),
    ("GPU only (alpha=1)", {"alpha": 1.0}, {}),
    ("CPU only (alpha=0)", {"alpha": 0.0}, {}),
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
    ap.add_argument("--pageable", action="store_true", help="the paper's setting: host weights not page-locked")
    a = ap.parse_args()
    variants = VARIANTS_PAGEABLE if a.pageable else VARIANTS
    bench.set_model(a.model)
    args = bench.parse_args(["--model", a.model, "--steps", str(a.steps), "--warmup", str(a.warmup)] +
                            (["--pageable"] if a.pageable else []))
    st = bench.prepare(args)
    hg = st["hg"]
    base_ctx = st["ctx"]
    rows = []
    sel = [int(i) for i in a.only.split(",")] if a.only else range(len(variants))
    for idx in sel:
        name, over, cfg = variants[idx]
        va = copy.copy(args)
        budget = over.get("budget", 0.0)
        for k, v in over.items():
            if k == "alpha" and v == "from_all":
                v = rows[0]["line"]["config"]["alpha"]
            if k != "budget":
                setattr(va, k, v)
        ctx, _ = bench.make_context(va, 0, 1, st["local"], **cfg)
        st["ctx"] = ctx
        va.parity = False  # the ablation compares timings; parity is the bench's and the tests' job
        line = bench.run_point(st, va, budget)
        line.pop("_trace", None)
        ctx.close()
        rows.append({"variant": name, "line": line})
        print(json.dumps({"variant": name, "value": line["value"], "e2e": line["e2e"]["value"],
                          "alpha": line["config"]["alpha"], "lanes": line["lanes"]}), flush=True)
    st["ctx"] = base_ctx
    ref = rows[0]["line"]["value"] if rows and rows[0]["variant"].startswith("all") else None
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
