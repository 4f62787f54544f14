#!/bin/bash
# GPU tests + smoke + bench lines at batch 1, 2, 4, 8 (+ replay rooflines per batch).
out=gpurun_out/${1:-batches}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -2 $out/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; tail -1 $out/smoke.txt
for b in 1 2 3 4 5 8; do B=$b timeout 120 python tools/replay_roofline.py >> $out/replay.jsonl 2>&1; done; cat $out/replay.jsonl
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]); print('B=1', d['value'], d['e2e']['value'], d['config']['alpha'], d['path_roofline']['frac_of_roof_at_plan'], d['roofline']['frac'], d['cpu_baseline']['value'])"
for b in 2 4 8; do timeout 900 python bench.py --batch $b --no-cpu-baseline > $out/bench_b$b.json 2> $out/bench_b$b.err; echo "b$b rc=$?"
python -c "import json; d=json.loads(open('$out/bench_b$b.json').read().strip().splitlines()[-1]); print('B=$b', d['value'], d['e2e']['value'], d['config']['alpha'], d['path_roofline']['frac_of_roof_at_plan'], d['lanes']['busy_frac'], d['roofline'].get('frac'), d['roofline'].get('kernel'))"; done
