#!/bin/bash
# GPU parity tests + smoke + the default bench line (+ optional extra command).
out=gpurun_out/${1:-quick}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -2 $out/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; tail -1 $out/smoke.txt
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]); print('default', d['value'], d['e2e']['value'], d['config']['alpha'], d['path_roofline']['frac_of_roof_at_plan'], d['roofline']['frac'], d['roofline'].get('single_launch'), d['roofline']['per_linear'], d['cpu_baseline']['value'])"
