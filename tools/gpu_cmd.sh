out=gpurun_out/r02c; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; tail -1 $out/smoke.txt
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]); print('default', d['value'], d['e2e']['value'], d['config']['alpha'], d['path_roofline']['frac_of_roof_at_plan'], d['roofline']['frac'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --pageable --no-cpu-baseline > $out/bench_pageable.json 2> $out/bench_pageable.err; echo "pageable rc=$?"
python -c "import json; d=json.loads(open('$out/bench_pageable.json').read().strip().splitlines()[-1]); print('pageable', d['value'], d['config']['alpha'], d['lanes'], d['alpha_bench'])"
for b in 4 8; do timeout 900 python bench.py --batch $b --no-cpu-baseline > $out/bench_b$b.json 2> $out/bench_b$b.err; echo "b$b rc=$?"
python -c "import json; d=json.loads(open('$out/bench_b$b.json').read().strip().splitlines()[-1]); print('B=$b', d['value'], d['e2e']['value'], d['config']['alpha'], d['path_roofline']['frac_of_roof_at_plan'], d['lanes']['busy_frac'], d['roofline'].get('frac'))"; done
timeout 2400 python tools/ablation.py --out $out/ablation.json > $out/ablation.txt 2>&1; echo "ablation rc=$?"; tail -12 $out/ablation.txt
