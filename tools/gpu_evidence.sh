out=gpurun_out/r02_evid; mkdir -p $out
for b in 2 4 8; do timeout 900 python bench.py --batch $b --no-cpu-baseline > $out/bench_b$b.json 2> $out/bench_b$b.err; echo "b$b rc=$?"
python -c "import json; d=json.loads(open('$out/bench_b$b.json').read().strip().splitlines()[-1]); print('B=$b', d['value'], d['e2e']['value'], round(d['config']['alpha'],4), d['path_roofline']['frac_of_roof_at_plan'], d['lanes']['busy_frac'], d['roofline'].get('frac'), d['step_ms']['p10'], d['step_ms']['p90'])"; done
bash tools/gpu_models.sh r02_models
timeout 900 python bench.py --no-cpu-baseline --hbm-budget-gb 20 --scheduler rows > $out/sched_rows20.json 2> $out/sched_rows20.err; echo rows20 rc=$?
timeout 900 python bench.py --no-cpu-baseline --hbm-budget-gb 20 --scheduler module > $out/sched_mod20.json 2> $out/sched_mod20.err; echo mod20 rc=$?
for f in sched_rows20 sched_mod20; do python -c "import json; d=json.loads(open('$out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['path_roofline']['frac_of_roof_at_plan'], d['scheduler'])"; done
