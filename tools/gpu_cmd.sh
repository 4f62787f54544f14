out=gpurun_out/r01t; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_linear.py -q -k "stats or tags" > $out/pytest.txt 2>&1; tail -2 $out/pytest.txt
for m in opt-6.7b opt-13b opt-30b; do
  timeout 900 python bench.py --model $m --no-cpu-baseline > $out/bench_$m.json 2> $out/bench_$m.err; echo "$m rc=$?"
  python -c "import json; d=json.loads(open('$out/bench_$m.json').read().strip().splitlines()[-1]); print('$m', d['value'], d['e2e']['value'], d['config']['alpha'], d['path_roofline']['frac_of_roof_at_plan'], d['rates_GBps'], d['lanes']['busy_frac'], d['alpha_bench']['alpha_bar'], d['alpha_bench']['clamped'])"
done
