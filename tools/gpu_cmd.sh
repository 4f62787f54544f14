out=gpurun_out/r01s; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -2 $out/pytest.txt
timeout 2400 python tools/ablation.py --out $out/ablation.json > $out/ablation.txt 2>&1; echo "ablation rc=$?"; tail -10 $out/ablation.txt
for m in opt-6.7b opt-13b; do
  timeout 900 python bench.py --model $m --no-cpu-baseline > $out/bench_$m.json 2> $out/bench_$m.err; echo "$m rc=$?"
  python -c "import json; d=json.loads(open('$out/bench_$m.json').read().strip().splitlines()[-1]); print('$m', d['value'], d['e2e']['value'], d['config']['alpha'], d['path_roofline']['frac_of_roof_at_plan'], d['roofline']['frac'])"
done
