out=gpurun_out/r01m; mkdir -p $out
python tools/prof_replay.py | tee $out/replay.txt
timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_layer.py -x -q 2>&1 | tail -2
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]); print(json.dumps({k:d.get(k) for k in ['value','e2e','path_roofline','rates_GBps','lanes','alpha_bench','cpu_baseline']})); print(d['roofline'])"
