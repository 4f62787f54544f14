out=gpurun_out/r02b; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -3 $out/pytest.txt
timeout 900 python bench.py --pageable --no-cpu-baseline > $out/bench_pageable.json 2> $out/bench_pageable.err; echo "pageable rc=$?"
python -c "import json; d=json.loads(open('$out/bench_pageable.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['config']['alpha'], d['config']['alpha_mode'], d['rates_GBps'], d['lanes'], d['path_roofline']['terms_ms'])" || tail -5 $out/bench_pageable.err
