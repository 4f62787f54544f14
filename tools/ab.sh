#!/bin/bash
# A/B experiments on one box (development): runtime switches via env.
out=gpurun_out/ab; mkdir -p $out
for rep in 1 2; do
  for cfg in "HG_HOST_ROWS=8 HG_ASYNC_POST=1" "HG_HOST_ROWS=4 HG_ASYNC_POST=1" "HG_HOST_ROWS=8 HG_ASYNC_POST=0"; do
    tag=$(echo $cfg | tr ' =' '__')
    env $cfg timeout 600 python bench.py --layers 12 --steps 4 --no-cpu-baseline > $out/$tag.r$rep.json 2>&1
    python -c "import json,sys; d=json.loads(open('$out/$tag.r$rep.json').read().strip().splitlines()[-1]); print('$cfg rep=$rep', d['value'], 'v_cpu', d['rates_GBps']['v_cpu'], 'lanes', d['lanes'], 'roof', (d['roofline'] or {}).get('achieved'))"
  done
done
