#!/bin/bash
# A/B experiments on one box (development).  AB_CFGS: one config per line, "ENV=V ... | bench args".
out=gpurun_out/${AB_TAG:-ab}; mkdir -p $out
LAYERS=${AB_LAYERS:-12}
for rep in 1 2; do
  while IFS= read -r cfg; do
    [ -z "$cfg" ] && continue
    envs="${cfg%%|*}"; args=""; [[ "$cfg" == *"|"* ]] && args="${cfg#*|}"
    tag=$(echo "$cfg" | tr ' =|-' '____')
    env $envs timeout 600 python bench.py --layers $LAYERS --steps 4 --no-cpu-baseline $args > $out/$tag.r$rep.json 2>&1
    python -c "import json,sys; d=json.loads(open('$out/$tag.r$rep.json').read().strip().splitlines()[-1]); print('$cfg rep=$rep', d['value'], 'alpha', round(d['config']['alpha'],4), 'rates', d['rates_GBps']['v_cpu'], d['rates_GBps']['v_link'], 'lanes', d['lanes'])" || tail -3 $out/$tag.r$rep.json
  done <<< "$AB_CFGS"
done
