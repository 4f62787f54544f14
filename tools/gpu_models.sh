#!/bin/bash
# Bench lines for the other BASELINE.json configurations (C2 OPT-6.7B r=0.5 and r=0, C3 OPT-13B B=1,2,4).
out=gpurun_out/${1:-models}; mkdir -p $out
run() { tag=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" > $out/$tag.json 2> $out/$tag.err; echo "$tag rc=$?"
python -c "import json; d=json.loads(open('$out/$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], round(d['config']['alpha'],4), d['config']['r_resident'], d['path_roofline']['t_roof_ms_at_plan_alpha'], d['path_roofline']['frac_of_roof_at_plan'], d['lanes']['busy_frac'], d['roofline'].get('frac'))"; }
run c2_r05 --model opt-6.7b --resident 0.5
run c2_r0 --model opt-6.7b
run c3_b1 --model opt-13b
run c3_b2 --model opt-13b --batch 2
run c3_b4 --model opt-13b --batch 4
