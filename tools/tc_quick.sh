#!/bin/bash
# tcgen05 GEMV quick check: replay roofline at B = 1, 2, 4, 8 (+ B=1 forced tcgen05) and B=8 stamps.
out=gpurun_out/${1:-tcq}; mkdir -p $out
shift
for b in 8 4 2 1; do B=$b timeout 120 python tools/replay_roofline.py >> $out/replay.jsonl 2>> $out/replay.err; done
B=1 TCMIN=1 timeout 120 python tools/replay_roofline.py >> $out/replay.jsonl 2>> $out/replay.err
python -c "
import sys, json
for l in open('$out/replay.jsonl'):
    d=json.loads(l); e=d['env']; print(d['B'], e.get('TCMIN','-'), {k:v for k,v in e.items() if k.startswith('HG_')}, d['frac'], d['per_linear'])
"
for b in ${STAMPS_B:-8}; do B=$b timeout 120 python tools/tc_stamps.py 2>&1 | grep warm | cut -c1-330; done
