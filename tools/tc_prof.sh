#!/bin/bash
# tcgen05 GEMV diagnosis: per-CTA stamps and ncu --set full of the replayed launches at B=2 and B=8.
out=gpurun_out/${1:-r02_tc2}; mkdir -p $out
for b in 2 8; do B=$b timeout 120 python tools/tc_stamps.py >> $out/stamps.txt 2>&1; done
cat $out/stamps.txt
for b in 2 8; do
  B=$b ALPHA=0.24 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:gemv_tc_stream" \
    -o $out/prof_b$b python tools/prof_replay.py > $out/prof_b$b.log 2>&1
  python tools/ncu_summary.py full $out/prof_b$b.ncu-rep > $out/full_b$b.md 2>&1
done
head -60 $out/full_b2.md; head -60 $out/full_b8.md
