out=gpurun_out/r02_tc7; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; echo "pytest rc=$?" >> $out/pytest.txt; tail -3 $out/pytest.txt
for cfg in "256 16" "512 8" "1024 16" "256 32" "512 32"; do
  set -- $cfg
  for b in 8 2; do
    HG_TC_SLICE_MIN=$1 HG_TC_SLICE_COUNT=$2 B=$b timeout 120 python tools/replay_roofline.py >> $out/replay.jsonl 2>> $out/replay.err
  done
  HG_TC_SLICE_MIN=$1 HG_TC_SLICE_COUNT=$2 B=1 TCMIN=1 timeout 120 python tools/replay_roofline.py >> $out/replay.jsonl 2>> $out/replay.err
done
python -c "
import json
for l in open('$out/replay.jsonl'):
    d=json.loads(l); e=d['env']; print(d['B'], e.get('HG_TC_SLICE_MIN'), e.get('HG_TC_SLICE_COUNT'), e.get('TCMIN','-'), d['frac'], d['per_linear'])
"
