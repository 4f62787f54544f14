#!/bin/bash
# One GPU call: parity tests, the bench line, the ncu launch list of the bench
# command and one `--set full` capture of the top kernel.  Outputs in gpurun_out/<tag>/.
#   bash tools/gpu_round.sh <tag> [what...]    what: tests bench launches full micro (default: all)
tag=${1:-run}; shift
what=${*:-tests bench launches full}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv > $out/smi.txt 2>&1
has() { [[ " $what " == *" $1 "* ]]; }
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
  tail -3 $out/pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "smoke rc=$?" >> $out/smoke.txt
fi
if has bench; then
  timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
  tail -c 3000 $out/bench.json
fi
if has micro; then
  timeout 600 python tools/microbench.py > $out/micro.txt 2>&1; tail -30 $out/micro.txt
fi
if has launches; then
  # launch list of the bench command's timed step (NVTX range hg_timed; serialised, cold-cache:
  # compare shares, not absolutes)
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "hg_timed/" \
    --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-breakdown --no-cpu-baseline > $out/launches_bench.json 2>&1
  echo "launches rc=$?"
  python tools/ncu_summary.py launches $out/launches.csv > $out/launches_summary.md 2>&1; head -20 $out/launches_summary.md
fi
if has full; then
  # the top kernel: the persistent GEMV inside the timed step (4 launches), and its replay
  timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hg_timed/" \
    -k "regex:gemv_(row|stream|tc_stream)" -c 4 -o $out/prof_gemv_step \
    python bench.py --layers 4 --steps 1 --warmup 3 --no-breakdown --no-cpu-baseline --no-abench \
    > $out/full_bench.log 2>&1
  echo "full rc=$?"
  python tools/ncu_summary.py full $out/prof_gemv_step.ncu-rep > $out/full_summary_step.md 2>&1
  ALPHA=0.24 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:gemv_(row|stream|tc_stream)" \
    -o $out/prof_gemv_replay python tools/prof_replay.py > $out/full_replay.log 2>&1
  python tools/ncu_summary.py full $out/prof_gemv_replay.ncu-rep > $out/full_summary_replay.md 2>&1
  python tools/ncu_summary.py traffic $out/prof_gemv_replay.ncu-rep 0.24 > $out/ncu_gemv_replay_traffic.json 2>&1
  head -40 $out/full_summary_replay.md
fi
if has batches; then
  for b in 1 2 4 8; do B=$b timeout 120 python tools/replay_roofline.py >> $out/replay.jsonl 2>&1; done; cat $out/replay.jsonl
  for b in 8; do timeout 900 python bench.py --batch $b --no-cpu-baseline > $out/bench_b$b.json 2> $out/bench_b$b.err; echo "b$b rc=$?"; done
fi
