#!/bin/bash
# Generic GPU call: run the given pytest selection and optional bench args; outputs in gpurun_out/<tag>/.
#   bash tools/gpu_cmd.sh <tag> "<pytest args or ->" "<bench args or ->"
tag=${1:-cmd}; out=gpurun_out/$tag; mkdir -p $out
if [ "${2:--}" != "-" ]; then
  timeout 1500 python -m pytest $2 -x -q > $out/pytest.txt 2>&1; echo "pytest rc=$?" >> $out/pytest.txt; tail -5 $out/pytest.txt
fi
if [ "${3:--}" != "-" ]; then
  timeout 900 python bench.py $3 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; tail -c 2500 $out/bench.json; tail -5 $out/bench.err
fi
