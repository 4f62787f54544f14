out=gpurun_out/r01g; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -5 $out/pytest_gpu.txt
timeout 300 python tools/microbench.py > $out/micro.txt 2>&1; echo "micro rc=$?"; head -13 $out/micro.txt
export BATCHES=1
N=7168 K=28672 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_stream -c 1 -o $out/prof_k28672 python tools/prof_gemv.py > $out/ncu1.log 2>&1
