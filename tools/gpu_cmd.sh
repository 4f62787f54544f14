out=gpurun_out/r01e; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -5 $out/pytest_gpu.txt
timeout 300 python tools/microbench.py > $out/micro.txt 2>&1; echo "micro rc=$?"; head -30 $out/micro.txt
