out=gpurun_out/r01r; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -3 $out/pytest.txt
timeout 1800 python tools/budget_sweep.py --budgets 0,10,20,30,40,50,60 --out $out/sweep.json > $out/sweep.txt 2>&1; echo "sweep rc=$?"; tail -9 $out/sweep.txt
