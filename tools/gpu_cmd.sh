out=gpurun_out/r01z9; mkdir -p $out
run() { tag=$1; shift; timeout 900 env "$@" > $out/$tag.json 2> $out/$tag.err; rc=$?; echo "$tag rc=$rc $(grep -o 'HgError:.*' $out/$tag.err | head -1 | cut -c1-200) $(grep -o '"value": [0-9.]*' $out/$tag.json | head -1)"; }
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
python tools/microbench.py 2>&1 | head -4
for i in 1 2; do run b3_$i python bench.py --batch 3 --no-cpu-baseline --no-breakdown --steps 2; run b4_$i python bench.py --batch 4 --no-cpu-baseline --no-breakdown --steps 2; run b2_$i python bench.py --batch 2 --no-cpu-baseline --no-breakdown --steps 2; done
