out=gpurun_out/r01j; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_layer.py -x -q > $out/pytest.txt 2>&1; tail -2 $out/pytest.txt
export AB_TAG=ab_join AB_LAYERS=48 AB_CFGS='HG_JOIN_MEMCPY=0 | --no-abench --alpha 0.23
HG_JOIN_MEMCPY=1 | --no-abench --alpha 0.23
HG_JOIN_MEMCPY=0 |'
bash tools/ab.sh
