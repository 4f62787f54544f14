out=gpurun_out/r01k; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -3 $out/pytest.txt
export AB_TAG=ab_mirror AB_LAYERS=48 AB_CFGS='HG_MIRROR_GLUE=1 | --no-abench --alpha 0.23
HG_MIRROR_GLUE=0 | --no-abench --alpha 0.23
HG_MIRROR_GLUE=1 |'
bash tools/ab.sh
