export AB_TAG=ab_zc2 AB_LAYERS=48 AB_CFGS='HG_STREAM_MODE=0 | --alpha 0.24
HG_STREAM_MODE=1 | --alpha 0.24
HG_STREAM_MODE=1 |'
bash tools/ab.sh
