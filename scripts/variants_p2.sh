# Phase-2 multi-RHS (NR = 16) ring variants, built side by side for one GPU timing call.
set -e
python -m paper_2604_09147_b200.build
build() { python -m paper_2604_09147_b200.build --variant "$@" > /dev/null; }
build alias_s2_w24 -DHH_MV_P2ALIAS=1 -DHH_MV_P2HI=24576 -DHH_MV_P2X=24576
build alias_s2_w28_x24 -DHH_MV_P2ALIAS=1 -DHH_MV_P2HI=28672 -DHH_MV_P2X=24576
build alias_s2_w32_x20 -DHH_MV_P2ALIAS=1 -DHH_MV_P2HI=32768 -DHH_MV_P2X=20480
build alias_s2_w24_x32 -DHH_MV_P2ALIAS=1 -DHH_MV_P2HI=24576 -DHH_MV_P2X=32768
build alias_s2_w28_x28 -DHH_MV_P2ALIAS=1 -DHH_MV_P2HI=28672 -DHH_MV_P2X=28672
ls paper_2604_09147_b200/*.so
