# Phase-2 multi-RHS (NR = 16) ring / peel variants, built side by side for one GPU timing call.
set -e
python -m paper_2604_09147_b200.build
build() { python -m paper_2604_09147_b200.build --variant "$@" > /dev/null; }
build peel -DHH_MV_PEEL=1
build p2s3_x8 -DHH_MV_P2STAGES=3 -DHH_MV_P2X=8192
build p2s3_x8_peel -DHH_MV_P2STAGES=3 -DHH_MV_P2X=8192 -DHH_MV_PEEL=1
build p2s2_w24_x8 -DHH_MV_P2HI=24576 -DHH_MV_P2X=8192
build p2s3_x6 -DHH_MV_P2STAGES=3 -DHH_MV_P2X=6144
ls paper_2604_09147_b200/*.so
