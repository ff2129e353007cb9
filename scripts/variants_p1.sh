# Phase-1 multi-RHS (NR >= 8) stage-geometry variants, built side by side for one GPU timing call.
set -e
python -m paper_2604_09147_b200.build
build() { python -m paper_2604_09147_b200.build --variant "$@" > /dev/null; }
build p1_w40_x12 -DHH_MV_P1HI=40960 -DHH_MV_P1X=12288
build p1_w48_x8 -DHH_MV_P1HI=49152 -DHH_MV_P1X=8192
build p1_w36_x16 -DHH_MV_P1HI=36864 -DHH_MV_P1X=16384
build p1_w44_x10 -DHH_MV_P1HI=45056 -DHH_MV_P1X=10240
ls paper_2604_09147_b200/*.so
