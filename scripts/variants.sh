# Build matvec variants side by side (CPU, nvcc cross-compile) for one GPU timing call.
set -e
python -m paper_2604_09147_b200.build
build() { python -m paper_2604_09147_b200.build --variant "$@" > /dev/null; }
build s2_wd48_x6 -DHH_MV_WDATA=49152 -DHH_MV_XDATA=6144
build s3_wd32 -DHH_MV_STAGES=3
build s2_wd40_x5 -DHH_MV_WDATA=40960 -DHH_MV_XDATA=5120
build s2_wd28 -DHH_MV_WDATA=28672
build s2_wd64_x8 -DHH_MV_WDATA=65536 -DHH_MV_XDATA=8192
ls paper_2604_09147_b200/*.so
