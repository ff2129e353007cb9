# Build matvec variants side by side (CPU, nvcc cross-compile) for one GPU timing call.
set -e
python -m paper_2604_09147_b200.build
python -m paper_2604_09147_b200.build --variant c2 -DHH_MV_CHAINS=2 > /dev/null &
python -m paper_2604_09147_b200.build --variant cvt -DHH_MV_CVT=1 > /dev/null &
python -m paper_2604_09147_b200.build --variant s4 -DHH_MV_STAGES=4 > /dev/null &
python -m paper_2604_09147_b200.build --variant cvt_s4 -DHH_MV_CVT=1 -DHH_MV_STAGES=4 > /dev/null &
wait
ls -la paper_2604_09147_b200/*.so
