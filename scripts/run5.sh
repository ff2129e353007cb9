timeout 1200 python bench.py > gpurun_out/bench_3dlarge.log 2>&1; echo bench rc $?
tail -1 gpurun_out/bench_3dlarge.log
python scripts/profile_matvec.py 3d_laplace 1 3 > gpurun_out/plain_3dlap.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/prof_v1_3dlap python scripts/profile_matvec.py 3d_laplace 1 3 > gpurun_out/ncu_v1.log 2>&1
echo ncu rc $?
