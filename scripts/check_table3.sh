timeout 1200 python -m pytest tests/test_gpu_table3.py -x -q -s 2>&1 | tail -5
python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/plain_nr16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase2 -s 1 -c 1 -o gpurun_out/prof_nr16b python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/ncu_nr16b.log 2>&1; echo ncu rc $?
