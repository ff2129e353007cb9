timeout 2400 python -m pytest tests/test_gpu_sweep.py -x -q -s > gpurun_out/pytest_sweep.log 2>&1; echo sweep rc $?
tail -3 gpurun_out/pytest_sweep.log
python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/plain_nr16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/prof_nr16 python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/ncu_nr16.log 2>&1; echo ncu rc $?
python scripts/profile_matvec.py 3d_laplace 1 1 > gpurun_out/plain_build.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(gemm_gen|qr|jacobi|resid|factors)" -s 40 -c 6 -o gpurun_out/prof_build python scripts/profile_matvec.py 3d_laplace 1 1 > gpurun_out/ncu_build.log 2>&1; echo ncu rc $?
