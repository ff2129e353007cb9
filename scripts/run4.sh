timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_gpu.log
python scripts/profile_matvec.py 3d_laplace 1 3 > gpurun_out/plain_3dlap.log 2>&1; echo rc $?
python scripts/profile_matvec.py 3d_laplace 4 3 >> gpurun_out/plain_3dlap.log 2>&1; echo rc $?
python scripts/profile_matvec.py 2d_medium 1 3 >> gpurun_out/plain_3dlap.log 2>&1; echo rc $?
cat gpurun_out/plain_3dlap.log
