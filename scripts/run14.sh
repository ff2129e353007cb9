timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity rc $?
tail -3 gpurun_out/pytest_parity.log
for r in 1 16; do echo "$(timeout 300 python scripts/profile_matvec.py 3d_exp_proxy $r 3 2>&1 | tail -1)"; done
HH_PROFILE_BUILD=1 timeout 300 python scripts/profile_matvec.py 3d_laplace 1 3 2>&1 | tail -4
timeout 1500 python -m pytest tests/test_gpu_sweep.py -x -q -k "s0" --durations=5 > gpurun_out/pytest_sweep_s0.log 2>&1; echo sweep-s0 rc $?
tail -8 gpurun_out/pytest_sweep_s0.log
