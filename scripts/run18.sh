timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity rc $?
tail -3 gpurun_out/pytest_parity.log
for c in 3d_exp_proxy 3d_laplace; do for r in 1 16; do echo "$(timeout 300 python scripts/profile_matvec.py $c $r 3 2>&1 | tail -1)"; done; done
bash scripts/sanitize.sh memcheck
