# round-2 run l: planned producer + division-free consumer trip counts — parity and timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf -x --durations=3 > gpurun_out/r02l_pytest.txt 2>&1; echo "pytest rc $?"
for r in 1 2; do
  for c in "2d_medium 1" "2d_tiny 1" "3d_sphere 1" "3d_exp_proxy 1" "3d_laplace 1" "3d_exp_proxy 16" "2d_medium 16"; do
    timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs=
  done
done > gpurun_out/r02l_ab.txt 2>&1
