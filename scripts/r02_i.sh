# round-2 run i: build profile of 3D N=2^20 (HH_PROFILE_BUILD), phase-2 producer prefetch on the
# small-leaf configs, parity of the changed producer
mkdir -p gpurun_out
for r in 1 2; do
  for c in "2d_medium 1" "2d_tiny 1" "3d_sphere 1" "3d_exp_proxy 1" "3d_laplace 1" "3d_exp_proxy 16"; do
    timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs=
  done
done > gpurun_out/r02i_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "check2 or determin or row_split or nrhs" > gpurun_out/r02i_pytest.txt 2>&1; echo "pytest rc $?"
HH_PROFILE_BUILD=1 timeout 900 python scripts/profile_matvec.py 3d_large 1 2 > gpurun_out/r02i_buildprof.txt 2>&1; echo "buildprof rc $?"
