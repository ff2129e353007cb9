# round-2 run b: parity + working precision + q43 on the GPU, A/B of the NR=1 vector consumers,
# bench, Fig. 9 backward-error experiment
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wp.py -q -rA --durations=10 > gpurun_out/r02b_pytest.txt 2>&1; echo "pytest rc $?"
for r in 1 2; do
  for v in default vec0; do
    if [ "$v" = default ]; then lib=paper_2604_09147_b200/libhh.so; else lib=paper_2604_09147_b200/libhh_$v.so; fi
    for c in "3d_laplace 1" "3d_exp_proxy 1" "2d_medium 1" "3d_sphere 1"; do
      HH_LIB=$PWD/$lib timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs= | sed "s/^/[$v] /"
    done
  done
done > gpurun_out/r02b_ab_vec1.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench.txt 2>&1; echo "bench rc $?"
timeout 1200 python scripts/backward_error.py --out gpurun_out/r02b_backward_error.json > gpurun_out/r02b_backward_error.log 2>&1; echo "bwd rc $?"
