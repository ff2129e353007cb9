# round-2 run q: whole DMMA K-steps per stage window (multi-RHS producers) — parity of the
# multi-RHS paths, timings, bench lines (default with the multi_rhs sub-record, --nrhs 16)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "check2 or nrhs or determin or row_split or geometry" --durations=3 > gpurun_out/r02q_pytest.txt 2>&1; echo "pytest rc $?"
for r in 1 2; do
  for c in "3d_exp_proxy 16" "3d_laplace 16" "3d_sphere 16" "3d_exp_proxy 8" "2d_medium 16" "3d_exp_proxy 1"; do
    timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs=
  done
done > gpurun_out/r02q_ab.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -k "3d_laplace or 2d_medium" > gpurun_out/r02q_pytest_fullsize.txt 2>&1; echo "fullsize rc $?"
python bench.py > gpurun_out/r02q_bench.txt 2>&1; echo "bench rc $?"
python bench.py --nrhs 16 --no-cpu-baseline > gpurun_out/r02q_bench_nrhs16.txt 2>&1; echo "bench16 rc $?"
