# round-2 run p: the full GPU suite and smoke() on the final HEAD (137 tests incl. the stage-geometry test)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r02p_pytest_gpu.txt 2>&1; echo "pytest rc $?"
python __graft_entry__.py smoke > gpurun_out/r02p_smoke.txt 2>&1; echo "smoke rc $?"
python bench.py --config 2d_medium --no-cpu-baseline > gpurun_out/r02p_bench_2d_medium.txt 2>&1; echo "bench2d rc $?"
