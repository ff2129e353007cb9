# round-2 validation run: host facts, GPU parity suite, default bench (nrhs=1 + 16-RHS record)
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv) > gpurun_out/r02a_host.txt 2>&1
timeout 3300 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/r02a_pytest_gpu.txt 2>&1; echo "pytest rc $?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.txt 2>&1; echo "bench rc $?"
