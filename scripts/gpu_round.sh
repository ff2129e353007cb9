# The GPU-side evidence of a round, as run through gpurun (one B200):
#   /usr/local/graft/bin/gpurun --timeout 5400 -- 'bash scripts/gpu_round.sh'
# 1. GPU parity suite (small configs, full BASELINE sizes, admissibility sweep)
# 2. bench.py at the default workload (3D N=2^20, nrhs=1) and nrhs=16
# 3. ncu: launch list of the bench command, then --set full on the two phase kernels
#    (each ncu run only after the same command exited 0 without ncu)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
python bench.py > gpurun_out/bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(gather|phase|p1_combine)" --csv \
    --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 6 -c 2 -o gpurun_out/prof \
    python bench.py > gpurun_out/ncu_full.log 2>&1; echo "bench/ncu rc $?"
python bench.py --nrhs 16 --no-cpu-baseline > gpurun_out/bench_nrhs16.log 2>&1; echo "bench16 rc $?"
# 4. (optional, ~15 min) BASELINE config 4 sweep + ledger-only storage baselines: bash scripts/run_sweep.sh
