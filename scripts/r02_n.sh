# round-2 run n: BASELINE config 4 admissibility sweep re-measured with the final kernels
mkdir -p gpurun_out
rm -f gpurun_out/r02_sweep.jsonl
timeout 2400 python scripts/sweep.py --out gpurun_out/r02_sweep.jsonl > gpurun_out/r02n_sweep.log 2>&1; echo sweep rc $?
