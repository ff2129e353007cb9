# round-2 closing evidence on the final code: full GPU suite, bench (nrhs 1 with multi_rhs
# sub-record; --nrhs 16), ncu launch list + full capture of the bench command, every other
# BASELINE config, NEXT-3 storage table
bash scripts/gpu_round.sh
bash scripts/bench_all.sh
timeout 1200 python scripts/next3_storage.py --out gpurun_out/r02_next3_storage.json > gpurun_out/next3_storage.log 2>&1; echo "next3 rc $?"
python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > gpurun_out/r02j_3dlarge_ncu.txt 2>&1
nvidia-smi --query-gpu=name,clocks.current.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02j_host.txt 2>&1
