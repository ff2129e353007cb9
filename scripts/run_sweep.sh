rm -f profiles/r01_sweep.jsonl
timeout 2400 python scripts/sweep.py > gpurun_out/sweep.log 2>&1; echo sweep rc $?
timeout 1800 python scripts/sweep.py --ledger-3d-large >> gpurun_out/sweep.log 2>&1; echo ledger rc $?
cp profiles/r01_sweep.jsonl gpurun_out/r01_sweep.jsonl
