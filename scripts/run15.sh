for v in "" p2hi16 p2hi24; do
  if [ -z "$v" ]; then export HH_LIB=""; tag=default; else export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v; fi
  for r in 8 16; do echo "[$tag] $(timeout 300 python scripts/profile_matvec.py 3d_exp_proxy $r 3 2>&1 | tail -1)"; done
  echo "[$tag] $(timeout 300 python scripts/profile_matvec.py 3d_laplace 16 3 2>&1 | tail -1)"
done
unset HH_LIB
rm -f profiles/r01_sweep.jsonl
timeout 2400 python scripts/sweep.py > gpurun_out/sweep.log 2>&1; echo sweep rc $?
timeout 1800 python scripts/sweep.py --ledger-3d-large >> gpurun_out/sweep.log 2>&1; echo ledger rc $?
cp profiles/r01_sweep.jsonl gpurun_out/ 2>/dev/null
tail -14 gpurun_out/sweep.log
