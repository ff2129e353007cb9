# round-2 run e: phase-2 leaf order at 16 RHS (Morton vs LPT) A/B, bench
mkdir -p gpurun_out
for r in 1 2; do
  for v in default lpt16; do
    if [ "$v" = default ]; then lib=paper_2604_09147_b200/libhh.so; else lib=paper_2604_09147_b200/libhh_$v.so; fi
    for c in "3d_exp_proxy 16" "3d_laplace 16" "3d_sphere 16" "3d_exp_proxy 8"; do
      HH_LIB=$PWD/$lib timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs= | sed "s/^/[$v] /"
    done
  done
done > gpurun_out/r02e_ab.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02e_bench.txt 2>&1; echo "bench rc $?"
