# round-2 run f (diagnostics): 2D medium phase-1 row-split threshold A/B (HH_P1_ROWS, no rebuild);
# ncu --set full of the 16-RHS phase kernels on the proxy in Morton order and of the NR=1
# kernels on 2D medium
mkdir -p gpurun_out
for r in 1 2; do
  for rows in 4096 2048 1024 512 256; do
    for c in "2d_medium 1" "2d_tiny 1"; do
      HH_P1_ROWS=$rows timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs= | sed "s/^/[rows=$rows] /"
    done
  done
done > gpurun_out/r02f_rows.txt 2>&1
python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/r02f_plain16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/r02f_prof16 \
    python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/r02f_ncu16.log 2>&1; echo "ncu16 rc $?"
python scripts/profile_matvec.py 2d_medium 1 3 > gpurun_out/r02f_plain2d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/r02f_prof2d \
    python scripts/profile_matvec.py 2d_medium 1 3 > gpurun_out/r02f_ncu2d.log 2>&1; echo "ncu2d rc $?"
python scripts/ncu_summary.py gpurun_out/r02f_prof16.ncu-rep > gpurun_out/r02f_proxy_nrhs16_ncu.txt 2>&1
python scripts/ncu_summary.py gpurun_out/r02f_prof2d.ncu-rep > gpurun_out/r02f_2dmedium_ncu.txt 2>&1
