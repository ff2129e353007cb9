# round-2 run h: K-quartered DMMA stages at 2 CTAs/SM (launch bounds), per-handle small-item
# stage geometry at one RHS (auto vs forced off), parity, ncu of the 16-RHS kernels on the proxy
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf -x --durations=5 > gpurun_out/r02h_pytest.txt 2>&1; echo "pytest rc $?"
for r in 1 2; do
  for v in default quart0; do
    if [ "$v" = default ]; then lib=paper_2604_09147_b200/libhh.so; else lib=paper_2604_09147_b200/libhh_$v.so; fi
    for c in "3d_exp_proxy 16" "3d_laplace 16" "3d_sphere 16" "3d_exp_proxy 8" "2d_medium 16"; do
      HH_LIB=$PWD/$lib timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs= | sed "s/^/[$v] /"
    done
  done
  for g in auto 00 10 01 11; do
    for c in "2d_medium 1" "2d_tiny 1" "3d_sphere 1" "3d_exp_proxy 1" "3d_laplace 1"; do
      if [ "$g" = auto ]; then
        timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs= | sed "s/^/[geom=$g] /"
      else
        HH_MV_GEOM1=${g:0:1} HH_MV_GEOM2=${g:1:1} timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs= | sed "s/^/[geom=$g] /"
      fi
    done
  done
done > gpurun_out/r02h_ab.txt 2>&1
python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/r02h_plain16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/r02h_prof16 \
    python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/r02h_ncu16.log 2>&1; echo "ncu16 rc $?"
python scripts/ncu_summary.py gpurun_out/r02h_prof16.ncu-rep > gpurun_out/r02h_proxy_nrhs16_ncu.txt 2>&1
