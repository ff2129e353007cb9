# round-2 run g: K-quartered DMMA stages (HH_MV_QUART) — parity, A/B against the linear stages,
# adaptive phase-1 row split on the 2D configs, ncu of the 16-RHS phase kernels on the proxy
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf -x --durations=5 > gpurun_out/r02g_pytest.txt 2>&1; echo "pytest rc $?"
for r in 1 2; do
  for v in default quart0; do
    if [ "$v" = default ]; then lib=paper_2604_09147_b200/libhh.so; else lib=paper_2604_09147_b200/libhh_$v.so; fi
    for c in "3d_exp_proxy 16" "3d_laplace 16" "3d_sphere 16" "3d_exp_proxy 8" "2d_medium 16" "2d_medium 1" "2d_tiny 1"; do
      HH_LIB=$PWD/$lib timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs= | sed "s/^/[$v] /"
    done
  done
done > gpurun_out/r02g_ab.txt 2>&1
python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/r02g_plain16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/r02g_prof16 \
    python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/r02g_ncu16.log 2>&1; echo "ncu16 rc $?"
python scripts/ncu_summary.py gpurun_out/r02g_prof16.ncu-rep > gpurun_out/r02g_proxy_nrhs16_ncu.txt 2>&1
