# round-2 run d: parity (accessor formats) + wp, A/B of the NR=1 phase-2 reduction / PDL / vec1, ncu NR=1 proxy
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wp.py -q -rf --durations=5 > gpurun_out/r02d_pytest.txt 2>&1; echo "pytest rc $?"
for r in 1 2; do
  for v in default red1 pdl0 vec0; do
    if [ "$v" = default ]; then lib=paper_2604_09147_b200/libhh.so; else lib=paper_2604_09147_b200/libhh_$v.so; fi
    for c in "2d_tiny 1" "2d_medium 1" "3d_laplace 1" "3d_exp_proxy 1" "3d_sphere 1"; do
      HH_LIB=$PWD/$lib timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs= | sed "s/^/[$v] /"
    done
  done
done > gpurun_out/r02d_ab.txt 2>&1
python scripts/profile_matvec.py 3d_exp_proxy 1 3 > gpurun_out/r02d_plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/r02d_prof1 \
    python scripts/profile_matvec.py 3d_exp_proxy 1 3 > gpurun_out/r02d_ncu1.log 2>&1; echo "ncu rc $?"
