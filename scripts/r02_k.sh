# round-2 run k: precomputed stage plan for the single-RHS product (planned producer) —
# parity, A/B against the on-the-fly producer (libhh_desc0), stage geometry A/B, cycle probes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf -x --durations=3 > gpurun_out/r02k_pytest.txt 2>&1; echo "pytest rc $?"
for c in 2d_medium 2d_tiny 3d_sphere 3d_exp_proxy; do
  HH_LIB=$PWD/paper_2604_09147_b200/libhh_probe0.so timeout 300 python scripts/probe_matvec.py $c 2>&1 | grep phase | sed "s/^/[on-the-fly] /"
  HH_LIB=$PWD/paper_2604_09147_b200/libhh_probe.so timeout 300 python scripts/probe_matvec.py $c 2>&1 | grep phase | sed "s/^/[planned auto] /"
  HH_MV_GEOM1=0 HH_MV_GEOM2=0 HH_LIB=$PWD/paper_2604_09147_b200/libhh_probe.so timeout 300 python scripts/probe_matvec.py $c 2>&1 | grep phase | sed "s/^/[planned 00] /"
  HH_MV_GEOM1=1 HH_MV_GEOM2=1 HH_LIB=$PWD/paper_2604_09147_b200/libhh_probe.so timeout 300 python scripts/probe_matvec.py $c 2>&1 | grep phase | sed "s/^/[planned 11] /"
done > gpurun_out/r02k_probe.txt 2>&1
for r in 1 2; do
  for c in "2d_medium 1" "2d_tiny 1" "3d_sphere 1" "3d_exp_proxy 1" "3d_laplace 1"; do
    HH_LIB=$PWD/paper_2604_09147_b200/libhh_desc0.so timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs= | sed "s/^/[on-the-fly] /"
    timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs= | sed "s/^/[planned auto] /"
    HH_MV_GEOM1=0 HH_MV_GEOM2=0 timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs= | sed "s/^/[planned 00] /"
    HH_MV_GEOM1=1 HH_MV_GEOM2=1 timeout 300 python scripts/profile_matvec.py $c 5 2>&1 | grep nrhs= | sed "s/^/[planned 11] /"
  done
done > gpurun_out/r02k_ab.txt 2>&1
