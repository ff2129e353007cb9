timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity rc $?
tail -3 gpurun_out/pytest_parity.log
for i in 1 2; do
for v in "" lpt; do
  if [ -z "$v" ]; then export HH_LIB=""; tag=morton; else export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v; fi
  for c in 3d_exp_proxy 3d_laplace; do echo "[$tag] $(timeout 300 python scripts/profile_matvec.py $c 1 3 2>&1 | tail -1)"; done
done
done
unset HH_LIB
echo "$(HH_PROFILE_BUILD=1 timeout 300 python scripts/profile_matvec.py 3d_laplace 16 3 2>&1 | tail -3)"
python scripts/profile_matvec.py 3d_laplace 1 1 > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(gemm|qr|jacobi|resid|factors|decide|dense)" --csv --log-file gpurun_out/launches_build.csv python scripts/profile_matvec.py 3d_laplace 1 1 > gpurun_out/ncu_b.log 2>&1; echo ncu rc $?
