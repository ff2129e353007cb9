python scripts/profile_matvec.py 3d_laplace 1 3 > gpurun_out/plain_3dlap.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/prof_v0_3dlap python scripts/profile_matvec.py 3d_laplace 1 3 > gpurun_out/ncu_v0.log 2>&1
echo rc $?
