python scripts/profile_matvec.py 2d_medium 1 3 > gpurun_out/plain_2d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/prof_2d python scripts/profile_matvec.py 2d_medium 1 3 > gpurun_out/ncu_2d.log 2>&1; echo ncu rc $?
