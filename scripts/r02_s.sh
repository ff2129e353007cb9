# round-2 run s: ncu --set full of the final 16-RHS phase kernels on the proxy
mkdir -p gpurun_out
python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/r02s_plain16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/r02s_prof16 \
    python scripts/profile_matvec.py 3d_exp_proxy 16 3 > gpurun_out/r02s_ncu16.log 2>&1; echo "ncu16 rc $?"
python scripts/ncu_summary.py gpurun_out/r02s_prof16.ncu-rep > gpurun_out/r02s_proxy_nrhs16_ncu.txt 2>&1
