# round-2 closing evidence on the final code (planned single-RHS producer): full GPU suite, bench
# (nrhs 1 with the multi_rhs sub-record; --nrhs 16), ncu launch list + full capture of the bench
# command, every other BASELINE config, ncu of the NR=1 kernels on 2D medium
bash scripts/gpu_round.sh
bash scripts/bench_all.sh
python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > gpurun_out/r02m_3dlarge_ncu.txt 2>&1
python scripts/profile_matvec.py 2d_medium 1 3 > gpurun_out/r02m_plain2d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 2 -o gpurun_out/r02m_prof2d \
    python scripts/profile_matvec.py 2d_medium 1 3 > gpurun_out/r02m_ncu2d.log 2>&1; echo "ncu2d rc $?"
python scripts/ncu_summary.py gpurun_out/r02m_prof2d.ncu-rep > gpurun_out/r02m_2dmedium_ncu.txt 2>&1
python __graft_entry__.py smoke > gpurun_out/r02m_smoke.txt 2>&1; echo "smoke rc $?"
