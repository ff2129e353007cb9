export HH_PROFILE_BUILD=1
python bench.py > gpurun_out/bench_3dlarge.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(gather|phase)" --csv --log-file gpurun_out/launches_3dlarge.csv python bench.py > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 6 -c 2 -o gpurun_out/prof_v2_3dlarge python bench.py > gpurun_out/ncu_full.log 2>&1
echo chain rc $?
tail -1 gpurun_out/bench_3dlarge.log | cut -c1-400
unset HH_PROFILE_BUILD
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -k "3d_large" > gpurun_out/pytest_full3dl.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_full3dl.log
