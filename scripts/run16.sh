python bench.py > gpurun_out/bench_3dlarge_nr1.log 2>&1; echo bench rc $?
python bench.py --nrhs 16 --no-cpu-baseline > gpurun_out/bench_3dlarge_nr16.log 2>&1; echo bench16 rc $?
tail -1 gpurun_out/bench_3dlarge_nr1.log | cut -c1-300
tail -1 gpurun_out/bench_3dlarge_nr16.log | cut -c1-300
timeout 3000 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest rc $?
tail -14 gpurun_out/pytest_gpu_all.log
