# round-2 run o: the new stage-geometry parity test and the neighbouring subprocess tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "geometry or row_split or determin" --durations=3 > gpurun_out/r02o_pytest.txt 2>&1; echo "pytest rc $?"
