timeout 600 python -m pytest tests/test_gpu_fastpaths.py tests/test_gpu_baseline_parity.py tests/test_gpu_reference_suites.py -x -q > gpurun_out/gpu_fast.log 2>&1; echo fast=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
ZSVD_NO_PDL=1 timeout 900 python bench.py > gpurun_out/bench_nopdl.json 2> gpurun_out/bench_nopdl.err; echo bench=$?
