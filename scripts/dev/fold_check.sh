timeout 900 python -m pytest tests/test_gpu_fastpaths.py tests/test_gpu_baseline_parity.py tests/test_gpu_reference_suites.py tests/test_gpu_search.py -x -q > gpurun_out/gpu_fast.log 2>&1; echo fast=$?
tail -2 gpurun_out/gpu_fast.log
python scripts/dev/fb_probe.py > gpurun_out/fb_probe.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv python scripts/query_once.py cfg2 500 320000 > gpurun_out/q_ncu.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
