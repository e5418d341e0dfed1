# fused-trim tests, fallback counts, query launch list, bench
timeout 300 python -m pytest tests/test_gpu_fastpaths.py -x -q > gpurun_out/gpu_fast.log 2>&1; echo fast=$?
tail -3 gpurun_out/gpu_fast.log
python scripts/dev/fb_probe.py > gpurun_out/fb_probe.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv python scripts/query_once.py cfg2 500 320000 > gpurun_out/q_ncu.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
