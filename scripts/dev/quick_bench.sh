timeout 300 python -m pytest tests/test_gpu_fastpaths.py tests/test_gpu_baseline_parity.py -x -q > gpurun_out/gpu_fast.log 2>&1; echo fast=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
ZSVD_DEV_LANES=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/storage_launches.csv python scripts/profile_run.py --blocks 500 --queries 1 --lengths 320000 > gpurun_out/ncu_launch.log 2>&1
