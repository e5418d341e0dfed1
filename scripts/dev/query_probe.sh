# Phase timing of cfg2 queries, GPU tests, optional launch list / bench.
set -x
ZSVD_PHASE_TIMES=1 python scripts/query_once.py cfg2 500 320000 > gpurun_out/qprobe.log 2>&1
python scripts/dev/fb_probe.py > gpurun_out/fb_probe.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fastpaths.py tests/test_gpu_wide.py -q > gpurun_out/gpu_fast.log 2>&1; echo fast=$?
timeout 1500 python -m pytest tests -m gpu -q ${TESTS:-} > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests.log
[ -n "$LAUNCHES" ] && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv python scripts/query_once.py cfg2 500 320000 > gpurun_out/q_ncu.log 2>&1
[ -n "$BENCH" ] && timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
true
