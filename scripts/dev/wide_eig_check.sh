set -x
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/we_wide.log 2>&1; echo wide=$?
tail -5 gpurun_out/we_wide.log
ZSVD_DEBUG=1 timeout 300 python scripts/wide_probe.py cfg3 100 3 > gpurun_out/we_probe.log 2>&1; echo p3=$?
ZSVD_DEBUG=1 timeout 300 python scripts/wide_probe.py cfg5 16 3 >> gpurun_out/we_probe.log 2>&1; echo p5=$?
grep -v "sweep" gpurun_out/we_probe.log | tail -20
timeout 300 python scripts/query_once.py cfg3 100 320000 2>&1 | grep -v sweep | tail -6
timeout 300 python scripts/query_once.py cfg5 17 131072 2>&1 | grep -v sweep | tail -6
timeout 300 python scripts/query_once.py cfg5 17 10000 2>&1 | grep -v sweep | tail -6
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/we_launches_q5.csv python scripts/query_once.py cfg5 17 131072 > gpurun_out/ncu_q5.log 2>&1
