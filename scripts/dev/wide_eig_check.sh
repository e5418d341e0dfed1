set -x
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/we_wide.log 2>&1; echo wide=$?
tail -5 gpurun_out/we_wide.log
timeout 300 python scripts/wide_probe.py cfg3 100 3 2>&1 | tail -3
timeout 300 python scripts/wide_probe.py cfg5 16 3 2>&1 | tail -3
timeout 300 python scripts/query_once.py cfg3 100 320000 2>&1 | tail -3
timeout 300 python scripts/query_once.py cfg5 17 131072 2>&1 | tail -3
timeout 300 python scripts/query_once.py cfg5 17 10000 2>&1 | tail -3
