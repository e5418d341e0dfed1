timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/gpu_wide.log 2>&1; echo wide=$?
tail -2 gpurun_out/gpu_wide.log
ZSVD_DEBUG=1 python scripts/wide_probe.py cfg3 64 > gpurun_out/wide_probe.log 2>&1; ZSVD_DEBUG=1 python scripts/wide_probe.py cfg5 8 >> gpurun_out/wide_probe.log 2>&1
ZSVD_TWO_PASS=1 python scripts/wide_probe.py cfg3 64 > gpurun_out/wide_probe_2pass.log 2>&1; ZSVD_TWO_PASS=1 python scripts/wide_probe.py cfg5 8 >> gpurun_out/wide_probe_2pass.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
