set -x
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/we_wide.log 2>&1; echo wide=$?
tail -15 gpurun_out/we_wide.log
ZSVD_DEBUG=1 timeout 300 python scripts/wide_probe.py cfg3 64 > gpurun_out/we_probe.log 2>&1; echo p3=$?
ZSVD_DEBUG=1 timeout 300 python scripts/wide_probe.py cfg5 8 >> gpurun_out/we_probe.log 2>&1; echo p5=$?
grep -v "sweep" gpurun_out/we_probe.log | tail -20
timeout 1200 python -m pytest tests/test_gpu_baseline_parity.py -x -q -k "cfg3 or cfg5" > gpurun_out/we_parity.log 2>&1; echo parity=$?
tail -15 gpurun_out/we_parity.log
