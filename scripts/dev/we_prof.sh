set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02n_gputests.log 2>&1; echo tests=$?
tail -5 gpurun_out/r02n_gputests.log
timeout 900 python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/bench.err; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02n_launches_wide_cfg5_8blk.csv python scripts/wide_probe.py cfg5 8 1 > gpurun_out/ncu_w5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02n_launches_wide_cfg3_64blk.csv python scripts/wide_probe.py cfg3 64 1 > gpurun_out/ncu_w3.log 2>&1
true
