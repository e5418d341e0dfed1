# Round-2 evidence: smoke, GPU tests, bench (default), ncu launch lists (each ncu pass after its plain run exited 0).
set -x
T=${TAG:-r02m}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/${T}_gputests.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/bench_ref.err; echo benchref=$?
python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/plain_profile_run.log 2>&1 || exit 1
ZSVD_DEV_LANES=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches_storage500_query.csv python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_bench_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1
ZSVD_DEBUG=1 python scripts/wide_probe.py cfg3 64 > gpurun_out/${T}_wide_probe.log 2>&1; ZSVD_DEBUG=1 python scripts/wide_probe.py cfg5 8 >> gpurun_out/${T}_wide_probe.log 2>&1
true
