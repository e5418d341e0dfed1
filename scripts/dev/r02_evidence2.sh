# Round-2 final evidence: smoke, GPU tests, bench (both arms), ncu launch lists, full captures of the new kernels.
set -x
T=${TAG:-r02t}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/${T}_gputests.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/bench_ref.err; echo benchref=$?
python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/plain_profile_run.log 2>&1 || exit 1
ZSVD_DEV_LANES=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches_storage500_query.csv python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_bench_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_wide_cfg5_16blk.csv python scripts/wide_probe.py cfg5 16 1 > gpurun_out/ncu_w5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_wide_cfg3_100blk.csv python scripts/wide_probe.py cfg3 100 1 > gpurun_out/ncu_w3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_query_cfg3.csv python scripts/query_once.py cfg3 100 320000 > gpurun_out/ncu_q3.log 2>&1
ZSVD_DEV_LANES=1 ncu --set full --import-source on --clock-control none -k regex:storage_eig_kernel -c 1 \
  -o gpurun_out/${T}_storage_eig python scripts/profile_run.py --blocks 500 --queries 1 --lengths 320000 > gpurun_out/ncu_full1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:wide_tridiag_kernel -c 1 \
  -o gpurun_out/${T}_wide_tridiag python scripts/wide_probe.py cfg5 16 1 > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out/*.ncu-rep
true
