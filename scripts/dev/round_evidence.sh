# Round evidence: smoke, GPU tests, bench (default), then ncu launch lists and
# full captures of the top kernels (each ncu pass after its plain run exited 0).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/plain_profile_run.log 2>&1 || exit 1
ZSVD_DEV_LANES=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01o_launches.csv python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01o_bench_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1
ZSVD_DEV_LANES=1 ncu --set full --import-source on --clock-control none -k regex:svd_phase_kernel --launch-skip 3 -c 1 \
  -o gpurun_out/r01o_storage_m2 python scripts/profile_run.py --blocks 500 --queries 1 --lengths 320000 > gpurun_out/ncu_full1.log 2>&1
ZSVD_DEV_LANES=1 ncu --set full --import-source on --clock-control none -k regex:svd_phase_kernel --launch-skip 4 -c 1 \
  -o gpurun_out/r01o_storage_p3 python scripts/profile_run.py --blocks 500 --queries 1 --lengths 320000 > gpurun_out/ncu_full2.log 2>&1
ncu --set full --clock-control none -k regex:trim_qr -c 1 -o gpurun_out/r01o_trim_qr python scripts/query_once.py cfg2 500 320000 > gpurun_out/ncu_full3.log 2>&1
true
