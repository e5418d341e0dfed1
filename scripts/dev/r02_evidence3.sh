# Round-2 closing evidence: smoke, GPU tests, bench (both arms), query phase stamps, ncu launch lists,
# full capture of the query eigensolver kernel.
set -x
T=${TAG:-r02w}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/${T}_gputests.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/bench_ref.err; echo benchref=$?
ZSVD_PHASE_TIMES=1 python scripts/query_once.py cfg2 500 320000 > gpurun_out/${T}_query_phase_cycles.log 2>&1
python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/plain_profile_run.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches_storage500_query.csv python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_bench_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gram_eig_kernel --launch-skip 2 -c 1 \
  -o gpurun_out/${T}_gram_eig python scripts/query_once.py cfg2 500 320000 > gpurun_out/ncu_full1.log 2>&1
bash scripts/dev/ncu_digest.sh gpurun_out/${T}_gram_eig.ncu-rep gram_eig_kernel > gpurun_out/${T}_gram_eig_digest.txt 2>&1
ls -la gpurun_out/*.ncu-rep
true
