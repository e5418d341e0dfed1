# Closing run at HEAD: smoke, GPU tests, bench (both arms).
set -x
T=${TAG:-r02y}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/${T}_gputests.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/bench_ref.err; echo benchref=$?
true
