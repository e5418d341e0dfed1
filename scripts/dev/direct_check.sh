set -x
ZSVD_PHASE_TIMES=1 timeout 300 python scripts/profile_run.py --blocks 500 --queries 2 --lengths 320000 2>&1 | grep -v "^\[zsvd\]   task0" | tail -30
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/dc_gputests.log 2>&1; echo tests=$?
tail -12 gpurun_out/dc_gputests.log
timeout 900 python bench.py > gpurun_out/dc_bench.json 2> gpurun_out/bench.err; echo bench=$?
python - <<'P'
import json
d=json.loads(open('gpurun_out/dc_bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'q p50',d['config'].get('query_p50_ms_L320000'),'e2e',d['e2e']['value'])
for c in ('cfg3','cfg5'):
    o=d['other_configs'][c]; print(c,o['storage_rows_s'],o['roofline']['frac'],o['query_p50_ms'])
P
