python scripts/csv_probe.py 1000000 2>&1 | tail -4
ZSVD_CSV_TRACE=1 python -c "
import sys; sys.path.insert(0,'.')
from paper_1805_00754_b200 import api
import time
for i in range(3):
    t=time.perf_counter(); f=api._CsvFile('/tmp/zsvd_csv_cfg2_1000000.csv', None); print(time.perf_counter()-t, flush=True)
"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/csv_launches.csv python -c "
import sys; sys.path.insert(0,'.')
from paper_1805_00754_b200 import api
f=api._CsvFile('/tmp/zsvd_csv_cfg2_1000000.csv', None)
" > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/csv_launches.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    try: v=float(r[vi].replace(',',''))
    except: continue
    a=agg[r[ki][:40]]; a[0]+=1; a[1]+=v
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{k:42s} {n:5d} {t/1e6:9.3f} ms")
PY
