# ncu evidence for this round's engine: serialised launch lists (time + DRAM bytes)
# of one 500-block cfg2 storage flush (one lane) plus 3 queries at L = 3.2e5, and
# full captures of the storage Mid-2 (Jacobi) and the query's fused trims / stitch Mid-2.
set -x
python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/plain_profile_run.log 2>&1 || exit 1
ZSVD_DEV_LANES=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01m_launches.csv python scripts/profile_run.py --blocks 500 --queries 3 --lengths 320000 > gpurun_out/ncu_launch.log 2>&1
ZSVD_DEV_LANES=1 ncu --set full --import-source on --clock-control none -k regex:svd_phase_kernel --launch-skip 3 -c 1 \
  -o gpurun_out/r01m_storage_m2 python scripts/profile_run.py --blocks 500 --queries 1 --lengths 320000 > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none -k regex:trim_qr -c 1 -o gpurun_out/r01m_trim_qr python scripts/query_once.py cfg2 500 320000 > gpurun_out/ncu_full2.log 2>&1
true
