ncu --set full --import-source on --clock-control none -k regex:trim_qr -c 2 -o gpurun_out/trim_qr2 python scripts/query_once.py cfg2 500 320000 > gpurun_out/ncu_trim.log 2>&1
ZSVD_ENGINE_TRIMS=1 python scripts/query_once.py cfg2 500 320000 > gpurun_out/q_engine_trims.log 2>&1
python scripts/query_once.py cfg2 500 320000 > gpurun_out/q_fused_trims.log 2>&1
