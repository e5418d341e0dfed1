for env in "" "ZSVD_SVD_TRIMS=1" "ZSVD_TWO_PASS=1" "ZSVD_SVD_TRIMS=1 ZSVD_TWO_PASS=1"; do
  echo "== $env"; env $env timeout 600 python -m pytest tests/test_gpu_wide.py -x -q 2>&1 | tail -4
done
