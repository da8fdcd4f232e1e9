timeout 900 python -m pytest -q -x tests/test_ops_gpu.py tests/test_net_gpu.py -p no:cacheprovider -k "pool or golden or random or kat or idempot" 2>&1 | tail -2
for v in 1 0 1; do echo "== HCB_POOL_SEG=$v"; HCB_POOL_SEG=$v timeout 300 python scripts/kbench_ref.py 64 2>&1 | grep -E "pool"; done
HCB_RES=512 HCB_BATCH=8 timeout 300 python scripts/kbench_ref.py 16 2>&1 | grep -E "pool"
