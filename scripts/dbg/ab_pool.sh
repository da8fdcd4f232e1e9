timeout 900 python -m pytest -q -x tests/test_ops_gpu.py -p no:cacheprovider -k "pool or golden or random or kat or idempot or full_size" 2>&1 | tail -2
for v in 1 0 1; do echo "== HCB_POOL_RUNS=$v"; HCB_POOL_RUNS=$v timeout 300 python scripts/kbench_ref.py 64 2>&1 | grep -E "C=.*pool"; done
HCB_RES=512 HCB_BATCH=8 timeout 300 python scripts/kbench_ref.py 16 2>&1 | grep -E "C=.*pool"
