timeout 900 python -m pytest -q -x tests/test_ops_gpu.py -p no:cacheprovider -k "pool or golden or random or kat or idempot or full_size" 2>&1 | tail -2
HCB_POOL_SPAN=2 timeout 900 python -m pytest -q -x tests/test_ops_gpu.py -p no:cacheprovider -k "pool or golden or random or kat or idempot" 2>&1 | tail -1
for v in 1 2 0; do echo "== HCB_POOL_SPAN=$v"; HCB_POOL_SPAN=$v timeout 300 python scripts/kbench_ref.py 64 2>&1 | grep -E "C=.*pool"; done
