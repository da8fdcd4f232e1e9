timeout 600 python -m pytest -q -x tests/test_ops_gpu.py -k "tiled_field_map or field_map or native" -p no:cacheprovider 2>&1 | tail -2
for r in 1 0 1 0; do HCB_K0_RUNS=$r timeout 300 python scripts/kbench.py 64 2>&1 | tail -1; done
