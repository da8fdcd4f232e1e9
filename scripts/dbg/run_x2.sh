timeout 300 python scripts/kbench_ref.py 64 2>&1 | grep -E "C=.*pool"
HCB_LIB_PATH=paper_1803_11385_b200/_var/stcs/libhcb200.so timeout 300 python scripts/kbench_ref.py 64 2>&1 | grep -E "C=.*pool"
