timeout 1800 python -m pytest -q tests/test_seg_parity.py tests/test_net_parity.py tests/test_net_dist_gpu.py tests/test_net_gpu.py -x 2>&1 | tail -25
