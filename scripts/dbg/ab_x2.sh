timeout 900 python -m pytest -q -x tests/test_conv_f32.py tests/test_net_gpu.py tests/test_dropin_cpp.py -p no:cacheprovider 2>&1 | tail -2
for c in "64 64" "64 32" "128 64" "32 64"; do timeout 300 python scripts/dbg/x2_probe.py time 256 8 $c 2>&1 | tail -1 | cut -c1-150; HCB_X2_RING=2 timeout 300 python scripts/dbg/x2_probe.py time 256 8 $c 2>&1 | tail -1 | cut -c1-150; done
