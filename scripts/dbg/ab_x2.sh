timeout 900 python -m pytest -q -x tests/test_conv_f32.py tests/test_conv_tc.py tests/test_dropin_cpp.py -p no:cacheprovider 2>&1 | tail -3
for c in "64 64" "16 16" "32 32" "128 128"; do HCB_X2_DW_TRI=1 timeout 300 python scripts/dbg/x2_probe.py time 256 8 $c | cut -c1-160; done
