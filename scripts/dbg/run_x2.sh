timeout 900 python -m pytest -q -x tests/test_conv_f32.py -k "random_maps or full_size" 2>&1 | tail -2
HCB_DW_DBUF=1 timeout 900 python -m pytest -q -x tests/test_conv_f32.py -k "random_maps or full_size" 2>&1 | tail -2
for D in 0 1; do for T in 16 32; do echo -n "D=$D T=$T "; HCB_DW_DBUF=$D HCB_X2_DW_TPS=$T timeout 300 python scripts/dbg/x2_probe.py time 256 8 64 64 2>&1 | tail -1 | cut -c60-140; done; done
