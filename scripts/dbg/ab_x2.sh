HCB_X2_RING=9 timeout 900 python -m pytest -q -x tests/test_conv_f32.py -p no:cacheprovider -k "random or shell or tiny" 2>&1 | tail -1
P="python scripts/dbg/x2_probe.py time 256 8 64 64"
for r in 8 9 8 9; do echo "ring $r"; HCB_X2_RING=$r timeout 300 $P 2>&1 | tail -1 | cut -c1-150; done
