timeout 900 python -m pytest -q -x tests/test_conv_f32.py tests/test_conv_tc.py -p no:cacheprovider 2>&1 | tail -1
P="python scripts/dbg/x2_probe.py time 256 8 64 64"
run() { echo "$* : "; env "$@" timeout 300 $P 2>&1 | tail -1 | cut -c1-150; }
run HCB_DW_PHASE=1
run HCB_DW_PHASE=0
run HCB_DW_PHASE=1
run HCB_DW_PHASE=0
for c in "128 128" "32 32"; do for ph in 1 0; do echo "C=$c phase=$ph"; HCB_DW_PHASE=$ph timeout 300 python scripts/dbg/x2_probe.py time 256 8 $c 2>&1 | tail -1 | cut -c1-150; done; done
