timeout 900 python -m pytest -q -x tests/test_conv_f32.py tests/test_conv_tc.py -p no:cacheprovider 2>&1 | tail -2
P="python scripts/dbg/x2_probe.py time 256 8 64 64"
run() { echo "$* : "; env "$@" timeout 300 $P 2>&1 | tail -1 | cut -c1-150; }
run HCB_DW_STRIDED=1
run HCB_DW_STRIDED=0
run HCB_DW_STRIDED=1
run HCB_DW_STRIDED=0
run HCB_DW_STRIDED=1 HCB_X2_DW_TPS=16
run HCB_DW_STRIDED=1 HCB_DW_DBUF=1
for c in "128 128" "32 32"; do for st in 1 0; do echo "C=$c strided=$st"; HCB_DW_STRIDED=$st timeout 300 python scripts/dbg/x2_probe.py time 256 8 $c 2>&1 | tail -1 | cut -c1-150; done; done
HCB_DW_STRIDED=1 timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:k_conv_dw -c 2 python scripts/dbg/x2_probe.py time 256 8 64 64 2>&1 | grep -E "dram|duration" 
HCB_DW_STRIDED=0 timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:k_conv_dw -c 2 python scripts/dbg/x2_probe.py time 256 8 64 64 2>&1 | grep -E "dram|duration" 
