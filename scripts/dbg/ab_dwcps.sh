# dW with the shared tri accumulator: CTAs per SM / producer warps / accumulator double-buffering
P="python scripts/dbg/x2_probe.py time 256 8"
for v in "HCB_DW_CPS=2" "HCB_DW_CPS=1" "HCB_DW_CPS=1 HCB_DW_PW=4" "HCB_DW_CPS=2 HCB_DW_DBUF=1" "HCB_DW_CPS=2" "HCB_DW_CPS=1"; do echo -n "C=64 $v: "; env $v timeout 300 $P 64 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['dw'],3), round(d['fwd'],3))"; done
