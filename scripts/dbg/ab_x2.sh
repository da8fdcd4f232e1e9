P="python scripts/dbg/x2_probe.py time 256 8"
for c in "64 64" "128 128"; do for v in "HCB_DW_PHASE=0" "HCB_DW_PHASE=1" "HCB_DW_PHASE=0" "HCB_DW_PHASE=1" "HCB_DW_PHASE=0" "HCB_DW_PHASE=1"; do echo -n "C=$c $v: "; env $v timeout 300 $P $c 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['dw'],3), round(d['fwd'],3))"; done; done
