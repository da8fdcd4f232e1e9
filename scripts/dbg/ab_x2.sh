P="python scripts/dbg/x2_probe.py time 256 8"
for c in "64 64" "32 32" "64 64" "32 32"; do for t in 1 0; do echo -n "C=$c shared=$t "; HCB_DW_TRI_SHARED=$t timeout 300 $P $c 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['dw'],3), round(d['fwd'],3))"; done; done
