P="python scripts/dbg/x2_probe.py time 256 8 64 64"
for v in "" bs3 nogather_nobload bs3_nn; do
  if [ -n "$v" ]; then export HCB_LIB_PATH=paper_1803_11385_b200/_var/$v/libhcb200.so; else unset HCB_LIB_PATH; fi
  echo "== $v"; timeout 300 $P 2>&1 | tail -1 | cut -c1-150
done
