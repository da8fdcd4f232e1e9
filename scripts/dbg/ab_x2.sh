for v in "" unroll4 unroll16 "" unroll4 unroll16; do
  if [ -n "$v" ]; then export HCB_LIB_PATH=paper_1803_11385_b200/_var/$v/libhcb200.so; else unset HCB_LIB_PATH; fi
  echo -n "$v: "; timeout 300 ncu --metrics gpu__time_duration.sum -k regex:k_reduce_dw -c 3 python scripts/dbg/x2_probe.py time 256 8 64 64 2>&1 | grep duration | tail -1
done
