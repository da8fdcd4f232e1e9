for v in "" poolminb6 poolminb8; do
  if [ -n "$v" ]; then export HCB_LIB_PATH=paper_1803_11385_b200/_var/$v/libhcb200.so; fi
  echo "== $v"; timeout 300 python scripts/kbench_ref.py 64 2>&1 | grep -E "C=" | head -12
done
