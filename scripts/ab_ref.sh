timeout 240 python -m pytest tests/test_ops_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for v in "HCB_C2H_CU=16" "HCB_C2H_CU=8" "HCB_C2H_CU=1"; do
  echo "== $v"; env $v python scripts/kbench_ref.py 16 > gpurun_out/ab.txt 2>&1; grep -E "C=.*col2hash" gpurun_out/ab.txt
  env $v python scripts/kbench_ref.py 64 > gpurun_out/ab.txt 2>&1; grep -E "C=.*col2hash" gpurun_out/ab.txt
done
