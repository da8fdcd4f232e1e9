# max_unpool with the switch-range scan folded into the unpool launch
timeout 900 python -m pytest -q -x tests/test_ops_gpu.py -p no:cacheprovider > gpurun_out/uc_t.log 2>&1; tail -1 gpurun_out/uc_t.log
for c in 16 64 128; do timeout 300 python scripts/kbench_ref.py $c 2>&1 | grep -E "C=.*unpool"; done
