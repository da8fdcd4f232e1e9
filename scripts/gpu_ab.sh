mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_conv_tc.py tests/test_net_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_tc.log
run() { env "$@" timeout 200 python scripts/kbench.py ${CS:-64} 2>&1 | grep -E "C=|Error|error" | tail -5; }
run HCB_X=default
