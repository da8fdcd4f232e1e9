# native conv: parity tests, then a kernel A/B sweep (env knobs and variant builds)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_conv_tc.py -q -x -p no:cacheprovider > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tc.log
run() { env "$@" timeout 200 python scripts/kbench.py ${CS:-64} 2>&1 | grep -E "C=|Error|error" | tail -4; }
run HCB_DW_PW=8
run HCB_DW_PW=4
run HCB_FWD_CPS=1 HCB_FWD_PW=4
