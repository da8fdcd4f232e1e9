mkdir -p gpurun_out
run() { env "$@" timeout 200 python scripts/kbench.py ${CS:-64} 2>&1 | grep -E "C=|Error|error" | tail -4; }
run HCB_X=default
run HCB_DW_PW=2 HCB_FWD_PW=2
