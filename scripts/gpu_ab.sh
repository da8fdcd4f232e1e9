mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
run() { env "$@" timeout 200 python scripts/kbench.py ${CS:-64} 2>&1 | grep -E "C=|Error|error" | tail -4; }
run HCB_X=default
for c in 16 64 256; do timeout 300 python scripts/kbench_ref.py $c 2>&1 | grep "C="; done
