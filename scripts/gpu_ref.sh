# reference-layout operators: parity tests + HBM-roofline table
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_ops.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ops.log
for c in ${CS:-16 64 256}; do timeout 300 python scripts/kbench_ref.py $c 2>&1 | grep "C="; done
