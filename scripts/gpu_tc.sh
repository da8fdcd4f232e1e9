mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_conv_tc.py -q -rf -x -p no:cacheprovider > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_tc.log
