# staged pooling + vectorised switch check: parity, timings, per-kernel launch times
timeout 900 python -m pytest -q -x tests/test_ops_gpu.py -p no:cacheprovider 2>&1 | tail -1
for c in 16 32 64 128; do timeout 300 python scripts/kbench_ref.py $c 2>&1 | grep -E "C=.*pool"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"pool|unpool|switch" --csv --log-file gpurun_out/pool_launch.csv python scripts/kbench_ref.py 64 > /dev/null 2>&1; echo rc=$?
