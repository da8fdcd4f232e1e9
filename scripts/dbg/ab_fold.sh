timeout 900 python -m pytest -q -x tests/test_net_gpu.py tests/test_net_parity.py tests/test_net_dist_gpu.py -p no:cacheprovider > gpurun_out/fold_t.log 2>&1; tail -2 gpurun_out/fold_t.log
for k in 1 2 3; do timeout 600 python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('net64 f32', round(d['ms_per_step'],4))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_bn_fold" --csv --log-file gpurun_out/fold_launch.csv python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 1 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
