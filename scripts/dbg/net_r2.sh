timeout 900 python -m pytest -q -x tests/test_net_gpu.py tests/test_net_parity.py tests/test_net_dist_gpu.py -p no:cacheprovider 2>&1 | tail -2
for dt in f32 bf16; do timeout 600 python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 20 --dtype $dt --no-cpu-baseline > gpurun_out/net64_$dt.json 2>gpurun_out/net64_$dt.err; echo "net64 $dt rc=$?"; done
python -c "
import json
for f in ['net64_f32','net64_bf16']:
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, round(d['ms_per_step'],3), 'ms', round(d['value']), 'shapes/s', d.get('gpu_launches'))
"
