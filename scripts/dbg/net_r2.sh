timeout 900 python -m pytest -q -x tests/test_net_gpu.py tests/test_net_parity.py tests/test_net_dist_gpu.py tests/test_seg_parity.py -p no:cacheprovider 2>&1 | tail -2
for dt in f32 bf16; do timeout 600 python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 20 --dtype $dt > gpurun_out/net64_$dt.json 2>gpurun_out/net64_$dt.err; echo "net64 $dt rc=$?"; tail -c 700 gpurun_out/net64_$dt.json | head -c 700; echo; done
timeout 600 python bench.py --workload net --res 128 --shapes-per-gpu 64 --steps 10 --dtype bf16 --no-cpu-baseline > gpurun_out/net128_bf16.json 2>gpurun_out/net128_bf16.err; echo "net128 rc=$?"
timeout 600 python bench.py --workload net --res 128 --shapes-per-gpu 64 --steps 10 --dtype f32 --no-cpu-baseline > gpurun_out/net128_f32.json 2>gpurun_out/net128_f32.err; echo "net128 f32 rc=$?"
python -c "
import json
for f in ['net64_f32','net64_bf16','net128_bf16','net128_f32']:
    try:
        d=json.load(open('gpurun_out/'+f+'.json')); print(f, round(d['ms_per_step'],3), 'ms', round(d['value']), 'shapes/s', d.get('vs_baseline'), (d.get('cpu_baseline') or {}).get('value'))
    except Exception as e: print(f, e)
"
