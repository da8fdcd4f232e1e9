# repeatability of the default bench line on one box: 5 back-to-back runs
for i in 1 2 3 4 5; do timeout 600 python bench.py --no-cpu-baseline --no-ref-kernels --steps 20 > gpurun_out/var_$i.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/var_$i.json')); print($i, round(d['ms_per_step'],3), 'ms', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'], {k:round(v['ms'],3) for k,v in d['kernels'].items() if 'ms' in v})"; done
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit,temperature.gpu --format=csv
