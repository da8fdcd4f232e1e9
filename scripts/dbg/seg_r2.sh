timeout 900 python -m pytest -q -x tests/test_seg_parity.py tests/test_net_gpu.py -p no:cacheprovider 2>&1 | tail -3
for dt in f32 bf16; do timeout 600 python bench.py --workload seg --cin 32 --steps 10 --dtype $dt --no-cpu-baseline > gpurun_out/seg_$dt.json 2>gpurun_out/seg_$dt.err; echo "seg $dt rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/seg_$dt.json')); print(d['dtype'], round(d['ms_per_step'],3), '%.3g'%d['value'])"; done
