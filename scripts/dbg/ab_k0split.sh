# K0 fused with the input split (hc_field_map_tiled_split) vs the two launches
timeout 900 python -m pytest -q -x tests/test_ops_gpu.py -p no:cacheprovider -k "field_map" > gpurun_out/k0s_t.log 2>&1; tail -1 gpurun_out/k0s_t.log
for v in 1 0 1 0; do HCB_BENCH_K0SPLIT=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('k0split=$v', round(d['ms_per_step'],3), {k:round(v['ms'],4) for k,v in d['kernels'].items() if 'ms' in v})"; done
