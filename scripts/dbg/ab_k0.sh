# K0 by column runs (k_field_map_runs) vs the 27-probe kernel: parity, then timings in the fused step
timeout 900 python -m pytest -q -x tests/test_ops_gpu.py -p no:cacheprovider -k "field_map or golden or random or full_size or shell" > gpurun_out/k0_t1.log 2>&1; tail -1 gpurun_out/k0_t1.log
timeout 900 python -m pytest -q -x tests/test_conv_tc.py tests/test_conv_f32.py -p no:cacheprovider > gpurun_out/k0_t2.log 2>&1; tail -1 gpurun_out/k0_t2.log
for v in 0 1 0 1; do HCB_K0_RUNS=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('K0_RUNS=$v', round(d['ms_per_step'],3), round(d['kernels']['field_map']['ms'],4))"; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_field_map_runs" -c 1 -o gpurun_out/k0runs python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels > /dev/null 2>&1; echo rc=$?
