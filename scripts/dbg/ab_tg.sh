# TMA row-gather (tile::gather4) producer for the split forward / dX (HCB_X2_RING=9) vs cp.async gathers (8)
HCB_X2_RING=9 timeout 900 python -m pytest -q -x tests/test_conv_f32.py tests/test_conv_tc.py -p no:cacheprovider > gpurun_out/tg_t.log 2>&1; tail -2 gpurun_out/tg_t.log
for r in 9 8 9 8; do HCB_X2_RING=$r timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels 2>gpurun_out/tg_b.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ring=$r', round(d['ms_per_step'],3), {k:round(v['ms'],4) for k,v in d['kernels'].items() if 'ms' in v})"; done
HCB_X2_RING=9 timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_conv_fwd_x2" -c 1 -o gpurun_out/tg python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels > /dev/null 2>&1; echo rc=$?
