# halo producers for narrow rows (HCB_FWD_HALO): parity, small-C bench at 256^3 x 8, net step
timeout 900 python -m pytest -q -x tests/test_conv_tc.py tests/test_conv_f32.py tests/test_net_gpu.py tests/test_seg_parity.py -p no:cacheprovider > gpurun_out/halo_t.log 2>&1; tail -3 gpurun_out/halo_t.log
for h in 1; do for dt in bf16 f32; do for cc in "16 16" "16 32" "32 32"; do set -- $cc
HCB_FWD_HALO=$h timeout 600 python bench.py --cin $1 --cout $2 --dtype $dt --steps 10 --no-cpu-baseline --no-ref-kernels --no-e2e 2>gpurun_out/halo_b.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('halo=$h $dt $1->$2', round(d['ms_per_step'],3), {k:round(v['ms'],4) for k,v in d['kernels'].items() if 'ms' in v})"
done; done
HCB_FWD_HALO=$h timeout 600 python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('halo=$h net64 f32', round(d['ms_per_step'],4))"
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_conv_fwd" -c 1 -o gpurun_out/halo python bench.py --cin 16 --cout 16 --dtype bf16 --steps 1 --warmup 3 --no-cpu-baseline --no-ref-kernels --no-e2e > /dev/null 2>&1; echo rc=$?
