# small-C tap-major producer mapping (HCB_SMALLC_TAPMAJOR) A/B: parity, bench at 256^3 x 8, net step
timeout 900 python -m pytest -q -x tests/test_conv_tc.py tests/test_conv_f32.py tests/test_net_gpu.py -p no:cacheprovider > gpurun_out/sc_t.log 2>&1; tail -1 gpurun_out/sc_t.log
for dt in f32 bf16; do for cc in "8 16" "16 16" "16 32"; do set -- $cc
timeout 600 python bench.py --cin $1 --cout $2 --dtype $dt --steps 10 --no-cpu-baseline --no-ref-kernels --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$dt $1->$2', round(d['ms_per_step'],3), {k:round(v['ms'],4) for k,v in d['kernels'].items() if 'ms' in v})"
done; done
timeout 600 python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('net64 f32', round(d['ms_per_step'],4))"
echo "== previous mapping (HCB_SMALLC_TAPMAJOR=0 build)"
for dt in f32 bf16; do for cc in "8 16" "16 16" "16 32"; do set -- $cc
HCB_LIB_PATH=_ab/libhcb200_off.so timeout 600 python bench.py --cin $1 --cout $2 --dtype $dt --steps 10 --no-cpu-baseline --no-ref-kernels --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$dt $1->$2', round(d['ms_per_step'],3), {k:round(v['ms'],4) for k,v in d['kernels'].items() if 'ms' in v})"
done; done
HCB_LIB_PATH=_ab/libhcb200_off.so timeout 600 python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('net64 f32', round(d['ms_per_step'],4))"
