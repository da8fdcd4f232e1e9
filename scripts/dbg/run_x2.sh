P=scripts/dbg/x2_probe.py
for G in 0 1; do HCB_FWD_GMAP=$G timeout 300 python $P time 256 8 64 64 2>&1 | tail -1 | cut -c1-260; done
for G in 0 1; do HCB_FWD_GMAP=$G timeout 300 python $P time 256 8 32 32 2>&1 | tail -1 | cut -c1-260; done
HCB_FWD_GMAP=1 timeout 300 python $P shell 64 2 64 64 2>&1 | tail -1
for G in 0 1; do HCB_FWD_GMAP=$G timeout 600 python bench.py --steps 20 --warmup 5 --dtype bf16 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bf16 G=$G', d['ms_per_step'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"; done
HCB_FWD_GMAP=1 timeout 600 python -m pytest -q -x tests/test_conv_tc.py 2>&1 | tail -2
