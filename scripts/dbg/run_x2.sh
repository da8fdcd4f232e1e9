P=scripts/dbg/x2_probe.py
for R in 1 2 4 8; do HCB_W_REPL=$R timeout 300 python $P time 256 8 64 64 2>&1 | tail -1 | cut -c1-200; done
for R in 1 4; do HCB_W_REPL=$R timeout 600 python bench.py --steps 20 --warmup 5 --dtype bf16 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bf16 R=$R', d['ms_per_step'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"; done
