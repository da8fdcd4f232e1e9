show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2)); print({k:(round(v['ms'],3) if 'ms' in v else v) for k,v in d['kernels'].items()})" $1; }
for o in 0 1 0 1; do HCB_BENCH_OVERLAP=$o python bench.py --no-cpu-baseline --no-ref-kernels --steps 20 > gpurun_out/b_ovl$o.json 2>gpurun_out/b_ovl$o.err; show gpurun_out/b_ovl$o.json; done
