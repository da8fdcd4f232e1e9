# fp32 and bf16 fused conv layer fwd+dW+dX at 256^3 x 8 over C (bench.py lines, one per config)
mkdir -p gpurun_out/csweep
for dt in f32 bf16; do for c in 16 32 64 128; do
  timeout 600 python bench.py --cin $c --cout $c --dtype $dt --steps 10 --no-cpu-baseline --no-ref-kernels --no-e2e > gpurun_out/csweep/${dt}_c$c.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/csweep/${dt}_c$c.json'))
k=d['kernels']; print('$dt C=$c', round(d['ms_per_step'],3), 'ms', '%.3g vox/s'%d['value'], ' '.join(f\"{n}={v['ms']:.3f}ms/{v.get('frac_tensor', v.get('frac',0)):.2f}\" for n,v in k.items() if 'ms' in v))"
done; done
