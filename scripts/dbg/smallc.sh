for dt in f32 bf16; do for cc in "8 16" "3 2" "16 16"; do set -- $cc
timeout 600 python bench.py --cin $1 --cout $2 --dtype $dt --steps 10 --no-cpu-baseline --no-ref-kernels --no-e2e > gpurun_out/smallc_${dt}_$1_$2.json 2>gpurun_out/smallc.err; echo "$dt $1->$2 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/smallc_${dt}_$1_$2.json')); print(round(d['ms_per_step'],3), {k:(round(v['ms'],3), round(v.get('frac',v.get('frac_tensor',0)),3)) for k,v in d['kernels'].items() if 'ms' in v})"
done; done
timeout 600 python - <<'PY'
import sys, time, torch; sys.path.insert(0,'.')
import bench
from paper_1803_11385_b200 import ops
from paper_1803_11385_b200.ops import ConvSpec
from paper_1803_11385_b200.psh import SuperPsh
lv = bench.shell_levels(256)
for b in (1,):
    s = SuperPsh.from_levels([lv[0]] * b); n = s.total_columns()
    for mode in ("exact", "fast"):
        ctx = ops.math_mode(mode); ctx.__enter__()
        x = torch.rand((64, n), device="cuda"); w = torch.rand((64, 64*27), device="cuda"); dy = torch.rand((64, n), device="cuda")
        sp = ConvSpec(3,1,0,64,64)
        for rep in range(2):
            torch.cuda.synchronize(); t=time.time()
            y = ops.conv_forward(s, x, s, w, sp)
            cols = ops.hash2col(s, x, s, sp)
            g = ops.conv_backward(dy, w, cols, s, s, sp)
            torch.cuda.synchronize(); dt=time.time()-t
        ctx.__exit__(None, None, None)
        print(f"reference-layout conv_forward+hash2col+conv_backward, 256^3 x {b} ({n} voxels), C 64->64, math={mode}: {dt*1e3:.1f} ms")
PY
