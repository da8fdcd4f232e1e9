# round-2 evidence pass at HEAD: gpu tests, smoke, default bench line (f32), bf16 line, reference arm,
# launch list + ncu --set full of the step's kernels, reference-layout kernel table, net / seg benches
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --dtype bf16 --no-cpu-baseline --no-ref-kernels > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err; echo "bench bf16 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 20 > gpurun_out/bench_net64.json 2>gpurun_out/bench_net64.err; echo "net64 rc=$?"
timeout 600 python bench.py --workload seg --cin 32 --steps 10 --no-cpu-baseline > gpurun_out/bench_seg.json 2>gpurun_out/bench_seg.err; echo "seg rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f32.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_conv|k_field_map|k_split|k_reduce" -s 12 -c 7 \
  -o gpurun_out/prof_f32 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels > gpurun_out/prof_f32.log 2>&1; echo "ncu full rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/bench.json')); print('f32', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['roofline']['kernel'], round(d['roofline']['frac'],3), {k:round(v['ms'],3) for k,v in d['kernels'].items() if 'ms' in v})
d=json.load(open('gpurun_out/bench_bf16.json')); print('bf16', round(d['ms_per_step'],3), '%.4g'%d['value'])
"
