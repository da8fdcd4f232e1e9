# quick iteration: native tests, then a fused bench sweep (+ optional ncu capture)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_conv_tc.py -q -x -p no:cacheprovider > gpurun_out/pytest_tc.log 2>&1; echo "pytest_tc rc=$?"; tail -15 gpurun_out/pytest_tc.log
for c in ${CS:-16 64 128}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --cin $c --cout $c --no-cpu-baseline --no-e2e > gpurun_out/it_c$c.json 2>gpurun_out/it_c$c.err; echo "c=$c rc=$?"; tail -2 gpurun_out/it_c$c.err
  python -c "import json;d=json.load(open('gpurun_out/it_c$c.json'));print('value %.3e ms %.3f'%(d['value'],d['ms_per_step']));[print('  %-10s %.3f ms %s'%(k,v['ms'],{kk:round(vv,3) for kk,vv in v.items() if kk in ('frac','frac_tensor','achieved_TFLOPs','achieved_GBps')})) for k,v in d['kernels'].items()]"
done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 4 -c 3 \
  -o gpurun_out/prof_iter python bench.py --steps 1 --warmup 1 --cin 64 --cout 64 --no-cpu-baseline --no-e2e > gpurun_out/ncu_iter.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_iter.log
fi
