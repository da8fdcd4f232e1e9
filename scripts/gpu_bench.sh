# bench sweep + ncu evidence for the fused path (run under gpurun)
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3"
for c in 16 32 64 128; do
  timeout 300 $B --cin $c --cout $c --no-cpu-baseline > gpurun_out/bench_fused_c$c.json 2> gpurun_out/bench_fused_c$c.err; echo "fused c=$c rc=$?"
  tail -c 1500 gpurun_out/bench_fused_c$c.json; echo; tail -3 gpurun_out/bench_fused_c$c.err
done
timeout 300 $B --path materialized --no-cpu-baseline --no-e2e > gpurun_out/bench_mat_c16.json 2> gpurun_out/bench_mat_c16.err; echo "mat rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_mat_c16.json'));print({k:(v['ms'],v.get('frac')) for k,v in d['kernels'].items()})"
# launch list (cold, serialised) of one short fused run
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fused_c64.csv \
  python bench.py --steps 2 --warmup 1 --cin 64 --cout 64 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
# full captures of the top kernels
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gather|k_field_map" -s 4 -c 4 \
  -o gpurun_out/prof_fused_c64 python bench.py --steps 1 --warmup 1 --cin 64 --cout 64 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -5 gpurun_out/ncu_full.log
ls -la gpurun_out
