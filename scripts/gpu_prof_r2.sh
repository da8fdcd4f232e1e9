# round-2 evidence: launch list + one ncu --set full capture of each kernel of the default (f32) step
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f32.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU:-k_conv|k_field_map_tiled|k_split}" -s ${SKIP:-10} -c ${COUNT:-6} \
  -o gpurun_out/${OUT:-prof_f32} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels ${ARGS} > gpurun_out/${OUT:-prof_f32}.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/${OUT:-prof_f32}.log | cut -c1-300
