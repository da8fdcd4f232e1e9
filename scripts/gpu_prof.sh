# ncu full capture (source-level) of selected kernels at C=$C
mkdir -p gpurun_out
C=${C:-64}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU:-k_gather}" -s ${SKIP:-4} -c ${COUNT:-3} \
  -o gpurun_out/${OUT:-prof} python bench.py --steps 1 --warmup 1 --cin $C --cout $C --no-cpu-baseline --no-e2e > gpurun_out/${OUT:-prof}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${OUT:-prof}.log | cut -c1-300
