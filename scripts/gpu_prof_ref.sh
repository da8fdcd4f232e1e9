# ncu --set full of the reference-layout HBM-bound operators at C=${C:-64}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU:-col2hash|field_map|unpool|max_pool}" -s ${SKIP:-0} -c ${COUNT:-8} \
  -o gpurun_out/${OUT:-prof_ref} python scripts/kbench_ref.py ${C:-64} > gpurun_out/${OUT:-prof_ref}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${OUT:-prof_ref}.log | cut -c1-300
