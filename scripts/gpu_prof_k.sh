# ncu --set full of the native conv kernels at C=${C:-64} (kbench driver: short, one GPU)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU:-k_conv}" -s ${SKIP:-2} -c ${COUNT:-2} \
  -o gpurun_out/${OUT:-prof_k} python scripts/kbench.py ${C:-64} > gpurun_out/${OUT:-prof_k}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${OUT:-prof_k}.log | cut -c1-300
