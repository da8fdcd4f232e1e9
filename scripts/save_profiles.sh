# copy the evidence of scripts/gpu_round.sh (gpurun_out/) into profiles/ (round prefix $1, default r01)
R=${1:-r01}
python scripts/ncu_summary.py gpurun_out/prof_round.ncu-rep gpurun_out/launches.csv > profiles/${R}_ncu_fused_c64.md
cp gpurun_out/launches.csv profiles/${R}_launches_fused_c64.csv
cp gpurun_out/bench.json profiles/${R}_bench_c64.json
cp gpurun_out/bench_ref.json profiles/${R}_bench_reference_c64.json
for f in net64 net128 net32 seg; do cp gpurun_out/bench_$f.json profiles/${R}_bench_$f.json; done
cp gpurun_out/kbench.txt profiles/${R}_kbench_native.txt
cp gpurun_out/kbench_net.txt profiles/${R}_kbench_net.txt
cp gpurun_out/psh_build.txt profiles/${R}_psh_build.txt
cat gpurun_out/kbench_ref_c*.txt | grep "C=" > profiles/${R}_kbench_ref.txt
cp gpurun_out/kbench_gemm.txt profiles/${R}_kbench_gemm.txt
cp gpurun_out/bench_materialized.json profiles/${R}_bench_materialized.json
