# full evidence pass: gpu tests, smoke, bench line, reference arm, kernel tables, launch list, ncu full capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
rm -f gpurun_out/kbench.txt; for c in 16 32 64 128 256; do timeout 300 python scripts/kbench.py $c >> gpurun_out/kbench.txt 2>&1; done; cat gpurun_out/kbench.txt
timeout 600 python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 20 > gpurun_out/bench_net64.json 2>gpurun_out/bench_net64.err; echo "net64 rc=$?"; tail -c 400 gpurun_out/bench_net64.json
timeout 600 python bench.py --workload net --res 128 --shapes-per-gpu 64 --steps 10 --no-cpu-baseline > gpurun_out/bench_net128.json 2>gpurun_out/bench_net128.err; echo "net128 rc=$?"
timeout 600 python bench.py --workload net --res 32 --shapes-per-gpu 1 --steps 20 > gpurun_out/bench_net32.json 2>gpurun_out/bench_net32.err; echo "net32 rc=$?"
timeout 600 python bench.py --workload seg --cin 32 --steps 10 > gpurun_out/bench_seg.json 2>gpurun_out/bench_seg.err; echo "seg rc=$?"; tail -c 300 gpurun_out/bench_seg.json
timeout 600 python -c "
import sys,time; sys.path.insert(0,'.')
from paper_1803_11385_b200.psh import PshLevel, VoxelSet
PshLevel.build_device(VoxelSet.sphere(16,True),0)
for res in (64, 128, 256, 512):
    s=VoxelSet.sphere(res, True); t=time.time(); g=PshLevel.build_device(s,1); print(res, s.n, 'gpu psh build %.3f s'%(time.time()-t), g.hash_dim, g.offset_dim)
" > gpurun_out/psh_build.txt 2>&1; cat gpurun_out/psh_build.txt
for c in 16 64 128; do timeout 300 python scripts/kbench_net.py $c; done > gpurun_out/kbench_net.txt 2>&1
for c in 16 64 128; do timeout 300 python scripts/kbench_gemm.py $c; done > gpurun_out/kbench_gemm.txt 2>&1
HCB_TC_GEMM=0 HCB_GEMM_MODES=fast timeout 300 python scripts/kbench_gemm.py 64 >> gpurun_out/kbench_gemm.txt 2>&1; cat gpurun_out/kbench_gemm.txt
timeout 600 python bench.py --path materialized --steps 5 > gpurun_out/bench_materialized.json 2>gpurun_out/bench_materialized.err; echo "materialized rc=$?"
for c in 16 64 256; do timeout 300 python scripts/kbench_ref.py $c > gpurun_out/kbench_ref_c$c.txt 2>&1; grep "C=" gpurun_out/kbench_ref_c$c.txt; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv|k_field_map_tiled" -s 8 -c 4 \
  -o gpurun_out/prof_round python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_round.log 2>&1; echo "ncu full rc=$?"
