# BASELINE config 5: 512^3 sphere shells, batch sweep b = 1/2/4/8 per GPU (fused fwd+bwd, f32 and bf16),
# and the reference-layout hash2col / col2hash / pool HBM sweep over C = 16..256 (b = 1; b = 8 where the
# materialised column matrix fits in HBM). Output: gpurun_out/cfg5_*.
mkdir -p gpurun_out
for dt in f32 bf16; do
  for b in 1 2 4 8; do
    timeout 600 python bench.py --res 512 --shapes-per-gpu $b --dtype $dt --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ref-kernels \
      > gpurun_out/cfg5_${dt}_b$b.json 2> gpurun_out/cfg5_${dt}_b$b.err; echo "$dt b=$b rc=$?"
  done
done
rm -f gpurun_out/cfg5_ref_b1.txt gpurun_out/cfg5_ref_b8.txt gpurun_out/cfg5_native.txt
for c in 16 32 64 128 256; do HCB_RES=512 HCB_BATCH=1 timeout 300 python scripts/kbench_ref.py $c 2>&1 | grep "C=" >> gpurun_out/cfg5_ref_b1.txt; done
for c in 16 32 64 128; do HCB_RES=512 HCB_BATCH=8 timeout 300 python scripts/kbench_ref.py $c 2>&1 | grep "C=" >> gpurun_out/cfg5_ref_b8.txt; done
for c in 16 32 64 128 256; do HCB_RES=512 HCB_BATCH=8 timeout 300 python scripts/kbench.py $c 2>&1 | grep "C=" >> gpurun_out/cfg5_native.txt; done
cat gpurun_out/cfg5_ref_b1.txt gpurun_out/cfg5_ref_b8.txt gpurun_out/cfg5_native.txt | head -60
