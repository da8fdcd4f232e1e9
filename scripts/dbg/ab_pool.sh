# staged pooling: 128 coarse voxels per block (modes 5, 6) vs 256 (default)
for c in 16 32 64 128; do for v in 1 5 6 1 5; do echo -n "C=$c mode=$v "; HCB_POOL_STAGED=$v timeout 300 python scripts/kbench_ref.py $c 2>&1 | grep -E "C=.*(max_pool|avg_pool)" | awk '{printf "%s %s %s  ", $3, $4, $8}'; echo; done; done
