# per-kernel times of the reference-layout pooling calls (warm caches, serialised launches)
for u in 0 1; do HCB_UNPOOL_STAGED=$u timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"pool|unpool|switch" --csv --log-file gpurun_out/pool_launch_$u.csv python scripts/kbench_ref.py 64 > /dev/null 2>&1; echo rc=$?; done
