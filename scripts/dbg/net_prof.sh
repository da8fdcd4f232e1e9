# per-kernel launch list of the native net step (no graph, so every launch is visible)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/net_launch_f32.csv python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 1 --warmup 3 --no-graph --no-cpu-baseline --dtype f32 > /dev/null 2>&1; echo rc=$?
