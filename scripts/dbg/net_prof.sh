for dt in f32 bf16; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/net_launch_$dt.csv python bench.py --workload net --res 64 --shapes-per-gpu 32 --steps 2 --warmup 3 --no-graph --no-cpu-baseline --dtype $dt > /dev/null 2>&1; echo rc=$?
done
