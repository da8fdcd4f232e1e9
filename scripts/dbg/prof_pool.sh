timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_pool_runs" -c 1 -o gpurun_out/poolruns python scripts/kbench_ref.py 64 > /dev/null 2>&1; echo rc=$?
