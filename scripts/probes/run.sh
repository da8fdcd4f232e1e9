cd scripts/probes
./ts_mma
timeout 120 ./mma_rate
