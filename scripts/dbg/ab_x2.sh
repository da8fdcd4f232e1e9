P="python scripts/dbg/x2_probe.py time 256 8 64 64"
for v in nobload nobload_nogather nogather; do echo $v; HCB_LIB_PATH=paper_1803_11385_b200/_var/$v/libhcb200.so timeout 300 $P | cut -c1-200; done
cd scripts/probes; ncu --metrics lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex.sum --clock-control none ./l1path 2>&1 | grep -E "k_ldg|lts|duration" | head -12
