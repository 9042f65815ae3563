#!/usr/bin/env bash
# ncu launch lists of the C5 sweep at 16, 128 and 512 MiB per array: per-launch
# device time and DRAM bytes, caches left as the previous kernel left them
# (--cache-control none), CUDA-graph replay of 3 timed iterations per size.
out=${1:-gpurun_out/ncu_mid}
mkdir -p "$out"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_active.avg \
  --clock-control none --cache-control none --graph-profiling node -c 200 --csv \
  --log-file "$out/launches_mid.csv" python bench.py --sweep --sweep-mib 16,128,512 --sweep-iters 3 \
  > "$out/launches_mid.log" 2>&1; echo "mid rc=$?" >> "$out/rc.txt"
