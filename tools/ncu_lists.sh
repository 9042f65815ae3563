#!/usr/bin/env bash
# ncu launch lists of the bench command (per-launch device time; C1 also
# per-launch DRAM bytes, caches left as the previous kernel left them).
out=${1:-gpurun_out/ncu}
mkdir -p "$out"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
  --log-file "$out/launches_c2.csv" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-ceilings --no-compare \
  > "$out/launches_c2.log" 2>&1; echo "c2 rc=$?" >> "$out/rc.txt"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none --cache-control none -c 80 --csv \
  --log-file "$out/launches_c1.csv" python bench.py --config c1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-ceilings --no-compare \
  > "$out/launches_c1.log" 2>&1; echo "c1 rc=$?" >> "$out/rc.txt"
