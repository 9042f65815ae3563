#!/usr/bin/env bash
# ncu --set full of one triad and one copy launch at C2, one triad at C3
# (after the warm-up iterations), for profiles/ and roofline.traffic.
out=${1:-gpurun_out/ncu_full}
mkdir -p "$out"
common="--set full --clock-control none --import-source on --kernel-name-base demangled -s 3 -c 1"
timeout 900 ncu $common -k regex:'op_triad' -o "$out/triad_c2" python bench.py --steps 2 --warmup 3 \
  --no-e2e --no-cpu-baseline --no-ceilings --no-compare > "$out/triad_c2.log" 2>&1; echo "triad c2 rc=$?" >> "$out/rc.txt"
timeout 900 ncu $common -k regex:'op_copy' -o "$out/copy_c2" python bench.py --steps 2 --warmup 3 \
  --no-e2e --no-cpu-baseline --no-ceilings --no-compare > "$out/copy_c2.log" 2>&1; echo "copy c2 rc=$?" >> "$out/rc.txt"
timeout 900 ncu $common -k regex:'op_triad' -o "$out/triad_c3" python bench.py --config c3 --steps 2 --warmup 3 \
  --no-e2e --no-cpu-baseline --no-ceilings --no-compare > "$out/triad_c3.log" 2>&1; echo "triad c3 rc=$?" >> "$out/rc.txt"
# summaries next to the reports (three reports exceed gpurun's 64 MiB return
# limit: KEEP_REPORTS=1 keeps them, otherwise only the summaries come back)
for k in triad_c2 copy_c2 triad_c3; do
  [ -f "$out/$k.ncu-rep" ] && python tools/ncu_summary.py full "$out/$k.ncu-rep" > "$out/$k.json"
done
[ -n "$KEEP_REPORTS" ] || rm -f "$out"/*.ncu-rep
