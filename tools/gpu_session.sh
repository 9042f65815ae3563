#!/usr/bin/env bash
# One gpurun session: box facts, smoke, GPU tests, bench, tuning sweep, ncu.
# usage: tools/gpu_session.sh [tag]   (outputs under gpurun_out/<tag>/)
tag=${1:-s}
out=gpurun_out/$tag
mkdir -p "$out"
{
  echo "## nproc"; nproc; echo "## mem"; free -g; echo "## lscpu"; lscpu | head -25
  echo "## numa"; for n in /sys/devices/system/node/node*/cpulist; do echo "$n: $(cat $n)"; done
  echo "## gpu"; nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv
  nvidia-smi topo -m 2>/dev/null | head -5
} > "$out/box.txt" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; echo "smoke rc=$?" >> "$out/rc.txt"
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -rf > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/rc.txt"
fi
timeout 600 python bench.py --steps 20 --warmup 5 > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/rc.txt"
if [ -n "$TUNE" ]; then
  for c in c2 c3 c1; do
    timeout 900 python bench.py --tune --steps 5 --config $c > "$out/tune_$c.jsonl" 2>&1; echo "tune $c rc=$?" >> "$out/rc.txt"
  done
fi
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file "$out/launches.csv" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > "$out/ncu_launches.log" 2>&1
  echo "ncu-launches rc=$?" >> "$out/rc.txt"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'op_triad' -s 3 -c 1 \
    -o "$out/prof_triad" python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > "$out/ncu_full.log" 2>&1
  echo "ncu-full rc=$?" >> "$out/rc.txt"
fi
if [ -n "$SWEEP" ]; then
  timeout 900 python bench.py --sweep --config c2 > "$out/sweep_c2.jsonl" 2>&1; echo "sweep rc=$?" >> "$out/rc.txt"
fi
