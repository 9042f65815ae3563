#!/usr/bin/env bash
# One gpurun session: box facts, smoke, GPU tests, bench lines, optional
# tuning sweep / size sweep / ncu captures.
# usage: [SKIP_TESTS=1] [CONFIGS=1] [ARMS=1] [TUNE=1] [AB=1] [PROBE=1] [LINK=1] [SWEEP=1]
#        [NCU=1] [COMPARE=1] [CHAIN=1] tools/gpu_session.sh <tag>
# outputs under gpurun_out/<tag>/
tag=${1:-s}
out=gpurun_out/$tag
mkdir -p "$out"
{
  echo "## nproc"; nproc; echo "## mem"; free -g; echo "## lscpu"; lscpu | head -25
  echo "## numa"; for n in /sys/devices/system/node/node*/cpulist; do echo "$n: $(cat $n)"; done
  echo "## gpu"; nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv
} > "$out/box.txt" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; echo "smoke rc=$?" >> "$out/rc.txt"
if [ -z "$SKIP_TESTS" ]; then
  COLOC_PERF_TESTS=1 timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -rf > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/rc.txt"
fi
timeout 600 python bench.py --steps 20 --warmup 5 > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/rc.txt"
if [ -n "$CONFIGS" ]; then
  for c in c1 c3; do
    timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > "$out/bench_$c.json" 2>> "$out/bench.err"
    echo "bench $c rc=$?" >> "$out/rc.txt"
  done
  timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-graph > "$out/bench_c1_nograph.json" 2>> "$out/bench.err"
  echo "bench c1 nograph rc=$?" >> "$out/rc.txt"
fi
if [ -n "$ARMS" ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > "$out/bench_torchrun1.json" 2> "$out/bench_torchrun1.err"
  echo "bench torchrun1 rc=$?" >> "$out/rc.txt"
  timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > "$out/bench_reference.json" 2> "$out/bench_reference.err"
  echo "bench reference rc=$?" >> "$out/rc.txt"
fi
if [ -n "$TUNE" ]; then
  for c in c2 c3 c1; do
    timeout 900 python bench.py --tune --steps 5 --config $c > "$out/tune_$c.jsonl" 2>&1; echo "tune $c rc=$?" >> "$out/rc.txt"
  done
fi
if [ -n "$AB" ]; then
  timeout 1200 python bench.py --tune-sizes 8192,1024,256 --tune-rounds 8 --config c2 > "$out/ab_c2.jsonl" 2>&1; echo "ab c2 rc=$?" >> "$out/rc.txt"
fi
if [ -n "$PROBE" ]; then
  for c in c2 c3 c1; do
    timeout 600 python bench.py --probe-hbm --config $c --steps 10 > "$out/probe_hbm_$c.jsonl" 2>&1; echo "probe $c rc=$?" >> "$out/rc.txt"
  done
fi
if [ -n "$LINK" ]; then
  timeout 900 python bench.py --probe-e2e > "$out/probe_e2e.jsonl" 2>&1; echo "probe e2e rc=$?" >> "$out/rc.txt"
  for c in c2 c1; do
    timeout 300 python bench.py --probe-torch --config $c --steps 10 >> "$out/probe_torch.jsonl" 2>&1
  done
  echo "probe torch rc=$?" >> "$out/rc.txt"
fi
if [ -n "$SWEEP" ]; then
  timeout 900 python bench.py --sweep --config c2 > "$out/sweep_c2.jsonl" 2>&1; echo "sweep rc=$?" >> "$out/rc.txt"
  timeout 900 python bench.py --sweep --config c2 --no-graph > "$out/sweep_c2_nograph.jsonl" 2>&1; echo "sweep nograph rc=$?" >> "$out/rc.txt"
fi
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file "$out/launches.csv" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-ceilings --no-compare > "$out/ncu_launches.log" 2>&1
  echo "ncu-launches rc=$?" >> "$out/rc.txt"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'op_triad' -s 3 -c 1 \
    -o "$out/prof_triad" python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ceilings --no-compare > "$out/ncu_full.log" 2>&1
  echo "ncu-full rc=$?" >> "$out/rc.txt"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'op_copy' -s 3 -c 1 \
    -o "$out/prof_copy" python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ceilings --no-compare > "$out/ncu_full_copy.log" 2>&1
  echo "ncu-full-copy rc=$?" >> "$out/rc.txt"
fi
if [ -n "$COMPARE" ]; then
  timeout 900 python bench.py --compare-baseline > "$out/compare_native.jsonl" 2>&1; echo "compare rc=$?" >> "$out/rc.txt"
fi
if [ -n "$CHAIN" ]; then
  timeout 1200 python bench.py --probe-chain --tune-rounds 3 --chain-shapes 512x2 > "$out/probe_chain.jsonl" 2>&1; echo "chain rc=$?" >> "$out/rc.txt"
  timeout 900 python bench.py --sweep --sweep-chain > "$out/sweep_chain.jsonl" 2>&1; echo "sweep chain rc=$?" >> "$out/rc.txt"
fi
