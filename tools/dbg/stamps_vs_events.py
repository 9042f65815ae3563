"""Per-kernel times: events around every kernel (record 1) vs completion
stamps on a side stream (record 3), same arrays, CUDA graph."""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench
from paper_2206_06302_b200 import native as N

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 76
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
n = (mib << 20) // 8
run = bench.StreamRun(N, bench.stream_config(N, "f64", n, 0, 0))
for rnd in range(3):
    for mode in (1, 3):
        run.iterate_many(3, 0, True)
        run.sync()
        N.stream().coloc_stream_clear_records(run.h)
        run.iterate_many(iters, mode, True)
        rows = run.kernel_ms()
        per = list(zip(*rows))
        print(json.dumps({"mib": mib, "mode": mode, "round": rnd,
                          "min_us": [round(min(k) * 1e3, 2) for k in per],
                          "median_us": [round(statistics.median(k) * 1e3, 2) for k in per],
                          "max_us": [round(max(k) * 1e3, 2) for k in per]}), flush=True)
run.close()
