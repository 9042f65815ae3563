"""Host cost of one blocking algorithm call: drop-in vs direct C ABI vs the
native loop at tiny n (the kernel is ~nothing), avg seconds per call."""
import ctypes as C
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2206_06302_b200 import native as N

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
for rep in range(3):
    row = {"n": n, "iters": iters}
    for arm in ("dropin", "cabi", "native"):
        t = N.Timing()
        if arm == "native":
            assert N.native_baseline().stream_native_run(0, 0, n, iters, C.byref(t)) == 0
        else:
            N.check(N.stream().coloc_stream_blocking_run(0 if arm == "dropin" else 1, 0, 0, n, iters,
                                                         C.byref(t)), arm, "stream")
        row[arm] = {"avg_us": [round(x * 1e6, 2) for x in t.avg_s], "min_us": [round(x * 1e6, 2) for x in t.min_s]}
    print(json.dumps(row), flush=True)
