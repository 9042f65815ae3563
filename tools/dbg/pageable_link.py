"""Blocking pageable copies (coloc_cuda_memcpy_async, cudaMemcpyAsync's
pageable semantics) and stream-ordered ones, 4 GiB each way, best of 3."""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
from paper_2206_06302_b200 import native as N

lib = N.cuda()
nb = 4 << 30
dev = N.DeviceBuffer(nb)
host = np.ones(nb // 8)
s = N.Stream(0)
row = {"env": {k: v for k, v in os.environ.items() if k.startswith("COLOC_STAGING")}}
for name, fn in (("h2d", lambda f: f(0, s.handle, dev.ptr, host.ctypes.data, nb)),
                 ("d2h", lambda f: f(0, s.handle, host.ctypes.data, dev.ptr, nb))):
    for mode, f in (("blocking", lib.coloc_cuda_memcpy_async), ("ordered", lib.coloc_cuda_memcpy_stream_ordered)):
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            N.check(fn(f), name)
            s.sync()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        row[f"{name}_{mode}_gbs"] = round(nb / best / 1e9, 1)
print(json.dumps(row), flush=True)
