"""e2e STREAM run from pageable (new[]) host arrays vs pinned, C2 by default."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench
from paper_2206_06302_b200 import harness as H
from paper_2206_06302_b200 import native as N

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
blocks_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,8").split(",")]
run_bytes = bench.E2E_NTIMES * 10 * n * 8
for hb in [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "2,1").split(",")]:
    for blocks in blocks_list:
        run = bench.StreamRun(N, bench.stream_config(N, "f64", n, 0, 0, host_buffers=hb, blocks=blocks))
        run.e2e_step(bench.E2E_NTIMES)
        ms = [run.e2e_step(bench.E2E_NTIMES) for _ in range(2)]
        ok = bench.validate(run, H.Dist(), n, "f64")["passed"]
        run.close()
        import os
        env = {k: v for k, v in os.environ.items() if k.startswith("COLOC_STAGING")}
        print(json.dumps({"host": "pageable" if hb == 2 else "pinned", "blocks": blocks, "env": env, "e2e_ms": ms,
                          "e2e_gbs": run_bytes / min(ms) / 1e6, "validated": ok}), flush=True)
