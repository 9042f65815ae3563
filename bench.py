#!/usr/bin/env python
"""STREAM (copy / scale / add / triad) on B200 through the coloc drop-in.

    python bench.py [--gpus N --steps K --warmup W] [--config c1|c2|c3]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...      # the reference CPU path, same metric
    python bench.py --sweep [--config c2]     # C5 size sweep (table, not the contract line)
    python bench.py --tune [--tune-tma]       # launch-shape sweeps
    python bench.py --tune-sizes 76,1024,8192 # interleaved A/B of launch variants by size
    python bench.py --probe-hbm               # read-only / write-only / launch-floor ceilings
    python bench.py --probe-e2e               # host-link ceilings, e2e pipeline depth
    python bench.py --compare-baseline        # drop-in vs C ABI vs native CUDA STREAM, 10-400 MB
    python bench.py --probe-chain             # plain / PDL / tile-chain launches, 4 timing modes

A step is one Listing-4 iteration over the resident
arrays: copy c=a, scale b=3c, add c=a+b, triad a=b+3c, each an sm_100a
kernel launched by coloc::copy / coloc::transform on the rank's target.
Every kernel is bracketed by CUDA events on its stream; per timed iteration
each kernel's time is the max over ranks; `value` is the triad's best-of-K
aggregate GB/s (STREAM convention, 3*N*8 bytes).  One process per GPU, each
owning partition_block(N*world, world)[rank]; no collective in the timed
loop ("scaling": "weak").  Arrays are 8 GiB each (64x the 133 MB L2), so
no L2 flush is needed between iterations.

Beside the contract keys the line carries `iteration` (whole Listing-4
iterations: all four kernels' bytes over their summed time; plus the
median back-to-back iteration timed by side-stream completion stamps),
`ceilings` (read-only / write-only HBM rates, the empty-kernel floor and
the per-kernel fixed cost, measured right after the timed region),
`kernels` (per-kernel best/avg) and `abstraction_vs_native` (the paper's
own claim: the drop-in vs the same kernels called directly vs a native
CUDA STREAM, blocking calls, host clock, 10-400 MB).  `e2e` runs one
STREAM run per step from pinned host buffers through the public API (see
DESIGN.md section 6).  One process per GPU: the barriers, max-over-ranks
and the validation sums go over the library's own NCCL communicator
(torch.distributed only for the rendezvous).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

from paper_2206_06302_b200 import harness as H  # noqa: E402

CONFIGS = {
    "c1": {"workload": "C1: STREAM f64, N=10,000,000 per array per GPU (STREAM default size)",
           "dtype": "f64", "n_per_gpu": 10_000_000},
    "c2": {"workload": "C2: STREAM f64, N=2^30 per array per GPU (8 GiB/array, 24 GiB)",
           "dtype": "f64", "n_per_gpu": 1 << 30},
    "c3": {"workload": "C3: STREAM f32, N=2^31 per array per GPU (8 GiB/array, float4/v8 path)",
           "dtype": "f32", "n_per_gpu": 1 << 31},
}
METRIC = "STREAM triad/copy/scale/add GB/s (device-timed, best of N) at 1/2/4/8 B200, % HBM peak"
REF_BIN = REPO / "oracle" / "_ref" / "ref_stream_cpu"
E2E_NTIMES = 10            # STREAM's default NTIMES: one e2e step = one STREAM run
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
B200_L2_BYTES = 132_644_864  # cudaDeviceProp::l2CacheSize on B200 (126.5 MiB)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------
# host / environment facts
# ----------------------------------------------------------------------------

def mem_available_bytes() -> int:
    try:
        for line in Path("/proc/meminfo").read_text().splitlines():
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 16 << 30


def hbm_peak() -> tuple[float, str]:
    p = REPO / "MEASURED_PEAKS.json"
    try:
        v = float(json.loads(p.read_text())["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs: torch copy_ of 1 Gi bf16, best of 10)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_for(config: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the
    committed ncu --set full capture (profiles/roofline_traffic.json)."""
    p = REPO / "profiles" / "roofline_traffic.json"
    try:
        return json.loads(p.read_text()).get(f"{config}:{kernel}")
    except (OSError, ValueError):
        return None


def sampled_gpus(single: bool, dev, d: H.Dist) -> str:
    """nvidia-smi -i list for rank 0's clock sampler: every GPU of the job
    on this node (one process: its GPUs; torchrun: the local ranks' GPUs)."""
    if single:
        return ",".join(str(g) for g in sorted(set(dev)))
    if d.active:
        m = os.environ.get("COLOC_DEVICE_MAP")
        local = int(os.environ.get("LOCAL_WORLD_SIZE", d.world))
        gpus = sorted({int(x) for x in m.split(",")[:local]}) if m else list(range(local))
        return ",".join(map(str, gpus))
    return str(dev)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpus = str(gpu)
        self.rows: list[tuple[float, list[str]]] = []
        self.window = (0.0, 0.0)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        t_end = time.time() + 5
        while not self.rows and time.time() < t_end:
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, start: float, end: float):
        self.window = (start, end)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        lo, hi = self.window
        inside = [r for t, r in self.rows if lo <= t <= hi + 0.06]
        note = "samples inside the timed region"
        if not inside:     # region shorter than the sampling period
            inside = [r for t, r in self.rows if lo - 0.5 <= t <= hi + 0.5] or [r for _, r in self.rows]
            note = "timed region shorter than the 50 ms sampling period: nearest samples"
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in inside if len(r) > 8 and num(r[1]) is not None]
        smax = [num(r[2]) for r in inside if len(r) > 8 and num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in inside if len(r) > 8
                          for j, v in enumerate(r[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(inside), "note": note, "gpus": self.gpus,
                "power_w_max": max((num(r[3]) or 0.0) for r in inside) if inside else None}


# ----------------------------------------------------------------------------
# reference CPU path (oracle/_ref: the unmodified reference library)
# ----------------------------------------------------------------------------

def run_reference_cpu(dtype: str, n: int, ntimes: int, warmup: int) -> dict:
    if not REF_BIN.exists():
        raise FileNotFoundError(f"{REF_BIN} missing (build on the dev box: make -C oracle ref)")
    cmd = [str(REF_BIN), "stream", "--dtype", dtype, "--n", str(n), "--ntimes", str(ntimes),
           "--warmup", str(warmup)]
    t0 = time.time()
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode not in (0,):
        raise RuntimeError(f"{' '.join(cmd)} failed ({out.returncode}): {out.stderr[-2000:]}")
    js = json.loads(out.stdout)
    js["wall_s"] = time.time() - t0
    js["cmd"] = " ".join(cmd[1:])
    return js


def reference_sample_n(dtype: str, n_wanted: int) -> int:
    """Largest n <= n_wanted whose three arrays fit in half the available RAM."""
    elem = 8 if dtype == "f64" else 4
    cap = mem_available_bytes() // 2 // (3 * elem)
    n = min(n_wanted, cap)
    return max(1 << 20, n)


def arm_config(cfg: dict, ngpu: int) -> dict:
    """The workload both arms report under `config` (identical dicts, so
    the driver's same_config check compares like with like); how each arm
    ran it goes under `setup`."""
    elem = 8 if cfg["dtype"] == "f64" else 4
    return {"workload": cfg["workload"], "dtype": cfg["dtype"], "n_per_gpu": cfg["n_per_gpu"],
            "n_total": cfg["n_per_gpu"] * ngpu, "bytes_per_array_per_gpu": cfg["n_per_gpu"] * elem,
            "ntimes_per_e2e_step": E2E_NTIMES,
            "l2": l2_regime(cfg["n_per_gpu"] * elem, B200_L2_BYTES)}


def best_window_gbs(iter_s: list[float], iter_bytes: int, window: int) -> tuple[float, float]:
    """The e2e rule on per-iteration times: best (least time) run of
    `window` consecutive Listing-4 iterations -> (GB/s, seconds)."""
    w = min(window, len(iter_s))
    best = min(sum(iter_s[i:i + w]) for i in range(len(iter_s) - w + 1))
    return w * iter_bytes / best / 1e9, best


def impl_reference(args) -> int:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    n_total = cfg["n_per_gpu"] * args.gpus
    n = reference_sample_n(cfg["dtype"], n_total)
    js = run_reference_cpu(cfg["dtype"], n, args.warmup + args.steps, args.warmup)
    k = js["kernels"]
    value = k["triad"]["best_gbs"]
    sample = (f"{cfg['dtype']} N={n} per array ({'full config' if n == n_total else f'capped from {n_total} by host RAM'}), "
              f"{args.warmup} warm-up + {args.steps} timed Listing-4 iterations, par.on(block_executor) "
              f"over {len(js['host']['numa'])} NUMA domain(s)")
    elem = 8 if cfg["dtype"] == "f64" else 4
    iter_bytes = sum(H.WORDS[x] for x in H.KERNELS) * n * elem
    timed = js["iter_time_s"][js["warmup"]:]
    e2e_gbs, e2e_s = best_window_gbs(timed, iter_bytes, E2E_NTIMES)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(k[x]["avg_time_s"] for x in H.KERNELS) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg["dtype"], "data": "synthetic (STREAM init a=1, b=2, c=0)",
        "config": arm_config(cfg, args.gpus),
        "setup": {"n_per_array": n, "path": "reference coloc CPU library, unmodified, built "
                  "from its sources (oracle/Makefile)"},
        "kernels": {x: {"best_gbs": k[x]["best_gbs"], "avg_gbs": k[x]["avg_gbs"]} for x in H.KERNELS},
        "validation": js["validation"],
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": js["host"]["pus_used"],
                         "kind": "reference", "sample": sample,
                         "numa": js["host"]["numa"], "cpu_model": js["host"]["cpu_model"],
                         "compile": js["host"]["compile"]},
        "e2e": {"value": e2e_gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "definition": f"the GPU arm's e2e rule: STREAM-rule bytes of all four kernels over "
                              f"the time of a whole run of {min(E2E_NTIMES, len(timed))} Listing-4 "
                              f"iterations (best window of the timed iterations; host memory, so no "
                              f"copies)", "best_run_s": e2e_s},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

def l2_regime(array_bytes: int, l2_bytes: int) -> str:
    """What the timed kernels measure at this array size (launch.cuh's
    auto_hint picks the cache policy by the same boundaries)."""
    mb = l2_bytes / 1e6
    if array_bytes >= 4 * l2_bytes:
        return (f"{array_bytes / 2**30:.3g} GiB arrays >> {mb:.0f} MB L2: every timed iteration "
                f"streams from HBM (no flush needed)")
    if 10 * array_bytes <= 8 * l2_bytes:
        return (f"{array_bytes / 1e6:.0f} MB arrays < {mb:.0f} MB L2: L2-assisted regime -- stores are "
                f"kept in L2 (evict-last) so each kernel reads its predecessor's output from L2; "
                f"GB/s by STREAM's byte rule, not an HBM measurement")
    return (f"{array_bytes / 1e6:.0f} MB arrays, {mb:.0f} MB L2: partly L2-resident across kernels; "
            f"GB/s by STREAM's byte rule")


def stream_config(N, dtype: str, count: int, first: int, device, *, init=0,
                  host_buffers=0, fma=0, synchronous=0, seed=0, blocks=1, chain=0):
    """Targets = `blocks` streams on each GPU in `device` (an ordinal or a
    list of them); the arrays are block-partitioned over the targets
    (partition_block), one stream per block."""
    gpus = list(device) if isinstance(device, (list, tuple)) else [device]
    ordinals = [g for g in gpus for _ in range(blocks)]
    devs = (C.c_int * len(ordinals))(*ordinals)
    cfg = N.StreamConfig(dtype=0 if dtype == "f64" else 1, init=init, fma=fma,
                         synchronous=synchronous, ntargets=len(ordinals), devices=devs, count=count,
                         first=first, seed=seed, scalar=3.0, triad_scalar=3.0,
                         host_buffers=host_buffers, chain=chain)
    cfg._devs = devs
    return cfg


class StreamRun:
    def __init__(self, N, cfg):
        self.N, self.lib = N, N.stream()
        h = C.c_void_p()
        N.check(self.lib.coloc_stream_create(C.byref(cfg), C.byref(h)), "coloc_stream_create", "stream")
        self.h = h

    def iterate(self, record: bool):
        self.N.check(self.lib.coloc_stream_iterate(self.h, int(record)), "iterate", "stream")

    def iterate_many(self, k: int, record: bool, graph: bool):
        self.N.check(self.lib.coloc_stream_iterate_many(self.h, k, int(record), int(graph)),
                     "iterate_many", "stream")

    def sync(self):
        self.N.check(self.lib.coloc_stream_sync(self.h), "sync", "stream")

    def kernel_ms(self) -> list[list[float]]:
        cnt = C.c_int()
        self.N.check(self.lib.coloc_stream_recorded(self.h, C.byref(cnt)), "recorded", "stream")
        out = []
        for i in range(cnt.value):
            ms = (C.c_double * 4)()
            self.N.check(self.lib.coloc_stream_kernel_ms(self.h, i, ms), "kernel_ms", "stream")
            out.append(list(ms))
        return out

    def err_sums(self):
        exp, sums = (C.c_double * 3)(), (C.c_double * 3)()
        self.N.check(self.lib.coloc_stream_err_sums(self.h, exp, sums, None), "err_sums", "stream")
        return list(exp), list(sums)

    def e2e_step(self, ntimes: int) -> float:
        ms = C.c_double()
        self.N.check(self.lib.coloc_stream_e2e_step(self.h, ntimes, C.byref(ms)), "e2e", "stream")
        return ms.value

    def close(self):
        if self.h:
            self.lib.coloc_stream_destroy(self.h)
            self.h = None


def validate(run: StreamRun, d: H.Dist, n_total: int, dtype: str) -> dict:
    """SPEC.md:539-547.  One process per GPU: the driver sums the per-rank
    error sums over the library's NCCL communicator (coloc_stream_set_comm);
    gloo runs (CPU tests, several ranks on one GPU) reduce on the host."""
    if d.comm is not None:
        run.N.check(run.lib.coloc_stream_set_comm(run.h, d.comm.handle), "set_comm", "stream")
        exp, sums = run.err_sums()
    else:
        exp, sums = run.err_sums()
        sums = H.all_reduce(sums, d, "sum")
    reduction = (run.lib.coloc_stream_reduction(run.h) or b"").decode()
    eps = 1e-8 if dtype == "f64" else 1e-6
    rel = [s / n_total / abs(e) if n_total else 0.0 for s, e in zip(sums, exp)]
    return {"expected": exp, "rel_err": rel, "epsilon": eps, "passed": all(r <= eps for r in rel),
            "reduction": reduction + ("" if d.comm is not None or not d.active else "+gloo")}


def gpu_arm(args) -> int:
    from paper_2206_06302_b200 import native as N
    t_start = time.time()
    d = H.init_from_env(args.dist_backend)
    cfg = CONFIGS[args.config]
    dtype, elem = cfg["dtype"], (8 if cfg["dtype"] == "f64" else 4)
    if N.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device visible (the product has no CPU path)")
    # One process per GPU under torchrun; without torchrun, --gpus G > 1 runs
    # the single-process form of C4: one vector block-partitioned over G
    # GPUs (cuda::block_allocator over G targets), per-kernel time = max over
    # the GPUs, validation sums combined by NCCL inside the driver.
    single, ngpu, dev = placement(args, d, N)
    n_total = cfg["n_per_gpu"] * ngpu
    first, count = (0, n_total) if single else H.partition_block(n_total, d.world)[d.rank]
    dev0 = dev[0] if single else dev
    info = N.device_info(dev0)

    # CPU baseline: the reference library on this host, bounded sample,
    # rank 0 at N=1 only, before any GPU work.
    cpu_baseline = None
    if ngpu == 1 and not args.no_cpu_baseline:
        try:
            n_cpu = reference_sample_n(dtype, cfg["n_per_gpu"])
            js = run_reference_cpu(dtype, n_cpu, 10, 1)
            cpu_baseline = {
                "value": js["kernels"]["triad"]["best_gbs"], "unit": "GB/s",
                "cores": js["host"]["pus_used"], "kind": "reference",
                "sample": f"{dtype} N={n_cpu} per array, NTIMES=10 (first excluded), triad best-of; "
                          f"unmodified reference coloc (par.on(block_executor) over "
                          f"{len(js['host']['numa'])} NUMA domain(s)), {js['wall_s']:.1f} s wall",
                "kernels_best_gbs": {x: js["kernels"][x]["best_gbs"] for x in H.KERNELS},
                "numa": js["host"]["numa"], "cpu_model": js["host"]["cpu_model"],
                "validation_passed": js["validation"].get("passed"),
            }
        except Exception as e:  # reported, not fatal: it is a baseline, not the product
            cpu_baseline = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference",
                            "sample": f"unavailable: {e}"}

    t_phase = time.time()
    if d.rank == 0:
        log(f"bench: cpu baseline done ({t_phase - t_start:.1f} s)")

    # ---- device-resident STREAM: the hot path ---------------------------------
    run = StreamRun(N, stream_config(N, dtype, count, first, dev))
    graph = not args.no_graph
    run.iterate_many(args.warmup, False, graph)
    run.sync()
    # W warm-up iterations, then more (untimed) until ~1 s of device work,
    # so short W never leaves the timed region on a cold GPU
    t_w = time.time()
    while time.time() - t_w < args.warmup_seconds:
        run.iterate_many(max(1, args.warmup), False, graph)
        run.sync()
    clocks = ClockSampler(sampled_gpus(single, dev, d)) if d.rank == 0 else None
    H.barrier(d)
    run.sync()
    launches0 = N.launch_count()
    t0 = time.time()
    # K Listing-4 iterations, each kernel between CUDA events; captured into
    # one CUDA graph (event-record nodes included) unless --no-graph
    run.iterate_many(args.steps, True, graph)
    run.sync()
    t1 = time.time()
    H.barrier(d)
    launches = N.launch_count() - launches0
    if clocks:
        clocks.mark(t0, t1)
    per_iter = run.kernel_ms()
    flat = H.all_reduce([x for row in per_iter for x in row], d, "max")
    per_iter = [flat[4 * i: 4 * i + 4] for i in range(len(per_iter))]
    stats = H.stream_stats(per_iter, n_total, elem)
    # after the timed region: the same K iterations back to back, timed by
    # completion stamps on a side stream (no event node between kernels);
    # per-kernel stamps jitter, so only the median iteration span is used
    b2b = back_to_back_iterations(N, run, args.steps, graph, d)
    validation = validate(run, d, n_total, dtype)
    run.close()
    clock_info = clocks.stop() if clocks else None
    launches_total = int(H.all_reduce([float(launches)], d, "sum")[0])
    if d.rank == 0:
        log(f"bench: device STREAM done ({time.time() - t_phase:.1f} s incl. construction)")
    t_phase = time.time()

    # ---- hardware ceilings next to the kernels (not timed as the metric) -----
    ceilings = None
    if ngpu == 1 and not args.no_ceilings:
        pr = hbm_probes(N, dtype, count, 5, only=("read_3arrays", "write_fill", "empty_kernel"))
        rd, wr = (pr[k][0] / (min(pr[k][1]) * 1e-3) / 1e9 for k in ("read_3arrays", "write_fill"))
        mix = 1.0 / ((2 / 3) / rd + (1 / 3) / wr)     # triad's 2:1 read:write bytes
        ceilings = {
            "read_only_gbs": rd, "write_only_gbs": wr,
            "triad_mix_gbs": mix,
            "triad_frac_of_mix": stats["triad"]["best_gbs"] / mix,
            "timed_kernel_floor_us": min(pr["empty_kernel"][1]) * 1e3,
            "how": "same tile shape and hints as the STREAM kernels: probe_read over a,b,c "
                   "(3 arrays), fill of one array, empty kernel between events; best of 5; "
                   "triad_mix = time-weighted read/write ceiling for 2 reads + 1 write per element",
            "kernel_fixed_cost": fixed_cost(N, dtype, dev0),
        }
        if d.rank == 0:
            log(f"bench: ceilings done ({time.time() - t_phase:.1f} s)")
        t_phase = time.time()

    # ---- abstraction vs native (the paper's own GPU claim) --------------------
    compare = None
    if ngpu == 1 and not args.no_compare and d.rank == 0:
        try:
            compare = compare_summary(compare_native(N, dtype, reps=5, dev=dev0))
        except Exception as e:   # reported, not fatal: a side measurement
            compare = {"unavailable": str(e)}
        log(f"bench: abstraction vs native done ({time.time() - t_phase:.1f} s)")
        t_phase = time.time()

    # ---- end to end: host buffers -> STREAM run -> host buffers ---------------
    e2e = None
    if not args.no_e2e:
        # Pinned host in+out copies of a, b, c for every rank on this node
        # must fit comfortably in host RAM; otherwise the e2e run uses the
        # largest per-rank prefix that does (reported as e2e.n_per_gpu).
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", d.world))
        fit = int(0.4 * mem_available_bytes()) // (6 * elem * max(local_world, 1))
        e_count = min(count, fit)
        if e_count < count:
            e_count -= e_count % 4096
        # pipeline depth: ~256 MiB per block and array, 8..32 blocks per GPU
        # (8 GiB arrays: 32 -> 1.53-1.61 TB/s vs 1.42-1.48 at 8; 80 MB
        # arrays: 8 -> 1.39 vs 1.14 at 32; profiles/r02_e2e_pinned_blocks.jsonl)
        if args.e2e_blocks <= 0:
            per_gpu_bytes = (e_count // (ngpu if single else 1)) * elem
            args.e2e_blocks = int(min(32, max(8, per_gpu_bytes // (256 << 20))))
        erun = StreamRun(N, stream_config(N, dtype, e_count, first, dev, host_buffers=1,
                                          blocks=args.e2e_blocks))
        erun.e2e_step(E2E_NTIMES)          # warm-up
        H.barrier(d)
        ems = [erun.e2e_step(E2E_NTIMES) for _ in range(args.e2e_steps)]
        H.barrier(d)
        ems = H.all_reduce(ems, d, "max")
        e_total = int(H.all_reduce([float(e_count)], d, "sum")[0])
        evalid = validate(erun, d, e_total, dtype)
        erun.close()
        run_bytes = E2E_NTIMES * sum(H.WORDS[k] for k in H.KERNELS) * e_total * elem
        best = min(ems)
        e2e = {
            "value": run_bytes / (best * 1e-3) / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": 3 * e_total * elem, "d2h_bytes_per_step": 3 * e_total * elem,
            "n_per_gpu": e_count // (ngpu if single else 1),
            "definition": f"one STREAM run per step through the public API: coloc::copy of a,b,c "
                          f"from pinned host buffers, {E2E_NTIMES} Listing-4 iterations, coloc::copy "
                          f"of a,b,c back; STREAM-rule bytes of all kernels / device time (events, "
                          f"max over ranks), best of {args.e2e_steps}; arrays block-partitioned over "
                          f"{args.e2e_blocks} stream target(s) per GPU with a stream-ordered executor, "
                          f"so block transfers overlap other blocks' kernels",
            "blocks_per_gpu": args.e2e_blocks,
            "ms_per_step": statistics.mean(ems), "best_ms": best,
            "validation_passed": evalid["passed"],
        }
        if d.rank == 0:
            log(f"bench: e2e done ({time.time() - t_phase:.1f} s incl. pinned host buffers)")
        t_phase = time.time()

        # the same step from a reference user's pageable arrays (new[]),
        # through the staging workers: host-DRAM bound
        if ngpu == 1 and not args.no_e2e_pageable:
            prun = StreamRun(N, stream_config(N, dtype, e_count, first, dev, host_buffers=2, blocks=4))
            prun.e2e_step(E2E_NTIMES)      # warm-up (staging rings, first touch)
            pms = min(prun.e2e_step(E2E_NTIMES) for _ in range(2))
            pvalid = validate(prun, d, e_total, dtype)
            prun.close()
            e2e["pageable"] = {
                "value": run_bytes / (pms * 1e-3) / 1e9, "unit": "GB/s", "best_ms": pms,
                "blocks_per_gpu": 4, "validation_passed": pvalid["passed"],
                "definition": "the e2e step from pageable new[] host arrays (a reference user's "
                              "std::vector): stream-ordered staging workers, best of 2",
            }
            if d.rank == 0:
                log(f"bench: pageable e2e done ({time.time() - t_phase:.1f} s)")

    H.finalize(d)
    if d.rank != 0:
        return 0
    peak, peak_src = hbm_peak()
    tri = stats["triad"]
    per_gpu = n_total // ngpu
    achieved = (3 * per_gpu * elem) / (tri["avg_ms"] * 1e-3) / 1e9  # one GPU's launch
    iter_bytes = sum(H.WORDS[k] for k in H.KERNELS) * n_total * elem
    iter_ms = [sum(r) for r in per_iter]
    line = {
        "metric": METRIC,
        "value": tri["best_gbs"], "unit": "GB/s", "n_gpus": ngpu,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(sum(r) for r in per_iter),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": dtype, "data": "synthetic (STREAM init a=1, b=2, c=0; scalar 3.0)",
        "config": arm_config(cfg, ngpu),
        "setup": {"parallelism": (f"one process, one vector block-partitioned over {ngpu} GPUs "
                                   f"(cuda::block_allocator), NCCL only for validation" if single else
                                   f"block partition over {ngpu} GPU(s), one block per rank; "
                                   f"no collective in the timed loop"),
                   "l2_bytes": info.l2_bytes,
                   "api": "coloc::copy/transform(par.on(cuda_block_executor)) on coloc::vector "
                          "over cuda::block_allocator -> libcoloc_cuda.so kernels",
                   "fma": False, "gpu": info.name.decode(),
                   "launch": "CUDA graph of the K timed iterations" if graph else "eager stream launches"},
        "kernels": {k: {"best_gbs": v["best_gbs"], "avg_gbs": v["avg_gbs"],
                        "best_frac_of_peak": v["best_gbs"] / (peak * ngpu),
                        "min_ms": v["min_ms"], "avg_ms": v["avg_ms"]} for k, v in stats.items()},
        # whole Listing-4 iterations: per-kernel times can trade L2
        # write-back work across kernel boundaries, an iteration cannot
        "iteration": {"best_gbs": iter_bytes / (min(iter_ms) * 1e-3) / 1e9,
                      "avg_gbs": iter_bytes / (statistics.mean(iter_ms) * 1e-3) / 1e9,
                      "bytes": iter_bytes,
                      "back_to_back_median_gbs": iter_bytes / (b2b * 1e-3) / 1e9,
                      "back_to_back_how": "the K iterations again after the timed region, kernels back "
                                          "to back in the graph, iteration span = consecutive triad "
                                          "completion stamps on a side stream (record mode 3), median"},
        "ceilings": ceilings,
        "frac_of_aggregate_peak": tri["best_gbs"] / (peak * ngpu),
        "frac_of_spec_8tbs": tri["best_gbs"] / (8000.0 * ngpu),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_for(args.config, "triad"),
                     "kernel": "triad (ew_pack_kernel<op_triad>)",
                     "algorithmic_bytes_per_launch": 3 * per_gpu * elem,
                     "peak_source": peak_src,
                     "achieved_from": "avg CUDA-event duration of the timed triad launches"},
        "cpu_baseline": cpu_baseline,
        "abstraction_vs_native": compare,
        "e2e": e2e,
        "gpu_launches": launches_total,
        "clocks": clock_info,
        "validation": validation,
    }
    print(json.dumps(line), flush=True)
    return 0 if validation["passed"] else 3


# ----------------------------------------------------------------------------
# extra modes: C5 sweep and launch-shape tuning (tables on stdout)
# ----------------------------------------------------------------------------

def placement(args, d: H.Dist, N) -> tuple[bool, int, object]:
    """(single-process form?, number of GPUs, device(s) of this process).
    One process per GPU under torchrun; without torchrun --gpus G > 1 runs
    one block-partitioned vector over G GPUs in this process."""
    single = not d.active and args.gpus > 1
    ngpu = args.gpus if single else d.world
    if single:
        dmap = os.environ.get("COLOC_DEVICE_MAP")    # e.g. "0,0": blocks share a GPU (tests)
        dev = [int(x) for x in dmap.split(",")][:ngpu] if dmap else list(range(ngpu))
        if len(dev) < ngpu or N.device_count() <= max(dev):
            raise SystemExit(f"bench.py: --gpus {ngpu} but only {N.device_count()} GPU(s) visible")
    else:
        dev = H.device_for(d)
    return single, ngpu, dev


def sweep(args) -> int:
    """C5: bytes per array per GPU = 2^k MiB, k = 0..14, on this process's
    GPU(s) (torchrun: one rank per GPU; --gpus G: one process over G GPUs).
    Per-kernel time per iteration = max over GPUs; aggregate GB/s."""
    from paper_2206_06302_b200 import native as N
    d = H.init_from_env(args.dist_backend)
    single, ngpu, dev = placement(args, d, N)
    dtype = CONFIGS[args.config]["dtype"]
    elem = 8 if dtype == "f64" else 4
    top = args.sweep_max_log2 if args.sweep_max_log2 >= 0 else 14
    mibs = ([int(x) for x in args.sweep_mib.split(",")] if args.sweep_mib else
            [1 << k for k in range(0, top + 1)])  # 1 MiB .. 16 GiB per array per GPU
    for mib in mibs:
        nbytes = mib << 20
        n = nbytes // elem
        n_total = n * ngpu
        first, count = (0, n_total) if single else (d.rank * n, n)
        # chains: always with --sweep-chain, else automatic (the iteration-
        # level timing below chains where it pays; per-kernel timing never)
        run = StreamRun(N, stream_config(N, dtype, count, first, dev, chain=1 if args.sweep_chain else 2))
        iters = args.sweep_iters or max(5, min(200, int(2e9 // (10 * nbytes)) + 5))
        run.iterate_many(3, False, not args.no_graph)
        run.sync()
        H.barrier(d)
        # per-kernel events, then (same arrays) events around whole iterations
        run.iterate_many(iters, 1, not args.no_graph)
        run.sync()
        H.barrier(d)
        per_iter = run.kernel_ms()
        flat = H.all_reduce([x for row in per_iter for x in row], d, "max")
        per_iter = [flat[4 * i: 4 * i + 4] for i in range(len(per_iter))]
        st = H.stream_stats(per_iter, n_total, elem)
        N.stream().coloc_stream_clear_records(run.h)
        run.iterate_many(iters, 2, not args.no_graph)
        run.sync()
        spans = []
        for i in range(iters):
            ms = C.c_double()
            N.check(N.stream().coloc_stream_iteration_ms(run.h, i, C.byref(ms)), "iteration_ms", "stream")
            spans.append(ms.value)
        spans = H.all_reduce(spans, d, "max")
        b2b = back_to_back_iterations(N, run, iters, not args.no_graph, d)
        # in-kernel spans (%globaltimer, record mode 4): kernel time without events
        N.stream().coloc_stream_clear_records(run.h)
        run.iterate_many(iters, 4, not args.no_graph)
        spn = run.kernel_ms()
        N.stream().coloc_stream_clear_records(run.h)
        flat = H.all_reduce([x for row in spn for x in row], d, "max")
        spn = [flat[4 * i: 4 * i + 4] for i in range(len(spn))]
        st_span = H.stream_stats(spn, n_total, elem)
        ok = validate(run, d, n_total, dtype)["passed"]
        run.close()
        if d.rank != 0:
            continue
        it_bytes = sum(H.WORDS[k] for k in H.KERNELS) * n_total * elem
        row = {"bytes_per_array_per_gpu": nbytes, "n_gpus": ngpu, "n_per_gpu": n, "iters": iters,
               "validated": ok, "graph": not args.no_graph,
               "chain": "always" if args.sweep_chain else "auto (iteration timing, arrays of 1-16 L2)",
               **{f"{k2}_best_gbs": v["best_gbs"] for k2, v in st.items()},
               "triad_min_us": st["triad"]["min_ms"] * 1e3,
               "iteration_best_gbs": it_bytes / (min(spans) * 1e-3) / 1e9,
               "iteration_timing": "events around whole iterations only",
               "iteration_back_to_back_median_gbs": it_bytes / (b2b * 1e-3) / 1e9,
               **{f"{k2}_span_best_gbs": v["best_gbs"] for k2, v in st_span.items()},
               "span_timing": "in-kernel %globaltimer span (earliest CTA start to latest CTA end)"}
        print(json.dumps(row), flush=True)
    H.finalize(d)
    return 0


def tune(args) -> int:
    from paper_2206_06302_b200 import native as N
    dtype = CONFIGS[args.config]["dtype"]
    elem = 8 if dtype == "f64" else 4
    n = args.tune_mib * (1 << 20) // elem if args.tune_mib else CONFIGS[args.config]["n_per_gpu"]
    run = StreamRun(N, stream_config(N, dtype, n, 0, 0))
    # (variant, threads, unroll, cache_hint, ctas_per_sm, exact_grid, chunk_bytes,
    #  stages, schedule); variant 1 = LDG/STG packs, 2 = TMA bulk; r01 sessions
    # showed exact grids beat persistent ones by ~7% (profiles/r01_tune_*)
    shapes = [(1, 0, 0, -1, 0, -1, 0, 0, 0)]                       # library default
    if args.tune_mib:    # tile size at mid sizes: (threads, unroll) only
        shapes += [(1, t, u, 1, 0, 1, 0, 0, 0) for t in (128, 256, 512, 1024) for u in (1, 2)]
    elif args.tune_tma:  # TMA pipeline space
        shapes += [(1, 1024, u, 1, 0, 1, 0, 0, 0) for u in (1, 2)]
        shapes += [(2, 0, 0, -1, c, -1, ch, st, sc)
                   for sc in (1, 2) for ch in (4096, 8192, 12288, 16384)
                   for st in (2, 4, 6, 8) for c in (0, 1, 2, 3, 4)]
    else:
        shapes += [(1, t, u, h, 0, 1, 0, 0, 0) for t in (256, 512, 1024) for u in (1, 2) for h in (0, 1, 2)]
        shapes += [(2, 0, 0, -1, c, -1, ch, 0, 0) for ch in (8192, 16384, 24576) for c in (0, 2)]
    best = None
    for shp in shapes:
        N.set_tuning(variant=shp[0], threads=shp[1], unroll=shp[2], cache_hint=shp[3],
                     ctas_per_sm=shp[4], exact_grid=shp[5], chunk_bytes=shp[6],
                     stages=shp[7], schedule=shp[8])
        run.iterate_many(2, False, not args.no_graph)
        run.sync()
        run.iterate_many(args.steps, True, not args.no_graph)
        st = H.stream_stats(run.kernel_ms(), n, elem)
        N.stream().coloc_stream_clear_records(run.h)
        row = {"variant": shp[0], "threads": shp[1], "unroll": shp[2], "hint": shp[3],
               "ctas_per_sm": shp[4], "exact": shp[5], "chunk": shp[6], "stages": shp[7],
               "schedule": shp[8], **{k: round(v["best_gbs"], 1) for k, v in st.items()}}
        print(json.dumps(row), flush=True)
        if best is None or row["triad"] > best["triad"]:
            best = row
    N.cuda().coloc_cuda_set_tuning(None)
    print(json.dumps({"best": best}), flush=True)
    run.close()
    return 0


# launch variants compared by --tune-sizes (names are what the rows report)
TUNE_AB = (("auto", {}),
           *((f"ldg_{t}x{u}", {"variant": 1, "threads": t, "unroll": u})
             for (t, u) in ((256, 1), (512, 2), (1024, 1), (1024, 2))),
           ("ldg_h0", {"variant": 1, "cache_hint": 0}), ("ldg_h4", {"variant": 1, "cache_hint": 4}))


def step_gbs(gbs: dict) -> float:
    """Whole Listing-4 iteration rate from per-kernel rates: STREAM bytes of
    the four kernels over the sum of their times.  Per-kernel rates can
    shift L2 write-back work across kernel boundaries; the step cannot."""
    return sum(H.WORDS[k] for k in H.KERNELS) / sum(H.WORDS[k] / gbs[k] for k in H.KERNELS)


def tune_sizes(args) -> int:
    """Library default vs forced LDG/STG vs TMA shapes, interleaved A/B
    rounds at several sizes (per-round best of `iters`; median over rounds
    is the number to compare -- run-to-run noise at 8 GiB is ~1%)."""
    from paper_2206_06302_b200 import native as N
    dtype = CONFIGS[args.config]["dtype"]
    elem = 8 if dtype == "f64" else 4
    # entries: MiB per array, or nN for N elements per array (n10000000 = C1)
    sizes = [int(x[1:]) * elem if x.startswith("n") else int(x) << 20
             for x in args.tune_sizes.split(",")]
    rounds = args.tune_rounds
    for nbytes in sizes:
        n = nbytes // elem
        run = StreamRun(N, stream_config(N, dtype, n, 0, 0))
        iters = max(5, min(100, int(4e9 // (10 * nbytes)) + 5))
        res = {name: {k: [] for k in H.KERNELS} for name, _ in TUNE_AB}
        for _ in range(rounds):
            for name, kw in TUNE_AB:
                N.set_tuning(**kw)
                run.iterate_many(2, False, not args.no_graph)
                run.sync()
                run.iterate_many(iters, True, not args.no_graph)
                st = H.stream_stats(run.kernel_ms(), n, elem)
                N.stream().coloc_stream_clear_records(run.h)
                for k in H.KERNELS:
                    res[name][k].append(st[k]["best_gbs"])
        N.cuda().coloc_cuda_set_tuning(None)
        run.close()
        for name, _ in TUNE_AB:
            print(json.dumps({"bytes_per_array": nbytes, "shape": name, "rounds": rounds,
                              "iters": iters,
                              **{k: round(statistics.median(v), 1) for k, v in res[name].items()},
                              "step": round(step_gbs({k: statistics.median(v) for k, v in res[name].items()}), 1),
                              "max": {k: round(max(v), 1) for k, v in res[name].items()}}),
                  flush=True)
    return 0


def hbm_probes(N, dtype: str, n: int, rounds: int, only=None, offset: int = 0) -> dict:
    """Hardware-side bounds for the STREAM kernels at n elements per array:
    read-only (probe_read over 1 and 3 arrays), write-only (fill), the four
    STREAM kernels and the launch floor (an empty kernel between events).
    Ops are interleaved round by round on one stream, each between its own
    CUDA events; returns {op: (bytes, [ms per round])}."""
    elem = 8 if dtype == "f64" else 4
    nb = n * elem
    lib = N.cuda()
    # `offset` staggers the arrays (b at +nb+offset, c at +2nb+2*offset):
    # STREAM's OFFSET knob, to see whether same-index elements of the
    # three arrays collide in the DRAM channels/banks
    buf = N.DeviceBuffer(3 * nb + 2 * offset + 64)
    a, b, c = buf.ptr, buf.ptr + nb + offset, buf.ptr + 2 * nb + 2 * offset
    sink = buf.ptr + 3 * nb + 2 * offset
    st = N.Stream(0)
    s = st.handle
    fill = getattr(lib, f"coloc_cuda_fill_{dtype}")
    for p, v in ((a, 1.0), (b, 2.0), (c, 0.0)):
        N.check(fill(0, s, p, n, v))
    ops = {
        "read_1array": (nb, lambda: lib.coloc_cuda_probe_read(0, s, a, nb, sink)),
        "read_3arrays": (3 * nb, lambda: lib.coloc_cuda_probe_read(0, s, a, 3 * nb, sink)),
        "write_fill": (nb, lambda: fill(0, s, a, n, 1.0)),
        "copy": (2 * nb, lambda: getattr(lib, f"coloc_cuda_copy_{dtype}")(0, s, c, a, n)),
        "scale": (2 * nb, lambda: getattr(lib, f"coloc_cuda_scale_{dtype}")(0, s, b, c, 3.0, n)),
        "add": (3 * nb, lambda: getattr(lib, f"coloc_cuda_add_{dtype}")(0, s, c, a, b, n)),
        "triad": (3 * nb, lambda: getattr(lib, f"coloc_cuda_triad_{dtype}")(0, s, a, b, c, 3.0, n, 0)),
        "empty_kernel": (0, lambda: lib.coloc_cuda_probe_empty(0, s)),
    }
    if only:
        ops = {k: v for k, v in ops.items() if k in only}
    evs = []
    for _ in range(2 * len(ops)):
        e = C.c_void_p()
        N.check(lib.coloc_cuda_event_create(0, C.byref(e)))
        evs.append(e)
    times = {k: [] for k in ops}
    try:
        for r in range(rounds + 2):
            for i, (k, (_, fn)) in enumerate(ops.items()):
                N.check(lib.coloc_cuda_event_record(0, evs[2 * i], s))
                N.check(fn(), k)
                N.check(lib.coloc_cuda_event_record(0, evs[2 * i + 1], s))
            st.sync()
            if r < 2:
                continue                       # warm-up rounds
            for i, k in enumerate(ops):
                ms = C.c_float()
                N.check(lib.coloc_cuda_event_elapsed_ms(evs[2 * i], evs[2 * i + 1], C.byref(ms)))
                times[k].append(ms.value)
    finally:
        for e in evs:
            lib.coloc_cuda_event_destroy(0, e)
        st.close()
        buf.close()
    return {k: (ops[k][0], times[k]) for k in ops}


def probe_torch(args) -> int:
    """The same four STREAM operations as PyTorch's own CUDA kernels (copy_,
    mul, add, add with alpha) on the config's arrays, CUDA-event timed on
    torch's stream, best of --steps: the vendor-library baseline next to
    the hand-written kernels.  Timing only (torch's triad may contract)."""
    import torch
    cfg = CONFIGS[args.config]
    dt = torch.float64 if cfg["dtype"] == "f64" else torch.float32
    n = cfg["n_per_gpu"]
    elem = 8 if cfg["dtype"] == "f64" else 4
    a = torch.full((n,), 1.0, dtype=dt, device="cuda")
    b = torch.full((n,), 2.0, dtype=dt, device="cuda")
    c = torch.zeros(n, dtype=dt, device="cuda")
    ops = {"copy": (2, lambda: c.copy_(a)), "scale": (2, lambda: torch.mul(c, 3.0, out=b)),
           "add": (3, lambda: torch.add(a, b, out=c)), "triad": (3, lambda: torch.add(b, c, alpha=3.0, out=a))}
    ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps + 2)] for k in ops}
    for it in range(args.steps + 2):
        for k, (_, fn) in ops.items():
            ev[k][it][0].record()
            fn()
            ev[k][it][1].record()
    torch.cuda.synchronize()
    row = {"probe": "torch", "config": args.config, "torch": torch.__version__}
    for k, (words, _) in ops.items():
        t = min(s.elapsed_time(e) for s, e in ev[k][2:])
        row[f"{k}_best_gbs"] = words * n * elem / (t * 1e-3) / 1e9
    print(json.dumps(row), flush=True)
    return 0


COMPARE_SIZES_MB = (10, 20, 40, 100, 200, 400)   # PAPER.md Fig. 5: "from 10 to 400 MB"


def back_to_back_iterations(N, run, k: int, graph: bool, d: H.Dist) -> float:
    """Median Listing-4 iteration span (ms, max over ranks) of k iterations
    timed by completion stamps on side streams (record mode 3)."""
    lib = N.stream()
    lib.coloc_stream_clear_records(run.h)
    run.iterate_many(k, 3, graph)
    run.sync()
    spans = []
    for i in range(k):
        ms = C.c_double()
        N.check(lib.coloc_stream_iteration_ms(run.h, i, C.byref(ms)), "iteration_ms", "stream")
        spans.append(ms.value)
    lib.coloc_stream_clear_records(run.h)
    spans = H.all_reduce(spans, d, "max")
    return statistics.median(spans)


def fixed_cost(N, dtype: str, dev: int, mib: int = 1, iters: int = 50) -> dict:
    """The per-kernel fixed cost at a size where the bytes are negligible
    (1 MiB arrays, L2-resident): the best Listing-4 iteration in a CUDA
    graph divided by its four kernels, timed with events around whole
    iterations only, and with events around every kernel (the bench's
    per-kernel rule) -- the difference is the cost of the event nodes."""
    elem = 8 if dtype == "f64" else 4
    n = (mib << 20) // elem
    run = StreamRun(N, stream_config(N, dtype, n, 0, dev))
    lib = N.stream()
    out = {"mib_per_array": mib, "iters": iters}
    try:
        for mode, key in ((2, "in_graph_us"), (1, "with_events_us")):
            run.iterate_many(3, False, True)
            run.sync()
            lib.coloc_stream_clear_records(run.h)
            run.iterate_many(iters, mode, True)
            best = None
            for i in range(iters):
                ms = C.c_double()
                N.check(lib.coloc_stream_iteration_ms(run.h, i, C.byref(ms)), "iteration_ms", "stream")
                best = ms.value if best is None else min(best, ms.value)
            out[key] = best * 1e3 / 4
            lib.coloc_stream_clear_records(run.h)
    finally:
        run.close()
    return out


def compare_native(N, dtype: str, sizes_mb=COMPARE_SIZES_MB, reps: int = 3, iterations: int = 10,
                   dev: int = 0) -> list[dict]:
    """Abstraction vs native (SPEC.md:549-567 run_baseline,
    size_sweep): at each size the three arms run `iterations` Listing-4
    iterations with the reference's blocking semantics, every kernel call
    timed by the host's steady clock (first iteration excluded):
      dropin  coloc::copy/transform(par.on(cuda_block_executor{synchronous}))
      cabi    coloc_cuda_<op> + coloc_cuda_stream_sync
      native  the hand-written CUDA STREAM (libstream_native.so)
    Arms interleave within each of `reps` rounds; rows carry medians."""
    lib, nat = N.stream(), N.native_baseline()
    dt = 0 if dtype == "f64" else 1
    elem = 8 if dtype == "f64" else 4
    rows = []
    for mb in sizes_mb:
        n = int(mb * 1e6) // elem
        per = {a: {k: [] for k in H.KERNELS} for a in ("dropin", "cabi", "native")}
        ok = True
        for _ in range(reps):
            for arm in ("dropin", "cabi", "native"):
                t = N.Timing()
                if arm == "native":
                    st = nat.stream_native_run(dt, dev, n, iterations, C.byref(t))
                    if st:
                        raise RuntimeError(f"stream_native_run: {nat.stream_native_last_error().decode()}")
                else:
                    N.check(lib.coloc_stream_blocking_run(0 if arm == "dropin" else 1, dt, dev, n,
                                                          iterations, C.byref(t)), "blocking_run", "stream")
                ok = ok and bool(t.validated)
                for j, k in enumerate(H.KERNELS):
                    per[arm][k].append(H.WORDS[k] * n * elem / t.avg_s[j] / 1e9)
        med = {a: {k: statistics.median(v) for k, v in d.items()} for a, d in per.items()}
        suite = {a: statistics.mean(m.values()) for a, m in med.items()}
        rows.append({
            "mb_per_array": mb, "n": n, "reps": reps, "iterations": iterations, "validated": ok,
            "avg_gbs": {a: {k: round(v, 1) for k, v in m.items()} for a, m in med.items()},
            "suite_avg_gbs": {a: round(v, 1) for a, v in suite.items()},
            "ratio_dropin_vs_native": {k: med["dropin"][k] / med["native"][k] for k in H.KERNELS},
            "ratio_cabi_vs_native": {k: med["cabi"][k] / med["native"][k] for k in H.KERNELS},
            "ratio_dropin_vs_cabi": {k: med["dropin"][k] / med["cabi"][k] for k in H.KERNELS},
            "suite_ratio_dropin_vs_native": suite["dropin"] / suite["native"],
            "suite_ratio_dropin_vs_cabi": suite["dropin"] / suite["cabi"],
        })
    return rows


def compare_summary(rows: list[dict]) -> dict:
    """The paper's claims in numbers: parity at 100 MB (SPEC criterion 2,
    >= 0.95 per kernel) and convergence (criterion 3: ratio at the largest
    size >= ratio at the smallest)."""
    by = {r["mb_per_array"]: r for r in rows}
    at100 = by.get(100) or rows[len(rows) // 2]
    lo, hi = rows[0], rows[-1]
    return {
        "timing": "host steady clock around each blocking call (reference semantics), first "
                  "iteration excluded, avg bandwidth, median of reps",
        "sizes_mb": [r["mb_per_array"] for r in rows],
        "at_mb": at100["mb_per_array"],
        "dropin_vs_native": {k: round(v, 4) for k, v in at100["ratio_dropin_vs_native"].items()},
        "dropin_vs_cabi": {k: round(v, 4) for k, v in at100["ratio_dropin_vs_cabi"].items()},
        "parity_ge_0_95": all(v >= 0.95 for v in at100["ratio_dropin_vs_native"].values()),
        "suite_ratio_by_size": {r["mb_per_array"]: round(r["suite_ratio_dropin_vs_native"], 4)
                                for r in rows},
        "suite_ratio_dropin_vs_cabi_by_size": {r["mb_per_array"]: round(r["suite_ratio_dropin_vs_cabi"], 4)
                                               for r in rows},
        "converges": hi["suite_ratio_dropin_vs_native"] >= lo["suite_ratio_dropin_vs_native"],
        "validated": all(r["validated"] for r in rows),
    }


def compare_baseline(args) -> int:
    from paper_2206_06302_b200 import native as N
    dtype = CONFIGS[args.config]["dtype"]
    sizes = [float(x) for x in args.compare_sizes.split(",")] if args.compare_sizes else COMPARE_SIZES_MB
    sizes = [int(x) if float(x).is_integer() else x for x in sizes]
    rows = compare_native(N, dtype, sizes, reps=args.compare_reps)
    for r in rows:
        print(json.dumps(r), flush=True)
    print(json.dumps({"summary": compare_summary(rows)}), flush=True)
    return 0


def probe_chain(args) -> int:
    """Fixed per-kernel cost and the launch chain: at
    each size, K Listing-4 iterations in one CUDA graph per target, timed
    with events around every kernel (the bench's per-kernel rule) or around
    whole iterations only, for: plain launches, programmatic dependent
    launch (PDL), and tile chains (kernels hand over tile by tile,
    coloc_cuda_chain_begin/end); rounds interleaved.  Rows report the
    whole-iteration rate (all four kernels' STREAM bytes / span)."""
    from paper_2206_06302_b200 import native as N
    cfg = CONFIGS[args.config]
    dtype, elem = cfg["dtype"], (8 if cfg["dtype"] == "f64" else 4)
    sizes = [int(x) for x in (args.chain_sizes or "1,4,16,32,64,128,256,512,1024,8192").split(",")]
    lib = N.stream()
    # (name, pdl, chain, timing mode, (threads, unroll) or None = automatic)
    variants = [("plain", 0, 0, 1, None), ("plain", 0, 0, 3, None), ("plain", 0, 0, 4, None),
                ("plain", 0, 0, 2, None),
                ("pdl", 1, 0, 2, None), ("chain", 0, 1, 2, None), ("chain", 0, 1, 1, None)]
    for shp in filter(None, args.chain_shapes.split(",")):
        t, u = (int(x) for x in shp.split("x"))
        variants.append((f"chain_{t}x{u}", 0, 1, 2, (t, u)))
    for mib in sizes:
        nbytes = mib << 20
        n = nbytes // elem
        runs = {c: StreamRun(N, stream_config(N, dtype, n, 0, 0, chain=c)) for c in (0, 1)}
        iters = max(5, min(200, int(2e9 // (10 * nbytes)) + 5))
        res = {}
        for _ in range(args.tune_rounds):
            for name, pdl, chain, mode, shape in variants:
                run = runs[chain]
                if shape:
                    N.set_tuning(pdl=pdl, threads=shape[0], unroll=shape[1])
                else:
                    N.set_tuning(pdl=pdl)
                run.iterate_many(2, False, True)
                run.sync()
                lib.coloc_stream_clear_records(run.h)
                run.iterate_many(iters, mode, True)
                cnt = C.c_int()
                N.check(lib.coloc_stream_recorded(run.h, C.byref(cnt)))
                spans = []
                for i in range(cnt.value):
                    ms = C.c_double()
                    N.check(lib.coloc_stream_iteration_ms(run.h, i, C.byref(ms)), "iteration_ms", "stream")
                    spans.append(ms.value)
                r = res.setdefault((name, mode), {"span_ms": [], "kernel_sum_ms": []})
                r["span_ms"].append(min(spans))
                if mode in (1, 3, 4):
                    r["kernel_sum_ms"].append(min(sum(row) for row in run.kernel_ms()))
                lib.coloc_stream_clear_records(run.h)
        N.cuda().coloc_cuda_set_tuning(None)
        ok = all(validate(r, H.Dist(), n, dtype)["passed"] for r in runs.values())
        for r in runs.values():
            r.close()
        it_bytes = sum(H.WORDS[k] for k in H.KERNELS) * n * elem
        for (name, mode), r in res.items():
            span = statistics.median(r["span_ms"])
            row = {"probe": "chain", "mib_per_array": mib, "launch": name,
                   "timing": {1: "events per kernel", 2: "events per iteration",
                              3: "completion stamps per kernel (side stream)",
                              4: "in-kernel spans (globaltimer)"}[mode],
                   "iters": iters, "rounds": args.tune_rounds, "validated": ok,
                   "span_us": span * 1e3, "iteration_gbs": it_bytes / (span * 1e-3) / 1e9}
            if r["kernel_sum_ms"]:
                ks = statistics.median(r["kernel_sum_ms"])
                row.update(kernel_sum_us=ks * 1e3, kernel_sum_gbs=it_bytes / (ks * 1e-3) / 1e9)
            print(json.dumps(row), flush=True)
    return 0


def probe_hbm(args) -> int:
    from paper_2206_06302_b200 import native as N
    cfg = CONFIGS[args.config]
    peak, _ = hbm_peak()
    # --probe-spacer-gib: allocate (and hold) this much device memory first,
    # so the arrays land on other physical pages (placement sensitivity)
    spacer = N.DeviceBuffer(args.probe_spacer_gib << 30) if args.probe_spacer_gib else None
    res = hbm_probes(N, cfg["dtype"], cfg["n_per_gpu"], args.steps, offset=args.probe_offset)
    if spacer:
        spacer.close()
    for k, (byts, t) in res.items():
        row = {"probe": k, "config": args.config, "offset": args.probe_offset,
               "spacer_gib": args.probe_spacer_gib, "bytes": byts,
               "min_us": min(t) * 1e3,
               "median_us": statistics.median(t) * 1e3}
        if byts:
            row.update(best_gbs=byts / (min(t) * 1e-3) / 1e9,
                       median_gbs=byts / (statistics.median(t) * 1e-3) / 1e9,
                       frac_of_measured_peak=byts / (min(t) * 1e-3) / 1e9 / peak)
        print(json.dumps(row), flush=True)
    return 0


def probe_e2e(args) -> int:
    """Host-link ceilings (pinned H2D, D2H, both at once) and the e2e STREAM
    run at several block counts per GPU (the copy/compute pipeline depth)."""
    from paper_2206_06302_b200 import native as N
    cfg = CONFIGS[args.config]
    elem = 8 if cfg["dtype"] == "f64" else 4
    n = cfg["n_per_gpu"]
    nbytes = 3 * n * elem
    lib = N.cuda()
    host, dev = C.c_void_p(), N.DeviceBuffer(nbytes)
    N.check(lib.coloc_cuda_host_alloc(nbytes, C.byref(host)), "host_alloc")
    s1, s2 = N.Stream(0), N.Stream(0)
    ev = [C.c_void_p() for _ in range(4)]
    for e in ev:
        N.check(lib.coloc_cuda_event_create(0, C.byref(e)))

    def timed(fn) -> float:
        N.check(lib.coloc_cuda_event_record(0, ev[0], s1.handle))
        N.check(lib.coloc_cuda_stream_wait_event(0, s2.handle, ev[0]))
        fn()
        N.check(lib.coloc_cuda_event_record(0, ev[1], s1.handle))
        N.check(lib.coloc_cuda_event_record(0, ev[2], s2.handle))
        s1.sync()
        s2.sync()
        a, b = C.c_float(), C.c_float()
        N.check(lib.coloc_cuda_event_elapsed_ms(ev[0], ev[1], C.byref(a)))
        N.check(lib.coloc_cuda_event_elapsed_ms(ev[0], ev[2], C.byref(b)))
        return max(a.value, b.value)

    half = nbytes // 2
    h2d = timed(lambda: N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, dev.ptr, host.value, nbytes)))
    d2h = timed(lambda: N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, host.value, dev.ptr, nbytes)))
    both = timed(lambda: (N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, dev.ptr, host.value, half)),
                          N.check(lib.coloc_cuda_memcpy_async(0, s2.handle, host.value + half,
                                                              dev.ptr + half, half))))
    print(json.dumps({"bytes": nbytes, "h2d_gbs": nbytes / h2d / 1e6, "d2h_gbs": nbytes / d2h / 1e6,
                      "bidir_total_gbs": nbytes / both / 1e6}), flush=True)
    # one direction split over two streams (two copy engines)
    h2d2 = timed(lambda: (N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, dev.ptr, host.value, half)),
                          N.check(lib.coloc_cuda_memcpy_async(0, s2.handle, dev.ptr + half,
                                                              host.value + half, half))))
    d2h2 = timed(lambda: (N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, host.value, dev.ptr, half)),
                          N.check(lib.coloc_cuda_memcpy_async(0, s2.handle, host.value + half,
                                                              dev.ptr + half, half))))
    print(json.dumps({"bytes": nbytes, "h2d_2streams_gbs": nbytes / h2d2 / 1e6,
                      "d2h_2streams_gbs": nbytes / d2h2 / 1e6}), flush=True)
    # the same transfers driven by SMs (the copy kernel dereferencing the
    # pinned host buffer through UVA) instead of the copy engines
    cp = lib.coloc_cuda_copy_bytes
    k_h2d = timed(lambda: N.check(cp(0, s1.handle, dev.ptr, host.value, nbytes)))
    k_d2h = timed(lambda: N.check(cp(0, s1.handle, host.value, dev.ptr, nbytes)))
    k_both = timed(lambda: (N.check(cp(0, s1.handle, dev.ptr, host.value, half)),
                            N.check(cp(0, s2.handle, host.value + half, dev.ptr + half, half))))
    mixed = timed(lambda: (N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, dev.ptr, host.value, half)),
                           N.check(cp(0, s2.handle, host.value + half, dev.ptr + half, half))))
    split_d2h = timed(lambda: (N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, host.value, dev.ptr, half)),
                               N.check(cp(0, s2.handle, host.value + half, dev.ptr + half, half))))
    split_h2d = timed(lambda: (N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, dev.ptr, host.value, half)),
                               N.check(cp(0, s2.handle, dev.ptr + half, host.value + half, half))))
    print(json.dumps({"bytes": nbytes, "ce_plus_kernel_d2h_gbs": nbytes / split_d2h / 1e6,
                      "ce_plus_kernel_h2d_gbs": nbytes / split_h2d / 1e6}), flush=True)
    print(json.dumps({"bytes": nbytes, "kernel_h2d_gbs": nbytes / k_h2d / 1e6,
                      "kernel_d2h_gbs": nbytes / k_d2h / 1e6,
                      "kernel_bidir_total_gbs": nbytes / k_both / 1e6,
                      "ce_h2d_plus_kernel_d2h_total_gbs": nbytes / mixed / 1e6}), flush=True)
    # pageable host memory (numpy), through the library's pinned staging
    # ring (copies >= 4 MiB); wall time around call + stream sync
    import numpy as np
    pb = min(nbytes, 4 << 30)
    pg = np.ones(pb // 8)
    rows = {}
    for name, fn in (("pageable_h2d_gbs", lambda: lib.coloc_cuda_memcpy_async(0, s1.handle, dev.ptr,
                                                                               pg.ctypes.data, pb)),
                     ("pageable_d2h_gbs", lambda: lib.coloc_cuda_memcpy_async(0, s1.handle, pg.ctypes.data,
                                                                               dev.ptr, pb))):
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            N.check(fn(), name)
            s1.sync()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        rows[name] = pb / best / 1e9
    print(json.dumps({"bytes": pb, **rows, "how": "coloc_cuda_memcpy_async from/to a numpy array "
                      "(pinned staging ring), wall time incl. stream sync, best of 3"}), flush=True)
    del pg
    # pinned memory from THP-backed anonymous pages (mmap + MADV_HUGEPAGE +
    # cudaHostRegister) instead of cudaHostAlloc: fewer IOMMU translations
    try:
        import mmap
        thp = Path("/sys/kernel/mm/transparent_hugepage/enabled").read_text().strip()
    except OSError:
        thp = "unknown"
    try:
        mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        mm.madvise(mmap.MADV_HUGEPAGE)
        base = C.addressof(C.c_char.from_buffer(mm))
        C.memset(base, 0, nbytes)
        N.check(lib.coloc_cuda_host_register(C.c_void_p(base), nbytes), "host_register")
        t_h2d = timed(lambda: N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, dev.ptr, base, nbytes)))
        t_d2h = timed(lambda: N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, base, dev.ptr, nbytes)))
        t_both = timed(lambda: (N.check(lib.coloc_cuda_memcpy_async(0, s1.handle, dev.ptr, base, half)),
                                N.check(lib.coloc_cuda_memcpy_async(0, s2.handle, base + half,
                                                                    dev.ptr + half, half))))
        huge = next((l for l in Path("/proc/meminfo").read_text().splitlines()
                     if l.startswith("AnonHugePages")), "")
        print(json.dumps({"bytes": nbytes, "thp": thp, "anon_huge": huge,
                          "thp_registered_h2d_gbs": nbytes / t_h2d / 1e6,
                          "thp_registered_d2h_gbs": nbytes / t_d2h / 1e6,
                          "thp_registered_bidir_total_gbs": nbytes / t_both / 1e6}), flush=True)
        lib.coloc_cuda_host_unregister(C.c_void_p(base))
    except Exception as e:    # measurement only
        print(json.dumps({"thp": thp, "thp_registered": f"failed: {e}"}), flush=True)
    if args.probe_link_only:
        lib.coloc_cuda_host_free(host)
        dev.close()
        return 0
    lib.coloc_cuda_host_free(host)
    dev.close()
    run_bytes = E2E_NTIMES * sum(H.WORDS[k] for k in H.KERNELS) * n * elem
    # a reference user's pageable arrays (host_buffers=2): staged copies
    for blocks in (1, 8):
        run = StreamRun(N, stream_config(N, cfg["dtype"], n, 0, 0, host_buffers=2, blocks=blocks))
        run.e2e_step(E2E_NTIMES)
        ms = min(run.e2e_step(E2E_NTIMES) for _ in range(2))
        ok = validate(run, H.Dist(), n, cfg["dtype"])["passed"]
        run.close()
        print(json.dumps({"host": "pageable", "blocks": blocks, "e2e_ms": ms,
                          "e2e_gbs": run_bytes / ms / 1e6, "validated": ok}), flush=True)
    for blocks in (1, 4, 8, 16, 32, 64):
        run = StreamRun(N, stream_config(N, cfg["dtype"], n, 0, 0, host_buffers=1, blocks=blocks))
        run.e2e_step(E2E_NTIMES)
        ms = min(run.e2e_step(E2E_NTIMES) for _ in range(2))
        ok = validate(run, H.Dist(), n, cfg["dtype"])["passed"]
        run.close()
        print(json.dumps({"blocks": blocks, "e2e_ms": ms, "e2e_gbs": run_bytes / ms / 1e6,
                          "validated": ok}), flush=True)
    return 0


def main() -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["coloc", "reference"], default="coloc")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--warmup-seconds", type=float, default=1.0,
                    help="after the W warm-up iterations, keep warming (untimed) for this long")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-blocks", type=int, default=0,
                    help="stream targets per GPU for the e2e arrays (copy/compute pipeline); "
                         "0 = ~256 MiB per block, 8..32")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-e2e-pageable", action="store_true",
                    help="skip the e2e step from pageable host arrays (e2e.pageable)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ceilings", action="store_true", help="skip the read/write ceiling probes")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--sweep-max-log2", type=int, default=-1,
                    help="--sweep: largest size 2^k MiB per array per GPU (default 14 = 16 GiB)")
    ap.add_argument("--sweep-mib", default="", help="--sweep: these MiB per array instead of 2^k")
    ap.add_argument("--sweep-iters", type=int, default=0, help="--sweep: timed iterations per size")
    ap.add_argument("--sweep-chain", action="store_true",
                    help="--sweep: kernels hand over tile by tile (cfg.chain)")
    ap.add_argument("--tune", action="store_true")
    ap.add_argument("--tune-mib", type=int, default=0, help="--tune at this many MiB per array")
    ap.add_argument("--tune-tma", action="store_true", help="--tune over the TMA pipeline space")
    ap.add_argument("--tune-rounds", type=int, default=5)
    ap.add_argument("--tune-sizes", default="",
                    help="comma-separated MiB per array: interleaved A/B of launch variants")
    ap.add_argument("--probe-e2e", action="store_true", help="host-link ceilings and e2e pipeline depth")
    ap.add_argument("--probe-link-only", action="store_true", help="--probe-e2e: host-link rows only")
    ap.add_argument("--probe-spacer-gib", type=int, default=0,
                    help="--probe-hbm: device memory held before the arrays are allocated")
    ap.add_argument("--probe-offset", type=int, default=0,
                    help="--probe-hbm: bytes between the arrays (STREAM's OFFSET)")
    ap.add_argument("--probe-torch", action="store_true",
                    help="the four STREAM ops as PyTorch CUDA kernels (vendor baseline)")
    ap.add_argument("--compare-baseline", action="store_true",
                    help="drop-in vs direct C ABI vs native CUDA STREAM, blocking calls, host clock")
    ap.add_argument("--compare-sizes", default="", help="--compare-baseline: MB per array")
    ap.add_argument("--compare-reps", type=int, default=3)
    ap.add_argument("--no-compare", action="store_true",
                    help="skip the abstraction-vs-native table in the bench line")
    ap.add_argument("--probe-chain", action="store_true",
                    help="per-kernel vs per-iteration timing, PDL off/on, over array sizes")
    ap.add_argument("--chain-sizes", default="", help="--probe-chain: MiB per array, comma-separated")
    ap.add_argument("--chain-shapes", default="",
                    help="--probe-chain: extra chained tile shapes, e.g. 256x2,512x2")
    ap.add_argument("--probe-hbm", action="store_true",
                    help="read-only / write-only / launch-floor bounds next to the STREAM kernels")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="torch.distributed backend for the plumbing (gloo: tests on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3 and not (args.sweep or args.tune or args.tune_sizes or args.probe_chain
                                or args.compare_baseline):
        log("bench.py: raising --warmup to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        return impl_reference(args)
    if args.sweep:
        return sweep(args)
    if args.tune_sizes:
        return tune_sizes(args)
    if args.tune:
        return tune(args)
    if args.probe_e2e:
        return probe_e2e(args)
    if args.probe_hbm:
        return probe_hbm(args)
    if args.probe_chain:
        return probe_chain(args)
    if args.compare_baseline:
        return compare_baseline(args)
    if args.probe_torch:
        return probe_torch(args)
    return gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
