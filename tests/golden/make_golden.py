"""Generate the golden fixtures that pin the CPU oracle.

Runs the UNMODIFIED reference library (built by `make -C oracle ref` from
/root/reference into oracle/_ref/ref_stream_cpu) and records its outputs:

  kernels_f64.npz / kernels_f32.npz   seeded random a,b,c and the outputs of
                                      copy/scale/add/triad via the reference
                                      algorithms (algorithms.hpp:359-526)
  reference.json                      partition_block tables, algorithm_shape
                                      dumps, Listing 3 output, STREAM
                                      validation expectations and chained
                                      random-STREAM checksums

Only needed when the fixtures change; run here (the GPU box has no
/root/reference):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import subprocess
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF = REPO / "oracle" / "_ref" / "ref_stream_cpu"
SEED = 0x220606302


def ref(*args: str) -> str:
    out = subprocess.run([str(REF), *args], check=True, capture_output=True, text=True)
    return out.stdout.strip()


def kernels(dtype: str, n: int) -> None:
    np_t = np.float64 if dtype == "f64" else np.float32
    with tempfile.TemporaryDirectory() as d:
        ref("kernels", "--dtype", dtype, "--n", str(n), "--seed", hex(SEED), "--out", d)
        arrays = {k: np.fromfile(Path(d) / f"{k}.bin", dtype=np_t)
                  for k in ("a", "b", "c", "copy", "scale", "add", "triad")}
    np.savez_compressed(HERE / f"kernels_{dtype}.npz", seed=np.uint64(SEED), **arrays)


def main() -> None:
    if not REF.exists():
        subprocess.run(["make", "-C", str(REPO / "oracle"), "ref"], check=True)
    kernels("f64", 4099)
    kernels("f32", 4099)

    doc: dict = {"generator": "tests/golden/make_golden.py", "seed": SEED}
    doc["partition"] = {}
    for n, k in [(10, 2), (10, 3), (2, 3), (0, 4), (1, 1), (17, 5), (1 << 30, 8),
                 (3 * (1 << 30) + 5, 8), (10, 0)]:
        doc["partition"][f"{n},{k}"] = json.loads(ref("partition", "--n", str(n), "--k", str(k)))
    doc["shape"] = {}
    for n, doms, off, ln in [(100, "0-5;6-11", 0, 100), (100, "0-5;6-11", 37, 40),
                             (7, "0;1;2", 0, 7), (1000, "0-3", 0, 1000), (50, "0-1;2-3;4-5", 10, 35)]:
        key = f"{n}|{doms}|{off}|{ln}"
        doc["shape"][key] = json.loads(ref("shape", "--n", str(n), "--domains", doms,
                                           "--offset", str(off), "--len", str(ln)))
    doc["helloworld"] = ref("helloworld")
    doc["stream_expected"] = {}
    for dtype in ("f64", "f32"):
        for nt in (1, 2, 10, 13):
            js = json.loads(ref("stream", "--dtype", dtype, "--n", "64", "--ntimes", str(nt)))
            doc["stream_expected"][f"{dtype},{nt}"] = js["validation"]
    doc["stream_random"] = {}
    for dtype in ("f64", "f32"):
        for n, nt in ((1001, 1), (4099, 10)):
            js = json.loads(ref("stream", "--dtype", dtype, "--n", str(n), "--ntimes", str(nt),
                                "--random", hex(SEED)))
            doc["stream_random"][f"{dtype},{n},{nt}"] = js["validation"]["checksums"]
    (HERE / "reference.json").write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
