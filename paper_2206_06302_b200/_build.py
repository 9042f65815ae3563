"""In-tree build of the native pieces (no JIT cache: the .so files must
travel to the GPU box with the gpurun snapshot).

  paper_2206_06302_b200/lib/libcoloc_cuda.so    C-ABI kernel library (nvcc, sm_100a)
  paper_2206_06302_b200/lib/libcoloc_stream.so  C++ drop-in API + STREAM driver (g++)
  paper_2206_06302_b200/lib/stream_b200         STREAM CLI (SPEC.md:594 flags)
  paper_2206_06302_b200/lib/test_api            C++ API test binary
  oracle/liboracle.so, oracle/_ref/*            CPU checkers (oracle/Makefile)

Rebuilds only when a source is newer than its output.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
INCLUDE = REPO / "include"
CXX_INCLUDE = PKG / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CUDA_SOURCES = ["runtime.cu", "kernels.cu", "reduce.cu", "probe.cu", "staging.cu"]
CXX_SOURCES_CUDA = ["nccl.cpp"]


def _newer(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


def _headers() -> list[Path]:
    hs = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    hs += list(CXX_INCLUDE.rglob("*.hpp")) + list(CXX_INCLUDE.rglob("*.cuh"))
    return hs


def build_cuda(verbose: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libcoloc_cuda.so"
    srcs = [CSRC / s for s in CUDA_SOURCES] + [CSRC / s for s in CXX_SOURCES_CUDA]
    if not _newer(out, srcs + _headers()):
        return out
    objdir = LIB / "obj"
    objdir.mkdir(exist_ok=True)
    cmds, objs = [], []
    for s in CUDA_SOURCES:
        o = objdir / (s + ".o")
        cmds.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", str(INCLUDE), "-I", str(CSRC),
                     "-I", str(CXX_INCLUDE),
                     "-c", str(CSRC / s), "-o", str(o)])
        objs.append(str(o))
    for s in CXX_SOURCES_CUDA:
        o = objdir / (s + ".o")
        cmds.append(["g++", "-O2", "-std=c++17", "-fPIC", "-I", str(INCLUDE), "-I", str(CSRC),
                     "-I", f"{CUDA_HOME}/include", "-c", str(CSRC / s), "-o", str(o)])
        objs.append(str(o))
    # translation units compile independently: in parallel
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        for f in [pool.submit(_run, c, verbose) for c in cmds]:
            f.result()
    tmp = out.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart", "-ldl",
          "-Xlinker", "-soname=libcoloc_cuda.so"], verbose)
    tmp.replace(out)
    return out


def build_native_baseline(verbose: bool = False) -> Path:
    """libstream_native.so: the hand-written native CUDA STREAM the
    abstraction is compared with (measurement baseline, not the product)."""
    LIB.mkdir(exist_ok=True)
    out = LIB / "libstream_native.so"
    src = CSRC / "native_stream.cu"
    if _newer(out, [src, INCLUDE / "stream_native.h", INCLUDE / "coloc_stream.h"]):
        tmp = out.with_suffix(".so.tmp")
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-I", str(INCLUDE), "-o", str(tmp), str(src), "-Xlinker", "-soname=libstream_native.so"],
             verbose)
        tmp.replace(out)
    return out


def build_stream(verbose: bool = False) -> list[Path]:
    """C++ drop-in layer consumers: libcoloc_stream.so, stream_b200, test_api,
    and the nvcc-compiled user-code tests.  Independent targets build in
    parallel; the CLI waits for libcoloc_stream.so."""
    LIB.mkdir(exist_ok=True)
    cuda = build_cuda(verbose)
    flags = ["-O2", "-std=c++20", "-pthread", "-I", str(INCLUDE), "-I", str(CXX_INCLUDE)]
    link = [f"-L{LIB}", "-lcoloc_cuda", f"-Wl,-rpath,$ORIGIN", "-ldl"]
    deps = _headers() + [cuda]
    so, cli = LIB / "libcoloc_stream.so", LIB / "stream_b200"
    src, cli_src = CSRC / "stream_driver.cpp", CSRC / "stream_cli.cpp"
    test_src = REPO / "tests" / "cpp" / "test_api.cpp"
    # user code compiled by nvcc with __device__ lambdas (device_lambda.cuh);
    # -fmad=false keeps Listing 4's `b + c*scalar` uncontracted, as the
    # reference's default build does
    lam_src = REPO / "tests" / "cpp" / "test_lambda.cu"
    pol_src = REPO / "tests" / "cpp" / "test_launch_policy.cu"

    def stream_lib_and_cli():
        if _newer(so, [src] + deps):
            _run(["g++", *flags, "-fPIC", "-shared", "-o", str(so), str(src), *link], verbose)
        nat = build_native_baseline(verbose)
        if cli_src.exists() and _newer(cli, [cli_src, so, nat] + deps):
            _run(["g++", *flags, "-o", str(cli), str(cli_src), f"-L{LIB}", "-lcoloc_stream",
                  "-lstream_native", *link], verbose)

    jobs, outs = [], []
    if src.exists():
        jobs.append(stream_lib_and_cli)
        outs += [so, cli]
    if test_src.exists():
        t = LIB / "test_api"
        if _newer(t, [test_src] + deps):
            jobs.append(lambda t=t: _run(["g++", *flags, "-o", str(t), str(test_src), *link], verbose))
        outs.append(t)
    if lam_src.exists():
        t = LIB / "test_lambda"
        if _newer(t, [lam_src] + deps):
            jobs.append(lambda t=t: _run(
                [NVCC, *ARCH, "-O3", "-std=c++20", "--extended-lambda", "-fmad=false",
                 "-I", str(INCLUDE), "-I", str(CXX_INCLUDE), "-o", str(t), str(lam_src),
                 f"-L{LIB}", "-lcoloc_cuda", "-Xlinker", "-rpath,$ORIGIN"], verbose))
        outs.append(t)
    if pol_src.exists():
        t = LIB / "test_launch_policy"
        if _newer(t, [pol_src] + deps):
            jobs.append(lambda t=t: _run(
                [NVCC, *ARCH, "-O2", "-std=c++20", "-I", str(INCLUDE), "-I", str(CXX_INCLUDE),
                 "-o", str(t), str(pol_src)], verbose))
        outs.append(t)
    with ThreadPoolExecutor(max_workers=max(1, len(jobs))) as pool:
        for f in [pool.submit(j) for j in jobs]:
            f.result()
    return outs


def build_oracle(verbose: bool = False) -> None:
    """CPU checkers.  The reference binary is only (re)built where
    /root/reference exists; the GPU box uses the prebuilt copy."""
    targets = ["oracle"]
    if Path("/root/reference/proj/include/coloc").is_dir():
        targets.append("ref")
    _run(["make", "-s", "-C", str(REPO / "oracle"), *targets], verbose)


def build_all(verbose: bool = False) -> None:
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    # the CPU checkers do not depend on the CUDA libraries: build them
    # alongside
    with ThreadPoolExecutor(max_workers=2) as pool:
        oracle = pool.submit(build_oracle, verbose)
        build_cuda(verbose)
        build_stream(verbose)
        oracle.result()


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv)
    print("built:", *sorted(p.name for p in LIB.iterdir() if p.is_file()))
