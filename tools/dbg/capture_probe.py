"""Bisects multi-stream graph capture through the C ABI (debug probe)."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2206_06302_b200 import native as N

lib = N.cuda()
n = 1 << 20
bufs = [N.DeviceBuffer(8 * n) for _ in range(4)]
ss = [N.Stream(0), N.Stream(0)]


def step(name, fn):
    st = fn()
    print(name, st, (lib.coloc_cuda_last_error() or b"").decode(), flush=True)
    return st


def trial(label, body):
    print("==", label, flush=True)
    for s in ss:
        step("begin", lambda: lib.coloc_cuda_graph_capture_begin(0, s.handle))
    body()
    devs = (C.c_int * 2)(0, 0)
    strs = (C.c_void_p * 2)(*[s.handle for s in ss])
    gs = (C.c_void_p * 2)()
    step("end_many", lambda: lib.coloc_cuda_graph_capture_end_many(2, devs, strs, gs))
    for s, g in zip(ss, gs):
        if g:
            lib.coloc_cuda_graph_launch(0, g, s.handle)
            s.sync()


trial("kernels only", lambda: [step("copy", lambda i=i: lib.coloc_cuda_copy_f64(0, ss[i].handle, bufs[2 * i].ptr, bufs[2 * i + 1].ptr, n)) for i in range(2)])


def with_events():
    for i in range(2):
        e = C.c_void_p()
        step("evcreate", lambda: lib.coloc_cuda_event_create(0, C.byref(e)))
        step("evrecord", lambda: lib.coloc_cuda_event_record(0, e, ss[i].handle))
        step("copy", lambda: lib.coloc_cuda_copy_f64(0, ss[i].handle, bufs[2 * i].ptr, bufs[2 * i + 1].ptr, n))


trial("events + kernels", with_events)

# through the driver
devs = (C.c_int * 2)(0, 0)
cfg = N.StreamConfig(dtype=0, init=0, fma=0, synchronous=0, ntargets=2, devices=devs, count=n,
                     first=0, seed=0, scalar=3.0, triad_scalar=3.0, host_buffers=0, reduction=0)
h = C.c_void_p()
N.check(N.stream().coloc_stream_create(C.byref(cfg), C.byref(h)), "create", "stream")
st = N.stream().coloc_stream_iterate_many(h, 1, 0, 1)
print("driver no-record", st, N.stream().coloc_stream_last_error())
st = N.stream().coloc_stream_iterate_many(h, 1, 1, 1)
print("driver record", st, N.stream().coloc_stream_last_error())
