"""A/B timing of liblocc builds through the round-1 subset of the ABI (create, load weights, set
shapes, locc_query on device buffers): C3 step time on the same box.  usage: python tools/ab_query.py a.so b.so ...
A path may carry environment switches read at context creation: lib.so@LOCC_CROP_2PASS=1 (comma-separated)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import locc_synth as ls  # noqa: E402


class Cfg(C.Structure):
    _fields_ = [("M", C.c_int32), ("H", C.c_int32), ("F", C.c_int32), ("precision", C.c_int32),
                ("device", C.c_int32), ("n_devices", C.c_int32), ("max_batch", C.c_int64),
                ("device_ids", C.c_void_p)]


def run(spec, pts, pairs, poses, flat, reps=4):
    path, _, envs = spec.partition("@")
    env = dict(e.split("=", 1) for e in envs.split(",") if e)
    os.environ.update(env)
    L = C.CDLL(path)
    vp = C.c_void_p
    L.locc_create.argtypes = [C.POINTER(Cfg), C.POINTER(vp)]
    L.locc_load_weights_mem.argtypes = [vp, vp, C.c_size_t]
    L.locc_set_shapes.argtypes = [vp, vp, C.c_int32, C.c_int32]
    L.locc_query.argtypes = [vp, vp, vp, C.c_int64, vp, vp, vp, vp]
    L.locc_destroy.argtypes = [vp]
    h = vp()
    cfg = Cfg(6, 256, 64, 1, 0, 0, int(os.environ.get("AB_MAX_BATCH", "0")), None)  # AB_MAX_BATCH: sub-batch size
    assert L.locc_create(C.byref(cfg), C.byref(h)) == 0
    assert L.locc_load_weights_mem(h, flat.ctypes.data, flat.size) == 0
    assert L.locc_set_shapes(h, pts.ctypes.data, pts.shape[0], pts.shape[1]) == 0
    N = len(pairs)
    dp, dq = torch.from_numpy(pairs).cuda(), torch.from_numpy(poses).cuda()
    pr = torch.empty(N, device="cuda")
    s = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        L.locc_query(h, dp.data_ptr(), dq.data_ptr(), N, pr.data_ptr(), None, None, s.cuda_stream)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            flush.zero_()
            e0.record(s)
        L.locc_query(h, dp.data_ptr(), dq.data_ptr(), N, pr.data_ptr(), None, None, s.cuda_stream)
        with torch.cuda.stream(s):
            e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1))
    L.locc_destroy(h)
    for k in env:
        del os.environ[k]
    return sum(ts) / len(ts), pr.cpu()


def main(paths):
    wl = ls.make_workload("C3")
    flat = ls.weight_set("spread")
    res = []
    for rnd in range(2):  # interleaved twice against clock drift
        for p in paths:
            ms, pr = run(p, wl.points, wl.pairs, wl.poses, flat)
            res.append((p, ms))
            print(f"{os.path.basename(p)}: {ms:.2f} ms/step = {len(wl.pairs) / ms * 1e3 / 1e6:.3f} M checks/s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
