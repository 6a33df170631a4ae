"""Thin ctypes binding of liblocc.so (include/locc.h) — argument marshalling only.

Every step of the query runs in the library's CUDA kernels; this module only passes pointers
(numpy arrays -> host pointers, torch tensors -> their data_ptr on host or device) and maps
status codes to exceptions.  If the library is missing it raises: there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOCC_LIB") or os.path.join(HERE, "liblocc.so")  # LOCC_LIB: a diagnostic build

LOCC_PREC_FP32 = 0
LOCC_PREC_BF16 = 1

EXPORTS = ("locc_create", "locc_load_weights", "locc_load_weights_mem", "locc_set_shapes", "locc_query",
           "locc_query_debug", "locc_query_grad", "locc_unet_n_params", "locc_load_unet_weights_mem",
           "locc_encode_shapes", "locc_set_unet_global_pool", "locc_get_cell_embeddings", "locc_query_cells", "locc_sim_run", "locc_set_precision", "locc_set_deterministic", "locc_set_timing", "locc_get_stats", "locc_destroy",
           "locc_comm_unique_id", "locc_comm_init", "locc_query_allgather",
           "locc_status_string", "locc_last_error", "locc_version")


class LoccError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("M", C.c_int32), ("H", C.c_int32), ("F", C.c_int32), ("precision", C.c_int32),
                ("device", C.c_int32), ("n_devices", C.c_int32), ("max_batch", C.c_int64),
                ("device_ids", C.POINTER(C.c_int32))]


class SimConfig(C.Structure):
    _fields_ = [("h", C.c_double), ("substeps", C.c_int32), ("detector", C.c_int32), ("gravity", C.c_float * 3),
                ("ks", C.c_float), ("kd", C.c_float), ("amp", C.c_float * 3), ("freq", C.c_float),
                ("slack", C.c_float)]

    @classmethod
    def from_dict(cls, d):
        return cls(d["h"], int(d["substeps"]), 1 if d.get("detector", "crop") == "cells" else 0,
                   (C.c_float * 3)(*d["gravity"]), d["ks"], d["kd"], (C.c_float * 3)(*d["amp"]), d["freq"],
                   d["slack"])


class Stats(C.Structure):
    _fields_ = [("pairs", C.c_int64), ("evaluated_pairs", C.c_int64), ("kept_rows", C.c_int64),
                ("nonempty_sides", C.c_int64), ("sub_batches", C.c_int64), ("kernel_launches", C.c_int64),
                ("encoder_ms", C.c_double), ("total_ms", C.c_double), ("head_ms", C.c_double),
                ("crop_ms", C.c_double), ("graph_replay", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load liblocc.so (raises if it was not built: run __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.locc_create.argtypes = [C.POINTER(Config), C.POINTER(vp)]
        L.locc_load_weights.argtypes = [vp, C.c_char_p]
        L.locc_load_weights_mem.argtypes = [vp, vp, C.c_size_t]
        L.locc_set_shapes.argtypes = [vp, vp, i32, i32]
        L.locc_query.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp]
        L.locc_query_debug.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.locc_query_grad.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, vp]
        L.locc_unet_n_params.argtypes = [i32, i32]
        L.locc_unet_n_params.restype = i64
        L.locc_load_unet_weights_mem.argtypes = [vp, vp, C.c_size_t]
        L.locc_encode_shapes.argtypes = [vp]
        L.locc_set_unet_global_pool.argtypes = [vp, i32]
        L.locc_get_cell_embeddings.argtypes = [vp, vp, vp]
        L.locc_query_cells.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]
        L.locc_sim_run.argtypes = [vp, C.POINTER(SimConfig), i32, vp, vp, vp, C.c_double, vp, vp]
        L.locc_set_precision.argtypes = [vp, i32]
        L.locc_set_timing.argtypes = [vp, i32]
        L.locc_set_deterministic.argtypes = [vp, i32]
        L.locc_comm_unique_id.argtypes = [vp]
        L.locc_comm_init.argtypes = [vp, i32, i32, vp]
        L.locc_query_allgather.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp]
        L.locc_get_stats.argtypes = [vp, C.POINTER(Stats)]
        L.locc_destroy.argtypes = [vp]
        L.locc_destroy.restype = None
        L.locc_status_string.argtypes = [C.c_int]
        L.locc_status_string.restype = C.c_char_p
        L.locc_last_error.restype = C.c_char_p
        L.locc_version.restype = C.c_char_p
        for name in EXPORTS[:9]:
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        L = lib()
        raise LoccError(rc, f"{L.locc_status_string(rc).decode()}: {L.locc_last_error().decode()}")


def _ptr(x, dtype=None, count=None):
    """Raw pointer of a numpy array or torch tensor; None -> NULL.  Checks contiguity, the element
    dtype (numpy dtype, matched by name for torch tensors) and that it holds >= `count` elements, so
    the library never reads or writes past the caller's allocation."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if dtype is not None and x.dtype != dtype:
            raise TypeError(f"expected {np.dtype(dtype)}, got {x.dtype}")
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        n, p = x.size, x.ctypes.data
    elif hasattr(x, "data_ptr"):  # torch.Tensor
        if dtype is not None and str(x.dtype).replace("torch.", "") != np.dtype(dtype).name:
            raise TypeError(f"expected {np.dtype(dtype)}, got {x.dtype}")
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        n, p = x.numel(), x.data_ptr()
    else:
        raise TypeError(type(x))
    if count is not None and n < count:
        raise ValueError(f"buffer holds {n} elements, the call needs {count}")
    return p


def comm_unique_id() -> bytes:
    """A new NCCL unique id (128 bytes) for locc_comm_init (rank 0 creates it and sends it to the others)."""
    buf = C.create_string_buffer(128)
    _check(lib().locc_comm_unique_id(buf))
    return buf.raw


class Locc:
    """One library context (locc_create / locc_destroy): on one CUDA device, or — devices=[d0, d1, ...]
    — a group that shards every query over those devices (d0 = home of device-resident buffers)."""

    def __init__(self, M=6, H=256, F=64, precision=LOCC_PREC_BF16, device=-1, max_batch=0, devices=None):
        self._h = C.c_void_p()
        n = len(devices) if devices else 0
        self._ids = (C.c_int32 * max(n, 1))(*(devices or [0]))
        self.cfg = Config(M, H, F, precision, device, n, max_batch, self._ids if n > 1 else None)
        _check(lib().locc_create(C.byref(self.cfg), C.byref(self._h)))
        self.M, self.H, self.F = M, H, F
        self.K = None

    def close(self):
        if self._h:
            lib().locc_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def load_weights(self, manifest_path: str):
        _check(lib().locc_load_weights(self._h, manifest_path.encode()))

    def load_weights_mem(self, flat):
        flat = np.ascontiguousarray(flat, np.float32)
        _check(lib().locc_load_weights_mem(self._h, _ptr(flat), flat.size))

    def set_shapes(self, points):
        S, K = int(points.shape[0]), int(points.shape[1])
        if isinstance(points, np.ndarray):
            points = np.ascontiguousarray(points, np.float32)
        _check(lib().locc_set_shapes(self._h, _ptr(points, np.float32, S * K * 3), S, K))
        self.K = K
        self.S = S

    def set_precision(self, precision):
        _check(lib().locc_set_precision(self._h, precision))

    def set_deterministic(self, on=True):
        """Bitwise batch-composition invariance of bf16 contexts (locc_set_deterministic)."""
        _check(lib().locc_set_deterministic(self._h, 1 if on else 0))

    def set_timing(self, on=True):
        _check(lib().locc_set_timing(self._h, 1 if on else 0))

    def stats(self):
        s = Stats()
        _check(lib().locc_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def query_into(self, pairs, poses, probs, labels=None, logits=None, stream=None):
        """locc_query on caller buffers (numpy = host, torch cuda tensors = device)."""
        N = int(pairs.shape[0])
        _check(lib().locc_query(self._h, *self._inputs(pairs, poses, N), N, _ptr(probs, np.float32, N),
                                _ptr(labels, np.uint8, N), _ptr(logits, np.float32, N), stream))

    @staticmethod
    def _inputs(pairs, poses, N):
        return _ptr(pairs, np.int32, 2 * N), _ptr(poses, np.float32, 14 * N)

    def query(self, pairs, poses):
        """Host convenience form: numpy in, numpy out (probs float32, labels uint8, logits float32)."""
        pairs = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
        poses = np.ascontiguousarray(poses, np.float32).reshape(-1, 2, 7)
        N = pairs.shape[0]
        probs = np.zeros(N, np.float32)
        labels = np.zeros(N, np.uint8)
        logits = np.zeros(N, np.float32)
        self.query_into(pairs, poses, probs, labels, logits)
        return probs, labels, logits

    # ------------------------------------------------------------- multi-process sharding (NCCL gather)
    def comm_init(self, world, rank, uid: bytes):
        """Join the NCCL world (locc_comm_init); uid from comm_unique_id() on rank 0."""
        if len(uid) != 128:
            raise ValueError("the NCCL unique id is 128 bytes")
        _check(lib().locc_comm_init(self._h, int(world), int(rank), C.c_char_p(uid)))

    def query_allgather_into(self, pairs, poses, probs, labels=None, logits=None, stream=None):
        """locc_query_allgather: this rank computes its contiguous shard of the GLOBAL batch (only that
        slice of pairs/poses is read) and every rank receives all N results."""
        N = int(pairs.shape[0])
        _check(lib().locc_query_allgather(self._h, *self._inputs(pairs, poses, N), N, _ptr(probs, np.float32, N),
                                          _ptr(labels, np.uint8, N), _ptr(logits, np.float32, N), stream))

    def query_grad_into(self, pairs, poses, probs, grad, labels=None, logits=None, stream=None):
        """locc_query_grad on caller buffers: grad [N][14] = d logit / d (q_A, t_A, q_B, t_B)."""
        N = int(pairs.shape[0])
        _check(lib().locc_query_grad(self._h, *self._inputs(pairs, poses, N), N, _ptr(probs, np.float32, N),
                                     _ptr(labels, np.uint8, N), _ptr(logits, np.float32, N),
                                     _ptr(grad, np.float32, 14 * N), stream))

    def query_grad(self, pairs, poses):
        """Host form of locc_query_grad -> (probs, labels, logits, grad [N][14])."""
        pairs = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
        poses = np.ascontiguousarray(poses, np.float32).reshape(-1, 2, 7)
        N = pairs.shape[0]
        probs = np.zeros(N, np.float32)
        labels = np.zeros(N, np.uint8)
        logits = np.zeros(N, np.float32)
        grad = np.zeros((N, 14), np.float32)
        self.query_grad_into(pairs, poses, probs, grad, labels, logits)
        return probs, labels, logits, grad

    # ------------------------------------------------------------- encode-once mode (NEXT-1)
    def load_unet_weights_mem(self, flat):
        flat = np.ascontiguousarray(flat, np.float32)
        _check(lib().locc_load_unet_weights_mem(self._h, _ptr(flat), flat.size))

    def set_unet_global_pool(self, mode):
        """0 = average (default), 1 = max; re-run encode_shapes afterwards."""
        _check(lib().locc_set_unet_global_pool(self._h, int(mode)))

    def encode_shapes(self):
        _check(lib().locc_encode_shapes(self._h))

    def cell_embeddings(self):
        """(E float32 [S][M^3][F] of the cached grids, device ms of the last encode)."""
        ms = C.c_double(0.0)
        out = np.zeros((self.S, self.M ** 3, self.F), np.float32)
        _check(lib().locc_get_cell_embeddings(self._h, _ptr(out), C.byref(ms)))
        return out, ms.value

    def encode_ms(self):
        """Device time (ms) of the last encode_shapes."""
        ms = C.c_double(0.0)
        _check(lib().locc_get_cell_embeddings(self._h, None, C.byref(ms)))
        return ms.value

    def query_cells_into(self, pairs, poses, probs, labels=None, logits=None, nsel=None, cells=None, emb=None,
                         stream=None):
        N = int(pairs.shape[0])
        words = (self.M ** 3 + 31) // 32
        _check(lib().locc_query_cells(self._h, *self._inputs(pairs, poses, N), N, _ptr(probs, np.float32, N),
                                      _ptr(labels, np.uint8, N), _ptr(logits, np.float32, N),
                                      _ptr(nsel, np.int32, 2 * N), _ptr(cells, np.uint32, 2 * N * words),
                                      _ptr(emb, np.float32, 2 * N * self.F), stream))

    def query_cells(self, pairs, poses, debug=False):
        """Host form of locc_query_cells -> dict (probs, labels, logits [, nsel, cells, emb])."""
        pairs = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
        poses = np.ascontiguousarray(poses, np.float32).reshape(-1, 2, 7)
        N = pairs.shape[0]
        o = dict(probs=np.zeros(N, np.float32), labels=np.zeros(N, np.uint8), logits=np.zeros(N, np.float32))
        if debug:
            o.update(nsel=np.zeros((N, 2), np.int32), cells=np.zeros((N, 2, (self.M ** 3 + 31) // 32), np.uint32),
                     emb=np.zeros((N, 2, self.F), np.float32))
        self.query_cells_into(pairs, poses, o["probs"], o["labels"], o["logits"], o.get("nsel"), o.get("cells"),
                              o.get("emb"))
        return o

    # ------------------------------------------------------------- closed loop (NEXT-3)
    def sim_run(self, sim, ids, body, state, t0=0.0, contacts=None, stream=None):
        """locc_sim_run on device tensors: ids int32 [E][3], body [E][3][4], state [E][3][13] (in place)."""
        cfg = SimConfig.from_dict(sim)
        E = int(ids.shape[0])
        _check(lib().locc_sim_run(self._h, C.byref(cfg), E, _ptr(ids, np.int32, 3 * E), _ptr(body, np.float32, 12 * E),
                                  _ptr(state, np.float32, 39 * E), float(t0), _ptr(contacts, np.int32, 3 * E),
                                  stream))

    def query_debug(self, pairs, poses):
        """Host form of locc_query_debug -> dict of every output and intermediate."""
        pairs = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
        poses = np.ascontiguousarray(poses, np.float32).reshape(-1, 2, 7)
        N = pairs.shape[0]
        words = (self.K + 31) // 32
        o = dict(probs=np.zeros(N, np.float32), labels=np.zeros(N, np.uint8), logits=np.zeros(N, np.float32),
                 kept=np.zeros((N, 2), np.int32), occ=np.zeros((N, 2), np.int32),
                 masks=np.zeros((N, 2, words), np.uint32), emb=np.zeros((N, 2, self.F), np.float32))
        _check(lib().locc_query_debug(self._h, _ptr(pairs), _ptr(poses), N, _ptr(o["probs"]), _ptr(o["labels"]),
                                      _ptr(o["logits"]), _ptr(o["kept"]), _ptr(o["occ"]), _ptr(o["masks"]),
                                      _ptr(o["emb"]), None))
        return o


def version():
    return lib().locc_version().decode()
