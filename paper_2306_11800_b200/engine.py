"""ctypes front-end of the B200 engine's C ABI (include/dqtg.h, libdqtg.so).

This is the device-resident API used by bench.py and the distributed driver:
checkpoints stay in HBM (``DevCheckpoint``), quantized states stay in HBM
(``DevState``) and records are produced on the device.  The reference-shaped
value API (``dqt`` module, include/dqt/*.hpp) sits on the same C ABI.

There is no CPU fallback: importing this module on a machine without the built
library raises, and creating an ``Engine`` without a Blackwell GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libdqtg.so")

# dqtg_status -> exception name of the reference (include/dqt/errors.hpp)
STATUS_NAMES = {
    1: "Error", 2: "BadMagic", 3: "TruncatedFile", 4: "ShapeMismatch", 5: "NonFiniteData",
    6: "IoError", 7: "AlphaOutOfRange", 8: "AlphaMismatch", 9: "EmptySketch",
    10: "MissingGradients", 11: "MissingScores", 12: "TooFewDistinctPoints", 13: "CorruptIndex",
    14: "CorruptBitstream", 15: "ChecksumMismatch", 16: "ChainCorrupt", 17: "CudaError",
}


class EngineError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, "Error")


class Config(C.Structure):
    """dqtg_config == dqt::QuantConfig (quantize.hpp:13-26)."""
    _fields_ = [("bins", C.c_uint32), ("embed_bins", C.c_uint32), ("prune_frac", C.c_double),
                ("protect_frac", C.c_double), ("metric", C.c_uint32), ("sigma", C.c_double),
                ("alpha", C.c_double)]

    def __init__(self, bins=16, embed_bins=32, prune_frac=0.0, protect_frac=0.005, metric=0,
                 sigma=0.2, alpha=0.01):
        super().__init__(bins, embed_bins, prune_frac, protect_frac, int(metric), sigma, alpha)

    def astuple(self):
        return (self.bins, self.embed_bins, self.prune_frac, self.protect_frac, self.metric,
                self.sigma, self.alpha)


class _Layout(C.Structure):
    _fields_ = [("n_tensors", C.c_uint32), ("names", C.POINTER(C.c_char_p)),
                ("types", C.POINTER(C.c_uint8)), ("ranks", C.POINTER(C.c_uint8)),
                ("dims", C.POINTER(C.c_uint64))]


class _Info(C.Structure):
    _fields_ = [("step", C.c_uint64), ("config", Config), ("codebook_len", C.c_uint32 * 7),
                ("max_levels", C.c_uint32), ("param_count", C.c_uint64),
                ("protected_total", C.c_uint64)]


_P = C.c_void_p


# void (*)(void* user, uint64_t k, const dqtg_record* record)
RECORD_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_void_p)
# void (*)(void* user, uint64_t k, const dqtg_qstate* state)
STATE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_void_p)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (make -C "
                          f"paper_2306_11800_b200/csrc)")
    L = C.CDLL(LIB_PATH)
    sig = {
        "dqtg_last_error": (C.c_char_p, []),
        "dqtg_engine_create": (C.c_int, [C.c_int, _P, C.POINTER(_P)]),
        "dqtg_engine_destroy": (None, [_P]),
        "dqtg_engine_sync": (C.c_int, [_P]),
        "dqtg_engine_launches": (C.c_uint64, [_P]),
        "dqtg_engine_profile": (C.c_int, [_P, C.c_int]),
        "dqtg_engine_profile_report": (C.c_int, [_P, C.c_char_p, C.c_uint64]),
        "dqtg_engine_sync_stats": (None, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
        "dqtg_sketch_range": (C.c_int, [C.c_double, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "dqtg_sketch_build": (C.c_int, [_P, _P, C.c_uint64, C.c_double, C.POINTER(C.c_uint64),
                                        _P, _P]),
        "dqtg_ema_update": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_double]),
        "dqtg_compute_scores": (C.c_int, [_P, _P, _P, C.c_uint64, _P, _P]),
        "dqtg_ckpt_create": (C.c_int, [_P, C.POINTER(_Layout), C.POINTER(_P)]),
        "dqtg_ckpt_destroy": (None, [_P]),
        "dqtg_ckpt_set_weights": (C.c_int, [_P, _P]),
        "dqtg_ckpt_set_scores": (C.c_int, [_P, _P, _P]),
        "dqtg_ckpt_set_ema": (C.c_int, [_P, _P]),
        "dqtg_ckpt_update_ema": (C.c_int, [_P, _P, C.c_double]),
        "dqtg_ckpt_param_count": (C.c_uint64, [_P]),
        "dqtg_ckpt_weights_dev": (_P, [_P]),
        "dqtg_ckpt_ema_dev": (_P, [_P]),
        "dqtg_ckpt_tensor_offset": (C.c_uint64, [_P, C.c_uint32]),
        "dqtg_ckpt_tensor_count": (C.c_uint32, [_P]),
        "dqtg_ckpt_tensor_info": (C.c_int, [_P, C.c_uint32, C.c_char_p, C.c_uint64,
                                            C.POINTER(C.c_uint8), C.POINTER(C.c_uint8), _P]),
        "dqtg_ckpt_download": (C.c_int, [_P, _P]),
        "dqtg_ckpt_set_types": (C.c_int, [_P, _P]),
        "dqtg_ckpt_read_dqt1": (C.c_int, [_P, C.c_char_p, C.c_int, C.c_int, C.POINTER(_P),
                                          C.POINTER(C.c_uint64), _P, C.c_uint64,
                                          C.POINTER(C.c_uint64)]),
        "dqtg_quantize": (C.c_int, [_P, _P, C.POINTER(Config), C.c_uint64, C.c_uint64,
                                    C.POINTER(_P)]),
        "dqtg_qstate_info_get": (C.c_int, [_P, C.POINTER(_Info)]),
        "dqtg_qstate_protected_counts": (C.c_int, [_P, _P]),
        "dqtg_qstate_download": (C.c_int, [_P, _P, _P, _P, _P]),
        "dqtg_qstate_upload": (C.c_int, [_P, C.POINTER(_Layout), C.c_uint64, C.POINTER(Config),
                                         _P, _P, _P, _P, _P, _P, C.POINTER(_P)]),
        "dqtg_qstate_destroy": (None, [_P]),
        "dqtg_qstate_tensor_count": (C.c_uint32, [_P]),
        "dqtg_qstate_tensor_info": (C.c_int, [_P, C.c_uint32, C.c_char_p, C.c_uint64,
                                              C.POINTER(C.c_uint8), C.POINTER(C.c_uint8), _P]),
        "dqtg_qstate_levels_dev": (_P, [_P]),
        "dqtg_dequantize": (C.c_int, [_P, _P, _P]),
        "dqtg_encode_record": (C.c_int, [_P, _P, _P, C.c_double, C.POINTER(_P)]),
        "dqtg_record_size": (C.c_uint64, [_P]),
        "dqtg_payload_bytes": (C.c_int, [_P, _P, _P, C.c_int, C.POINTER(C.c_uint64)]),
        "dqtg_record_copy": (C.c_int, [_P, _P]),
        "dqtg_record_dev": (_P, [_P]),
        "dqtg_record_destroy": (None, [_P]),
        "dqtg_decode_record": (C.c_int, [_P, C.c_char_p, C.c_uint64, _P, C.POINTER(_P)]),
        "dqtg_compress_step": (C.c_int, [_P, _P, C.POINTER(Config), C.c_uint64, C.c_uint64, _P,
                                         C.c_double, C.POINTER(_P), C.POINTER(_P)]),
        "dqtg_eval_batch": (C.c_int, [_P, _P, _P, _P, C.c_uint32, _P, _P]),
        "dqtg_partition": (C.c_int, [_P, _P, C.POINTER(Config), _P]),
        "dqtg_proxy_quality": (C.c_int, [_P, _P, _P, _P, C.POINTER(C.c_double)]),
        "dqtg_qstate_equal": (C.c_int, [_P, _P, _P, C.POINTER(C.c_int)]),
        "dqtg_ckpt_release": (C.c_int, [_P]),
        "dqtg_engine_trim": (C.c_int, [_P]),
        "dqtg_decode_chain": (C.c_int, [_P, C.c_uint32, _P, _P, _P, _P, _P, C.POINTER(_P)]),
        "dqtg_shard_hist_len": (C.c_uint64, [_P, C.POINTER(Config), C.c_int]),
        "dqtg_shard_stage1": (C.c_int, [_P, _P, C.POINTER(Config), _P]),
        "dqtg_shard_stage2": (C.c_int, [_P, _P, C.POINTER(Config), _P, _P]),
        "dqtg_shard_stage3": (C.c_int, [_P, _P, C.POINTER(Config), C.c_uint64, C.c_uint64, _P,
                                        C.POINTER(_P)]),
        "dqtg_encode_record_shard": (C.c_int, [_P, _P, _P, C.c_double, C.c_uint32, C.c_uint32,
                                               C.POINTER(_P), C.POINTER(C.c_uint64)]),
        "dqtg_approx_kmeans": (C.c_int, [_P, _P, C.c_uint64, C.c_uint32, C.c_double, C.c_double,
                                         C.c_uint64, _P, C.POINTER(C.c_uint32)]),
        "dqtg_kmeanspp_init": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint64, _P]),
        "dqtg_lloyd": (C.c_int, [_P, _P, _P, C.c_uint64, _P, C.c_uint32, C.c_double, C.c_uint32,
                                 C.POINTER(C.c_uint32)]),
        "dqtg_sq_loss": (C.c_int, [_P, _P, _P, C.c_uint64, _P, C.c_uint32,
                                   C.POINTER(C.c_double)]),
        "dqtg_delta_compute": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, _P]),
        "dqtg_delta_apply": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, _P]),
        "dqtg_crc32": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_uint32)]),
        "dqtg_pipe_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(_P)]),
        "dqtg_pipe_destroy": (None, [_P]),
        "dqtg_pipe_launches": (C.c_uint64, [_P]),
        "dqtg_pipe_set_stream": (None, [_P, _P]),
        "dqtg_pipe_set_comms": (C.c_int, [_P, _P, C.c_int, C.c_uint32]),
        "dqtg_comm_unique_id": (C.c_int, [_P]),
        "dqtg_comm_init": (C.c_int, [_P, _P, C.c_int, C.c_int, C.POINTER(_P)]),
        "dqtg_comm_destroy": (None, [_P]),
        "dqtg_comm_rank": (C.c_int, [_P]),
        "dqtg_comm_size": (C.c_int, [_P]),
        "dqtg_comm_allreduce_u64": (C.c_int, [_P, _P, _P, C.c_uint64]),
        "dqtg_compress_sharded": (C.c_int, [_P, _P, _P, C.POINTER(Config), C.c_uint64,
                                            C.c_uint64, _P, C.c_double, C.c_uint32,
                                            C.POINTER(_P), C.POINTER(_P)]),
        "dqtg_pipe_run": (C.c_int, [_P, C.POINTER(_Layout), _P, C.c_uint64, _P, _P,
                                    C.POINTER(Config), C.c_uint64, _P, C.c_double, RECORD_FN, _P,
                                    C.POINTER(_P)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


LIB = _load()


def _check(rc):
    if rc:
        raise EngineError(rc, LIB.dqtg_last_error().decode(errors="replace"))


def _ptr(a):
    return a.ctypes.data if isinstance(a, np.ndarray) else int(a)


class _Meta:
    """Keeps the ctypes arrays of a dqtg_layout alive."""

    def __init__(self, names, types, shapes):
        self.names = list(names)
        self.types = [int(t) for t in types]
        self.shapes = [tuple(int(d) for d in s) for s in shapes]
        n = len(self.names)
        self._names = (C.c_char_p * max(n, 1))(*[s.encode() for s in self.names])
        self._types = np.array(self.types or [0], np.uint8)
        self._ranks = np.array([len(s) for s in self.shapes] or [0], np.uint8)
        self._dims = np.array([d for s in self.shapes for d in s] or [0], np.uint64)
        self.c = _Layout(n, self._names, self._types.ctypes.data_as(C.POINTER(C.c_uint8)),
                         self._ranks.ctypes.data_as(C.POINTER(C.c_uint8)),
                         self._dims.ctypes.data_as(C.POINTER(C.c_uint64)))
        self.numel = [int(np.prod(s, dtype=np.uint64)) for s in self.shapes]


def _as_buf(a):
    """numpy arrays stay host buffers; ints are raw (host or device) pointers."""
    if isinstance(a, (int, np.integer)):
        return int(a)
    return np.ascontiguousarray(a, np.float32)


def _ptr_array(arrs):
    return (C.c_void_p * max(len(arrs), 1))(*[_ptr(a) for a in arrs])


@dataclass
class HostState:
    """Host copy of a quantized state (dqt::QuantizedCheckpoint)."""
    step: int
    config: tuple
    codebooks: list
    names: list
    types: list
    shapes: list
    levels: list
    prot_pos: list = field(default_factory=list)
    prot_val: list = field(default_factory=list)


class DevCheckpoint:
    def __init__(self, engine, names, types, shapes):
        self.engine = engine
        self.meta = _Meta(names, types, shapes)
        h = _P()
        _check(LIB.dqtg_ckpt_create(engine.h, C.byref(self.meta.c), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and LIB is not None:
            LIB.dqtg_ckpt_destroy(self.h)
            self.h = None

    def set_weights(self, arrays):
        arrs = [_as_buf(a) for a in arrays]
        _check(LIB.dqtg_ckpt_set_weights(self.h, _ptr_array(arrs)))

    def release(self):
        """Free the device buffers (the next set_weights / set_ema allocates them again)."""
        _check(LIB.dqtg_ckpt_release(self.h))

    def set_scores(self, mag, sens=None):
        m = [_as_buf(a) for a in mag]
        s = None if sens is None else [_as_buf(a) for a in sens]
        _check(LIB.dqtg_ckpt_set_scores(self.h, _ptr_array(m), None if s is None else _ptr_array(s)))

    def set_ema(self, ema):
        e = None if ema is None else [_as_buf(a) for a in ema]
        _check(LIB.dqtg_ckpt_set_ema(self.h, None if e is None else _ptr_array(e)))

    def update_ema(self, grads, beta=0.9):
        g = [_as_buf(a) for a in grads]
        _check(LIB.dqtg_ckpt_update_ema(self.h, _ptr_array(g), beta))

    @property
    def weights_dev(self):
        return LIB.dqtg_ckpt_weights_dev(self.h)

    @property
    def ema_dev(self):
        return LIB.dqtg_ckpt_ema_dev(self.h)

    def tensor_offset(self, i):
        return LIB.dqtg_ckpt_tensor_offset(self.h, i)

    def tensor_ptrs(self):
        """Device pointers of the per-tensor weight slices (inputs to other calls)."""
        base = self.weights_dev
        return [base + 4 * self.tensor_offset(i) for i in range(len(self.meta.names))]

    def _same_layout(self, other):
        if other.meta.shapes != self.meta.shapes:
            raise EngineError(4, "EMA/gradient checkpoint does not match the layout")

    def set_ema_from(self, ema_ckpt):
        """EMA from a device checkpoint (e.g. an ingested ema.dqt), copied in HBM."""
        self._same_layout(ema_ckpt)
        _check(LIB.dqtg_ckpt_set_ema(self.h, _ptr_array(ema_ckpt.tensor_ptrs())))

    def update_ema_from(self, grads_ckpt, beta=0.9):
        """ema_update (ranker.cpp:21-37) with gradients already in HBM."""
        self._same_layout(grads_ckpt)
        _check(LIB.dqtg_ckpt_update_ema(self.h, _ptr_array(grads_ckpt.tensor_ptrs()), beta))

    @classmethod
    def _wrap(cls, engine, h):
        """Adopt a checkpoint handle made by the engine (e.g. dqtg_ckpt_read_dqt1)."""
        self = cls.__new__(cls)
        self.engine, self.h = engine, h
        names, types, shapes = [], [], []
        buf = C.create_string_buffer(1 << 16)
        dims = np.zeros(256, np.uint64)
        t, r = C.c_uint8(), C.c_uint8()
        for i in range(LIB.dqtg_ckpt_tensor_count(h)):
            _check(LIB.dqtg_ckpt_tensor_info(h, i, buf, len(buf), C.byref(t), C.byref(r),
                                             dims.ctypes.data))
            names.append(buf.value.decode("utf-8", "surrogateescape"))
            types.append(t.value)
            shapes.append(tuple(int(d) for d in dims[:r.value]))
        self.meta = _Meta(names, types, shapes)
        return self

    def set_types(self, types):
        """Replace the layer types (apply_layer_rules, src/tensor.cpp:225-227)."""
        t = np.array([int(x) for x in types] or [0], np.uint8)
        _check(LIB.dqtg_ckpt_set_types(self.h, t.ctypes.data))
        self.meta = _Meta(self.meta.names, t[:len(types)].tolist(), self.meta.shapes)

    def download(self):
        """Per-tensor float32 host copies of the weights."""
        out = [np.empty(n, np.float32) for n in self.meta.numel]
        _check(LIB.dqtg_ckpt_download(self.h, _ptr_array(out)))
        return out


def parse_dqt1_meta(raw):
    """u32 count | {u16 len, key | u32 len, value} (tensor.cpp:83-88) -> dict
    (a std::map in the reference: later duplicate keys win)."""
    import struct
    n, = struct.unpack_from("<I", raw, 0)
    at, out = 4, {}
    for _ in range(n):
        k, = struct.unpack_from("<H", raw, at)
        key = raw[at + 2:at + 2 + k].decode("utf-8", "surrogateescape")
        at += 2 + k
        v, = struct.unpack_from("<I", raw, at)
        out[key] = raw[at + 4:at + 4 + v].decode("utf-8", "surrogateescape")
        at += 4 + v
    return out


def state_meta(h) -> "_Meta":
    """Layout of a state handle (names, types, shapes) from the engine."""
    names, types, shapes = [], [], []
    buf = C.create_string_buffer(4096)
    dims = np.zeros(8, np.uint64)
    t, r = C.c_uint8(), C.c_uint8()
    for i in range(LIB.dqtg_qstate_tensor_count(h)):
        _check(LIB.dqtg_qstate_tensor_info(h, i, buf, len(buf), C.byref(t), C.byref(r),
                                           dims.ctypes.data))
        names.append(buf.value.decode("utf-8", "surrogateescape"))
        types.append(t.value)
        shapes.append(tuple(int(d) for d in dims[:r.value]))
    return _Meta(names, types, shapes)


class DevState:
    def __init__(self, engine, h, meta):
        self.engine, self.h, self.meta = engine, h, meta

    def __del__(self):
        if getattr(self, "h", None) and LIB is not None:
            LIB.dqtg_qstate_destroy(self.h)
            self.h = None

    def info(self):
        i = _Info()
        _check(LIB.dqtg_qstate_info_get(self.h, C.byref(i)))
        return i

    @property
    def levels_dev(self):
        return LIB.dqtg_qstate_levels_dev(self.h)

    def download(self) -> HostState:
        info = self.info()
        m = self.meta
        nt = len(m.names)
        counts = np.zeros(max(nt, 1), np.uint64)
        _check(LIB.dqtg_qstate_protected_counts(self.h, counts.ctypes.data))
        levels = [np.zeros(n, np.uint16) for n in m.numel]
        pp = [np.zeros(int(c), np.uint64) for c in counts[:nt]]
        pv = [np.zeros(int(c), np.uint16) for c in counts[:nt]]
        cbs = [np.zeros(info.codebook_len[lt], np.float32) for lt in range(7)]
        _check(LIB.dqtg_qstate_download(self.h, _ptr_array(levels), _ptr_array(pp),
                                        _ptr_array(pv), _ptr_array(cbs)))
        return HostState(int(info.step), info.config.astuple(), cbs, list(m.names),
                         list(m.types), list(m.shapes), levels, pp, pv)

    def dequantize(self):
        outs = [np.zeros(n, np.float32) for n in self.meta.numel]
        _check(LIB.dqtg_dequantize(self.engine.h, self.h, _ptr_array(outs)))
        return outs


# cudaStreamLegacy: the handle of the legacy default stream (value 0 is NULL in the
# C ABI, which means "the engine creates its own non-blocking stream")
_CUDA_STREAM_LEGACY = 1


class Engine:
    def __init__(self, device=0, stream=None):
        """stream: a CUDA stream handle the engine works on, e.g.
        ``torch.cuda.current_stream().cuda_stream``; None = the engine's own stream.
        Handle 0 (torch's default stream) is the legacy default stream, so the engine
        stays ordered with torch work issued there (a NULL handle would give the engine
        a private non-blocking stream that races with it)."""
        h = _P()
        if stream is not None and int(stream) == 0:
            stream = _CUDA_STREAM_LEGACY
        _check(LIB.dqtg_engine_create(device, stream, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and LIB is not None:  # LIB is None at interpreter exit
            LIB.dqtg_engine_destroy(self.h)
            self.h = None

    def sync(self):
        _check(LIB.dqtg_engine_sync(self.h))

    def read_ema_dqt1(self, path, direct=False, threads=0):
        """ema_load (ranker.cpp:50-61) into HBM: (DevCheckpoint of the EMA, beta,
        step_count); IoError when the beta/step_count meta is missing."""
        ck, _, meta = self.read_dqt1(path, direct, threads)
        if "beta" not in meta or "step_count" not in meta:
            raise EngineError(6, f"{path}: missing beta/step_count meta")
        return ck, float(meta["beta"]), int(meta["step_count"])

    def read_dqt1(self, path, direct=False, threads=0):
        """DQT1 file -> (DevCheckpoint, step, meta dict) via dqtg_ckpt_read_dqt1
        (replaces read_checkpoint, src/tensor.cpp:110-149)."""
        h, step, mlen = _P(), C.c_uint64(), C.c_uint64()
        meta = C.create_string_buffer(1 << 16)
        path_b = os.fsencode(path)
        _check(LIB.dqtg_ckpt_read_dqt1(self.h, path_b, 1 if direct else 0, int(threads), C.byref(h),
                                       C.byref(step), meta, len(meta), C.byref(mlen)))
        ck = DevCheckpoint._wrap(self, h)
        raw = meta.raw[:mlen.value]
        if mlen.value > len(meta):  # large meta section: fetch it whole
            big = C.create_string_buffer(mlen.value)
            h2 = _P()
            _check(LIB.dqtg_ckpt_read_dqt1(self.h, path_b, 0, int(threads), C.byref(h2), None, big,
                                           len(big), None))
            LIB.dqtg_ckpt_destroy(h2)
            raw = big.raw[:mlen.value]
        return ck, step.value, parse_dqt1_meta(raw)

    @property
    def launches(self):
        return LIB.dqtg_engine_launches(self.h)

    def sync_stats(self):
        """(host syncs so far, ms blocked in them)"""
        n, ms = C.c_uint64(), C.c_double()
        LIB.dqtg_engine_sync_stats(self.h, C.byref(n), C.byref(ms))
        return n.value, ms.value

    def profile(self, enable=True):
        _check(LIB.dqtg_engine_profile(self.h, 1 if enable else 0))

    def profile_report(self):
        """{kernel: (launches, total_ms)} since the last report (CUDA events)."""
        import json

        buf = C.create_string_buffer(1 << 16)
        _check(LIB.dqtg_engine_profile_report(self.h, buf, len(buf)))
        return {k: tuple(v) for k, v in json.loads(buf.value.decode()).items()}

    # -- sketch ------------------------------------------------------------
    @staticmethod
    def sketch_range(alpha):
        a, b = C.c_int64(), C.c_int64()
        _check(LIB.dqtg_sketch_range(alpha, C.byref(a), C.byref(b)))
        return a.value, b.value

    def sketch_build(self, x, alpha):
        x = np.ascontiguousarray(x, np.float32)
        kmin, kmax = self.sketch_range(alpha)
        pos = np.zeros(kmax - kmin + 1, np.uint64)
        neg = np.zeros_like(pos)
        z = C.c_uint64()
        _check(LIB.dqtg_sketch_build(self.h, x.ctypes.data, x.size, alpha, C.byref(z),
                                     pos.ctypes.data, neg.ctypes.data))
        return kmin, z.value, pos, neg

    # -- checkpoints / quantize ------------------------------------------------
    def checkpoint(self, names, types, shapes, weights=None, mag=None, sens=None, ema=None):
        c = DevCheckpoint(self, names, types, shapes)
        if weights is not None:
            c.set_weights(weights)
        if mag is not None:
            c.set_scores(mag, sens)
        elif ema is not None:
            c.set_ema(ema)
        return c

    def quantize(self, ckpt: DevCheckpoint, cfg: Config, seed=1, step=0) -> DevState:
        h = _P()
        _check(LIB.dqtg_quantize(self.h, ckpt.h, C.byref(cfg), seed, step, C.byref(h)))
        return DevState(self, h, ckpt.meta)

    def upload_state(self, st: HostState) -> DevState:
        meta = _Meta(st.names, st.types, st.shapes)
        cfg = Config(*st.config)
        cbl = np.array([len(c) for c in st.codebooks], np.uint32)
        cbs = [np.ascontiguousarray(c, np.float32) for c in st.codebooks]
        lv = [np.ascontiguousarray(x, np.uint16).ravel() for x in st.levels]
        npr = np.array([len(p) for p in st.prot_pos] or [0], np.uint64)
        pp = [np.ascontiguousarray(p, np.uint64) for p in st.prot_pos]
        pv = [np.ascontiguousarray(p, np.uint16) for p in st.prot_val]
        h = _P()
        _check(LIB.dqtg_qstate_upload(self.h, C.byref(meta.c), st.step, C.byref(cfg),
                                      cbl.ctypes.data, _ptr_array(cbs), _ptr_array(lv),
                                      npr.ctypes.data, _ptr_array(pp), _ptr_array(pv),
                                      C.byref(h)))
        return DevState(self, h, meta)

    # -- records -------------------------------------------------------------------
    def encode_record(self, target: DevState, base: DevState = None, quality=0.0) -> bytes:
        r = _P()
        _check(LIB.dqtg_encode_record(self.h, None if base is None else base.h, target.h,
                                      quality, C.byref(r)))
        try:
            n = LIB.dqtg_record_size(r)
            out = np.empty(n, np.uint8)
            _check(LIB.dqtg_record_copy(r, out.ctypes.data))
            return out.tobytes()
        finally:
            LIB.dqtg_record_destroy(r)

    @staticmethod
    def record_bytes(r, destroy=True) -> bytes:
        """Bytes of a record handle (dqtg_record_copy); destroys the handle by default."""
        try:
            n = LIB.dqtg_record_size(r)
            out = np.empty(n, np.uint8)
            _check(LIB.dqtg_record_copy(r, out.ctypes.data))
            return out.tobytes()
        finally:
            if destroy:
                LIB.dqtg_record_destroy(r)

    def trim(self):
        """Release scratch buffers and cached device blocks (dqtg_engine_trim)."""
        _check(LIB.dqtg_engine_trim(self.h))

    def states_equal(self, a: DevState, b: DevState) -> bool:
        """Device comparison of two states (levels, protected entries, codebooks, step)."""
        r = C.c_int()
        _check(LIB.dqtg_qstate_equal(self.h, a.h, b.h, C.byref(r)))
        return bool(r.value)

    def payload_bytes(self, base: DevState, target: DevState, variant=0) -> int:
        """payload_bytes_pe (0) / _rle (1) / _he (2) (codec.cpp:615-646) on the device."""
        n = C.c_uint64()
        _check(LIB.dqtg_payload_bytes(self.h, base.h, target.h, int(variant), C.byref(n)))
        return n.value

    def encode_record_handle(self, target, base=None, quality=0.0):
        r = _P()
        _check(LIB.dqtg_encode_record(self.h, None if base is None else base.h, target.h,
                                      quality, C.byref(r)))
        return r

    def decode_chain(self, records, base: DevState = None, on_state=None):
        """Chain::restore over host records (dqtg_decode_chain): record k+1's host walk
        overlaps the device decode of record k.  on_state(k, state_handle) is called
        with a borrowed dqtg_qstate handle for every record; returns the last state."""
        recs = [bytes(r) for r in records]
        n = len(recs)
        ptrs = (C.c_char_p * max(n, 1))(*recs)
        sizes = np.array([len(r) for r in recs] or [0], np.uint64)
        cb = STATE_FN((lambda user, k, st: on_state(int(k), st)) if on_state else 0)
        out = _P()
        _check(LIB.dqtg_decode_chain(self.h, n, C.cast(ptrs, C.c_void_p), sizes.ctypes.data,
                                     None if base is None else base.h, cb if on_state else None,
                                     None, C.byref(out)))
        if not out:
            return None
        return DevState(self, out, state_meta(out))

    def decode_record(self, rec: bytes, base: DevState = None) -> DevState:
        """decode_delta_record (codec.cpp:459-597) on the device."""
        h = _P()
        _check(LIB.dqtg_decode_record(self.h, rec, len(rec), None if base is None else base.h,
                                      C.byref(h)))
        return DevState(self, h, state_meta(h))

    def compress_step(self, ckpt, cfg, seed, step, base=None, quality=0.0):
        s, r = _P(), _P()
        _check(LIB.dqtg_compress_step(self.h, ckpt.h, C.byref(cfg), seed, step,
                                      None if base is None else base.h, quality, C.byref(s),
                                      C.byref(r)))
        return DevState(self, s, ckpt.meta), r

    # -- tensor-sharded quantization (multi-GPU) ------------------------------------
    def compress_sharded(self, comm, ckpt, cfg, seed, step, base=None, quality=0.0,
                         n_tensors_total=0):
        """One sharded Chain::append step over the NCCL communicator `comm`
        (dqtg_compress_sharded): returns (this rank's DevState, record handle on rank 0
        or None).  The caller owns the record handle (dqtg_record_destroy)."""
        s, r = _P(), _P()
        _check(LIB.dqtg_compress_sharded(self.h, comm.h, ckpt.h, C.byref(cfg), seed, step,
                                         None if base is None else base.h, quality,
                                         int(n_tensors_total), C.byref(s), C.byref(r)))
        return DevState(self, s, ckpt.meta), (r if r else None)

    def shard_hist_len(self, cfg, which):
        return LIB.dqtg_shard_hist_len(self.h, C.byref(cfg), which)

    def shard_stage1(self, ckpt, cfg, score_hist_dev):
        _check(LIB.dqtg_shard_stage1(self.h, ckpt.h, C.byref(cfg), score_hist_dev))

    def shard_stage2(self, ckpt, cfg, score_hist_dev, value_hist_dev):
        _check(LIB.dqtg_shard_stage2(self.h, ckpt.h, C.byref(cfg), score_hist_dev, value_hist_dev))

    def shard_stage3(self, ckpt, cfg, seed, step, value_hist_dev) -> DevState:
        h = _P()
        _check(LIB.dqtg_shard_stage3(self.h, ckpt.h, C.byref(cfg), seed, step, value_hist_dev,
                                     C.byref(h)))
        return DevState(self, h, ckpt.meta)

    def encode_record_shard(self, target, base, quality, global_B, global_tensors):
        """Returns (record handle, body_offset)."""
        r, off = _P(), C.c_uint64()
        _check(LIB.dqtg_encode_record_shard(self.h, None if base is None else base.h, target.h,
                                            quality, global_B, global_tensors, C.byref(r),
                                            C.byref(off)))
        return r, off.value

    def partition(self, ckpt, cfg):
        masks = [np.zeros(n, np.uint8) for n in ckpt.meta.numel]
        _check(LIB.dqtg_partition(self.h, ckpt.h, C.byref(cfg), _ptr_array(masks)))
        return masks

    def proxy_quality(self, names, types, shapes, orig, recon):
        """proxy_quality_delta (search.cpp:30-61) of per-tensor host arrays."""
        meta = _Meta(names, types, shapes)
        o = [np.ascontiguousarray(x, np.float32).ravel() for x in orig]
        r = [np.ascontiguousarray(x, np.float32).ravel() for x in recon]
        out = C.c_double()
        _check(LIB.dqtg_proxy_quality(self.h, C.byref(meta.c), _ptr_array(o), _ptr_array(r),
                                      C.byref(out)))
        return out.value

    def eval_batch(self, ckpt, cfgs, seeds):
        m = len(cfgs)
        arr = (Config * max(m, 1))(*cfgs)
        sd = np.ascontiguousarray(seeds, np.uint64)
        q = np.zeros(max(m, 1), np.float64)
        e = np.zeros(max(m, 1), np.float64)
        _check(LIB.dqtg_eval_batch(self.h, ckpt.h, C.cast(arr, C.c_void_p), sd.ctypes.data, m,
                                   q.ctypes.data, e.ctypes.data))
        return q[:m], e[:m]

    # -- clustering / primitives ------------------------------------------------------
    def approx_kmeans(self, values, k, sigma=0.2, alpha=0.01, seed=1):
        v = np.ascontiguousarray(values, np.float32).ravel()
        out = np.zeros(max(k, 1), np.float32)
        n = C.c_uint32()
        _check(LIB.dqtg_approx_kmeans(self.h, v.ctypes.data, v.size, k, sigma, alpha, seed,
                                      out.ctypes.data, C.byref(n)))
        return out[:n.value].copy()

    def crc32(self, data: bytes):
        b = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
        c = C.c_uint32()
        _check(LIB.dqtg_crc32(self.h, b.ctypes.data, len(data), C.byref(c)))
        return c.value

    def ema_update(self, ema, g, beta=0.9):
        e = np.ascontiguousarray(ema, np.float32).copy()
        g = np.ascontiguousarray(g, np.float32)
        _check(LIB.dqtg_ema_update(self.h, e.ctypes.data, g.ctypes.data, e.size, beta))
        return e

    def compute_scores(self, w, ema=None):
        w = np.ascontiguousarray(w, np.float32)
        mag = np.zeros_like(w)
        sens = None if ema is None else np.zeros_like(w)
        e = None if ema is None else np.ascontiguousarray(ema, np.float32)
        _check(LIB.dqtg_compute_scores(self.h, w.ctypes.data, None if e is None else e.ctypes.data,
                                       w.size, mag.ctypes.data,
                                       None if sens is None else sens.ctypes.data))
        return mag, sens

    def delta_compute(self, prev, cur, B):
        p = np.ascontiguousarray(prev, np.uint16)
        c = np.ascontiguousarray(cur, np.uint16)
        out = np.zeros(max(p.size, 1), np.uint16)
        _check(LIB.dqtg_delta_compute(self.h, p.ctypes.data, c.ctypes.data, p.size, B,
                                      out.ctypes.data))
        return out[:p.size]

    def kmeanspp_init(self, pts, w, k, seed):
        p = np.ascontiguousarray(pts, np.float64)
        ww = np.ascontiguousarray(w, np.float64)
        out = np.zeros(k, np.float64)
        _check(LIB.dqtg_kmeanspp_init(self.h, p.ctypes.data, ww.ctypes.data, p.size, k, seed,
                                      out.ctypes.data))
        return out

    def lloyd(self, pts, w, centers, tol=1e-6, max_iter=100):
        p = np.ascontiguousarray(pts, np.float64)
        ww = np.ascontiguousarray(w, np.float64)
        c = np.array(centers, np.float64)
        it = C.c_uint32()
        _check(LIB.dqtg_lloyd(self.h, p.ctypes.data, ww.ctypes.data, p.size, c.ctypes.data,
                              c.size, tol, max_iter, C.byref(it)))
        return c, it.value

    def sq_loss(self, pts, w, centers):
        p = np.ascontiguousarray(pts, np.float64)
        ww = np.ascontiguousarray(w, np.float64)
        c = np.ascontiguousarray(centers, np.float64)
        out = C.c_double()
        _check(LIB.dqtg_sq_loss(self.h, p.ctypes.data, ww.ctypes.data, p.size, c.ctypes.data,
                                c.size, C.byref(out)))
        return out.value


_DEFAULT = None


class Comm:
    """NCCL communicator of the engine library (dqtg_comm_*): one per rank, built from
    the id rank 0 makes (``Comm.unique_id()``) and hands to every rank out of band."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(LIB.dqtg_comm_unique_id(buf))
        return buf.raw

    def __init__(self, engine, uid: bytes, nranks: int, rank: int):
        h = _P()
        _check(LIB.dqtg_comm_init(engine.h, uid, int(nranks), int(rank), C.byref(h)))
        self.h = h
        self.engine = engine

    @property
    def rank(self):
        return LIB.dqtg_comm_rank(self.h)

    @property
    def size(self):
        return LIB.dqtg_comm_size(self.h)

    def allreduce_u64(self, ptr, n):
        _check(LIB.dqtg_comm_allreduce_u64(self.engine.h, self.h, ptr, int(n)))

    def __del__(self):
        if getattr(self, "h", None) and LIB is not None:
            LIB.dqtg_comm_destroy(self.h)
            self.h = None


class Pipe:
    """Native pipelined delta chain (dqtg_pipe_*, pipe.cu): `workers` engines with
    their own streams and host threads; snapshot k runs on worker k mod W."""

    def __init__(self, device=0, workers=2):
        h = _P()
        _check(LIB.dqtg_pipe_create(device, workers, C.byref(h)))
        self.h = h
        self.workers = workers
        self._nominal = None  # engine used for calls on returned states

    def __del__(self):
        if getattr(self, "h", None) and LIB is not None:
            LIB.dqtg_pipe_destroy(self.h)
            self.h = None

    @property
    def launches(self):
        return LIB.dqtg_pipe_launches(self.h)

    def set_stream(self, stream_ptr):
        """Runs fork from / join into this CUDA stream (events on it time a run)."""
        LIB.dqtg_pipe_set_stream(self.h, stream_ptr or None)

    def set_comms(self, comms, n_tensors_total=0):
        """Tensor-sharded multi-GPU runs: one engine Comm per worker (dqtg_pipe_set_comms)."""
        self._comms = list(comms)
        arr = (_P * max(1, len(self._comms)))(*[c.h for c in self._comms])
        _check(LIB.dqtg_pipe_set_comms(self.h, arr, len(self._comms), int(n_tensors_total)))

    def run(self, names, types, shapes, snapshots, cfg, seed=1, steps=None, ema=None,
            base=None, quality=0.0, on_record=None, engine=None, emas=None):
        """snapshots[k] = per-tensor arrays or raw (host/device) pointers of snapshot
        k; ema = per-tensor arrays/pointers shared by every snapshot, or emas[k] =
        snapshot k's own (None for both: magnitude scores only).  on_record(k,
        record_handle) is called on a worker thread.  Returns the last snapshot's
        DevState."""
        meta = _Meta(names, types, shapes)
        nt = len(meta.names)
        n = len(snapshots)
        bufs = [_as_buf(a) for snap in snapshots for a in snap]
        if len(bufs) != n * nt:
            raise ValueError("every snapshot needs one array per tensor")
        wptr = _ptr_array(bufs)
        if ema is not None and emas is not None:
            raise ValueError("pass either a shared ema or per-snapshot emas")
        if ema is not None:
            emas = [ema] * n
        ebufs = None if emas is None else [_as_buf(a) for e in emas for a in e]
        if ebufs is not None and len(ebufs) != n * nt:
            raise ValueError("every snapshot's EMA needs one array per tensor")
        eptr = None if ebufs is None else _ptr_array(ebufs)
        st = None
        if steps is not None:
            st = np.ascontiguousarray(steps, np.uint64)
        cb = RECORD_FN(0) if on_record is None else RECORD_FN(lambda u, k, r: on_record(int(k), r))
        h = _P()
        _check(LIB.dqtg_pipe_run(self.h, C.byref(meta.c), wptr, n,
                                 None if st is None else st.ctypes.data, eptr, C.byref(cfg), seed,
                                 None if base is None else base.h, quality, cb, None, C.byref(h)))
        if not h:
            return base
        if engine is None:
            if self._nominal is None:
                self._nominal = Engine(0)
            engine = self._nominal
        ds = DevState(engine, h, meta)
        ds._owner = self  # the state's memory belongs to a pipe worker engine
        return ds


def default_engine() -> Engine:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Engine(int(os.environ.get("DQT_DEVICE", "0")))
    return _DEFAULT
