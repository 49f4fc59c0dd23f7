"""ctypes front-end for the plain-C oracle (oracle/dqt_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py as the checker.  The product package never
imports this module.

Data model (mirrors the reference value types, /root/reference/proj/include/dqt):
  * a checkpoint is a list of ``Tensor(name, type, shape, data)``;
  * a quantized state is a ``QState`` (step, config, 7 codebooks, per-tensor
    levels + protected (pos, bf16) entries), like dqt::QuantizedCheckpoint
    (quantize.hpp:86-110).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libdqt_oracle.so")


def build():
    subprocess.check_call(["make", "-s", "-C", HERE, "port"])


def _load():
    if not os.path.exists(LIB_PATH):
        build()
    return C.CDLL(LIB_PATH)


class Config(C.Structure):
    """dqt::QuantConfig (quantize.hpp:13-26)."""
    _fields_ = [("bins", C.c_uint32), ("embed_bins", C.c_uint32), ("prune_frac", C.c_double),
                ("protect_frac", C.c_double), ("metric", C.c_uint32), ("sigma", C.c_double),
                ("alpha", C.c_double)]

    def __init__(self, bins=16, embed_bins=32, prune_frac=0.0, protect_frac=0.005, metric=0,
                 sigma=0.2, alpha=0.01):
        super().__init__(bins, embed_bins, prune_frac, protect_frac, int(metric), sigma, alpha)

    def astuple(self):
        return (self.bins, self.embed_bins, self.prune_frac, self.protect_frac, self.metric,
                self.sigma, self.alpha)


class _Ckpt(C.Structure):
    _fields_ = [("nt", C.c_uint32), ("names", C.POINTER(C.c_char_p)),
                ("types", C.POINTER(C.c_uint8)), ("ranks", C.POINTER(C.c_uint8)),
                ("dims", C.POINTER(C.c_uint64)), ("data", C.POINTER(C.c_float))]


@dataclass
class Tensor:
    name: str
    type: int
    shape: tuple
    data: np.ndarray  # float32, flat or shaped

    @property
    def size(self):
        return int(np.prod(self.shape, dtype=np.uint64)) if len(self.shape) else 0


@dataclass
class QState:
    step: int
    config: tuple
    codebooks: list                     # 7 float32 arrays (empty when unused)
    names: list
    types: list
    shapes: list
    levels: list                        # per tensor uint16 flat
    prot_pos: list = field(default_factory=list)  # per tensor uint64
    prot_val: list = field(default_factory=list)  # per tensor uint16 (bf16 bits)

    def max_levels(self):
        return max((len(self.codebooks[t]) + 2 for t in self.types), default=0)

    def __eq__(self, o):
        if not isinstance(o, QState):
            return NotImplemented
        return (self.step == o.step and tuple(self.config) == tuple(o.config)
                and all(np.array_equal(a.view(np.uint32), b.view(np.uint32))
                        for a, b in zip(self.codebooks, o.codebooks))
                and self.names == o.names and self.types == o.types
                and [tuple(s) for s in self.shapes] == [tuple(s) for s in o.shapes]
                and all(np.array_equal(a, b) for a, b in zip(self.levels, o.levels))
                and all(np.array_equal(a, b) for a, b in zip(self.prot_pos, o.prot_pos))
                and all(np.array_equal(a, b) for a, b in zip(self.prot_val, o.prot_val)))


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle error {code} {what}")
        self.code = code


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class Oracle:
    def __init__(self):
        L = self.lib = _load()
        L.dqo_bucket_index.restype = C.c_int64
        L.dqo_bucket_index.argtypes = [C.c_double, C.c_double]
        L.dqo_representative.restype = C.c_double
        L.dqo_representative.argtypes = [C.c_double, C.c_int64]
        L.dqo_sketch_range.argtypes = [C.c_double, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.dqo_sketch_dense.argtypes = [C.c_void_p, C.c_size_t, C.c_double, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64), C.POINTER(C.c_uint64), C.c_void_p,
                                       C.c_void_p]
        L.dqo_mix_seed.restype = C.c_uint64
        L.dqo_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.dqo_kmeanspp_init.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32,
                                        C.c_uint64, C.c_void_p]
        L.dqo_lloyd.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint32,
                                C.c_double, C.c_uint32, C.POINTER(C.c_uint32)]
        L.dqo_sq_loss.restype = C.c_double
        L.dqo_sq_loss.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint32]
        L.dqo_approx_kmeans.argtypes = [C.c_void_p, C.c_size_t, C.c_uint32, C.c_double,
                                        C.c_double, C.c_uint64, C.c_void_p,
                                        C.POINTER(C.c_uint32)]
        L.dqo_ema_update.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_double]
        L.dqo_scores.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
        L.dqo_partition.argtypes = [C.POINTER(_Ckpt), C.c_void_p, C.c_void_p,
                                    C.POINTER(Config), C.c_void_p]
        L.dqo_quantize.argtypes = [C.POINTER(_Ckpt), C.c_uint64, C.c_void_p, C.c_void_p,
                                   C.POINTER(Config), C.c_uint64, C.POINTER(C.c_void_p)]
        L.dqo_q_free.argtypes = [C.c_void_p]
        L.dqo_q_levels.argtypes = [C.c_void_p, C.c_void_p]
        L.dqo_q_nprot.argtypes = [C.c_void_p, C.c_void_p]
        L.dqo_q_prot.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.dqo_q_codebook.restype = C.c_uint32
        L.dqo_q_codebook.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.dqo_q_param_count.restype = C.c_uint64
        L.dqo_q_param_count.argtypes = [C.c_void_p]
        L.dqo_q_make.restype = C.c_void_p
        L.dqo_q_make.argtypes = [C.POINTER(_Ckpt), C.c_uint64, C.POINTER(Config), C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dqo_dequantize.argtypes = [C.c_void_p, C.c_void_p]
        L.dqo_encode_record.argtypes = [C.c_void_p, C.c_void_p, C.c_double,
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
        L.dqo_decode_record.argtypes = [C.c_char_p, C.c_size_t, C.c_void_p,
                                        C.POINTER(C.c_void_p)]
        L.dqo_free.argtypes = [C.c_void_p]
        L.dqo_crc32.restype = C.c_uint32
        L.dqo_crc32.argtypes = [C.c_char_p, C.c_size_t]
        L.dqo_rle_encode.restype = C.c_size_t
        L.dqo_rle_encode.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
        L.dqo_huffman_encode.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_size_t), C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_size_t)]
        L.dqo_delta_compute.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32,
                                        C.c_void_p]
        L.dqo_rearrange.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32)]
        L.dqo_proxy_quality.restype = C.c_double
        L.dqo_proxy_quality.argtypes = [C.POINTER(_Ckpt), C.c_void_p]
        L.dqo_estimate_compression.restype = C.c_double
        L.dqo_estimate_compression.argtypes = [C.POINTER(_Ckpt), C.c_void_p]
        L.dqo_config_hash.restype = C.c_uint64
        L.dqo_config_hash.argtypes = [C.POINTER(Config)]
        L.dqo_quantize_seed.restype = C.c_uint64
        L.dqo_quantize_seed.argtypes = [C.c_uint64, C.POINTER(Config)]
        L.dqo_payload_bytes.restype = C.c_uint64
        L.dqo_payload_bytes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.dqo_generate_trajectory.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double,
                                              C.c_double, C.c_double, C.c_uint64, C.c_void_p,
                                              C.c_void_p]
        L.dqo_default_layout.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        L.dqo_sort_f32.argtypes = [C.c_void_p, C.c_size_t]
        L.dqo_sort_pairs_desc.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]

    # -- sketch ------------------------------------------------------------
    def bucket_index(self, alpha, x):
        return self.lib.dqo_bucket_index(alpha, x)

    def representative(self, alpha, k):
        return self.lib.dqo_representative(alpha, k)

    def sketch_range(self, alpha):
        a, b = C.c_int64(), C.c_int64()
        self.lib.dqo_sketch_range(alpha, C.byref(a), C.byref(b))
        return a.value, b.value

    def sketch_dense(self, x, alpha):
        """Returns (kmin, zero, pos[kmin..kmax], neg[kmin..kmax]) like sketch_build."""
        x = np.ascontiguousarray(x, np.float32)
        kmin, kmax = self.sketch_range(alpha)
        pos = np.zeros(kmax - kmin + 1, np.uint64)
        neg = np.zeros_like(pos)
        a, b, z = C.c_int64(), C.c_int64(), C.c_uint64()
        rc = self.lib.dqo_sketch_dense(x.ctypes.data, x.size, alpha, C.byref(a), C.byref(b),
                                       C.byref(z), pos.ctypes.data, neg.ctypes.data)
        if rc:
            raise OracleError(rc, "sketch")
        return kmin, z.value, pos, neg

    # -- clustering --------------------------------------------------------
    def approx_kmeans(self, values, k, sigma=0.2, alpha=0.01, seed=1):
        v = np.ascontiguousarray(values, np.float32).ravel()
        out = np.zeros(max(k, 1), np.float32)
        n = C.c_uint32()
        rc = self.lib.dqo_approx_kmeans(v.ctypes.data, v.size, k, sigma, alpha, seed,
                                        out.ctypes.data, C.byref(n))
        if rc:
            raise OracleError(rc, "approx_kmeans")
        return out[:n.value].copy()

    def kmeanspp_init(self, pts, w, k, seed):
        pts = np.ascontiguousarray(pts, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        out = np.zeros(k, np.float64)
        rc = self.lib.dqo_kmeanspp_init(pts.ctypes.data, w.ctypes.data, pts.size, k, seed,
                                        out.ctypes.data)
        if rc:
            raise OracleError(rc, "kmeanspp")
        return out

    def lloyd(self, pts, w, centers, tol=1e-6, max_iter=100):
        pts = np.ascontiguousarray(pts, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        c = np.array(centers, np.float64)
        it = C.c_uint32()
        rc = self.lib.dqo_lloyd(pts.ctypes.data, w.ctypes.data, pts.size, c.ctypes.data, c.size,
                                tol, max_iter, C.byref(it))
        if rc:
            raise OracleError(rc, "lloyd")
        return c, it.value

    def sq_loss(self, pts, w, centers):
        pts = np.ascontiguousarray(pts, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        c = np.ascontiguousarray(centers, np.float64)
        return self.lib.dqo_sq_loss(pts.ctypes.data, w.ctypes.data, pts.size, c.ctypes.data,
                                    c.size)

    def mix_seed(self, seed, salt):
        return self.lib.dqo_mix_seed(seed, salt)

    # -- checkpoint plumbing -----------------------------------------------
    def _ckpt(self, tensors, data=None):
        nt = len(tensors)
        keep = {}
        names = (C.c_char_p * max(nt, 1))(*[t.name.encode() for t in tensors])
        types = np.array([t.type for t in tensors] or [0], np.uint8)
        ranks = np.array([len(t.shape) for t in tensors] or [0], np.uint8)
        dims = np.array([d for t in tensors for d in t.shape] or [0], np.uint64)
        if data is None:
            data = (np.concatenate([np.ascontiguousarray(t.data, np.float32).ravel()
                                    for t in tensors]) if nt else np.zeros(1, np.float32))
        data = np.ascontiguousarray(data, np.float32)
        keep.update(names=names, types=types, ranks=ranks, dims=dims, data=data)
        ck = _Ckpt(nt, names, _p(types, C.c_uint8), _p(ranks, C.c_uint8), _p(dims, C.c_uint64),
                   _p(data, C.c_float))
        return ck, keep

    def _to_qstate(self, h, tensors_meta):
        L = self.lib
        names, types, shapes = tensors_meta
        N = L.dqo_q_param_count(h)
        lv = np.zeros(max(N, 1), np.uint16)
        L.dqo_q_levels(h, lv.ctypes.data)
        nt = len(names)
        npr = np.zeros(max(nt, 1), np.uint64)
        L.dqo_q_nprot(h, npr.ctypes.data)
        tot = int(npr[:nt].sum())
        pp = np.zeros(max(tot, 1), np.uint64)
        pv = np.zeros(max(tot, 1), np.uint16)
        L.dqo_q_prot(h, pp.ctypes.data, pv.ctypes.data)
        cbs = []
        for lt in range(7):
            n = L.dqo_q_codebook(h, lt, None)
            a = np.zeros(max(n, 1), np.float32)
            L.dqo_q_codebook(h, lt, a.ctypes.data)
            cbs.append(a[:n].copy())
        sizes = [int(np.prod(s, dtype=np.uint64)) for s in shapes]
        levels, ppos, pval = [], [], []
        o = po = 0
        for i in range(nt):
            levels.append(lv[o:o + sizes[i]].copy())
            o += sizes[i]
            k = int(npr[i])
            ppos.append(pp[po:po + k].copy())
            pval.append(pv[po:po + k].copy())
            po += k
        return cbs, levels, ppos, pval

    def _handle(self, q: QState):
        tensors = [Tensor(n, t, tuple(s), None) for n, t, s in zip(q.names, q.types, q.shapes)]
        ck, keep = self._ckpt(tensors, data=np.zeros(1, np.float32))
        cfg = Config(*q.config)
        cbl = np.array([len(c) for c in q.codebooks], np.uint32)
        cbf = (np.concatenate([np.asarray(c, np.float32) for c in q.codebooks])
               if cbl.sum() else np.zeros(1, np.float32))
        lv = (np.concatenate([np.asarray(x, np.uint16).ravel() for x in q.levels])
              if q.levels else np.zeros(1, np.uint16))
        npr = np.array([len(p) for p in q.prot_pos] or [0], np.uint64)
        pp = (np.concatenate([np.asarray(p, np.uint64) for p in q.prot_pos])
              if npr.sum() else np.zeros(1, np.uint64))
        pv = (np.concatenate([np.asarray(p, np.uint16) for p in q.prot_val])
              if npr.sum() else np.zeros(1, np.uint16))
        h = self.lib.dqo_q_make(C.byref(ck), q.step, C.byref(cfg), cbl.ctypes.data,
                                cbf.ctypes.data, lv.ctypes.data, npr.ctypes.data, pp.ctypes.data,
                                pv.ctypes.data)
        return h

    # -- quantize ------------------------------------------------------------
    def partition(self, tensors, mag, sens, cfg: Config):
        ck, keep = self._ckpt(tensors)
        N = keep["data"].size
        part = np.zeros(N, np.uint8)
        m = np.ascontiguousarray(mag, np.float32)
        s = None if sens is None else np.ascontiguousarray(sens, np.float32)
        rc = self.lib.dqo_partition(C.byref(ck), m.ctypes.data,
                                    None if s is None else s.ctypes.data, C.byref(cfg),
                                    part.ctypes.data)
        if rc:
            raise OracleError(rc, "partition")
        return part

    def quantize(self, tensors, step, mag, sens, cfg: Config, seed=1) -> QState:
        ck, keep = self._ckpt(tensors)
        m = np.ascontiguousarray(mag, np.float32)
        s = None if sens is None else np.ascontiguousarray(sens, np.float32)
        h = C.c_void_p()
        rc = self.lib.dqo_quantize(C.byref(ck), step, m.ctypes.data,
                                   None if s is None else s.ctypes.data, C.byref(cfg), seed,
                                   C.byref(h))
        if rc:
            raise OracleError(rc, "quantize")
        try:
            meta = ([t.name for t in tensors], [t.type for t in tensors],
                    [tuple(t.shape) for t in tensors])
            cbs, lv, pp, pv = self._to_qstate(h, meta)
        finally:
            self.lib.dqo_q_free(h)
        return QState(step, cfg.astuple(), cbs, meta[0], meta[1], meta[2], lv, pp, pv)

    def dequantize(self, q: QState):
        h = self._handle(q)
        try:
            N = sum(int(np.prod(s, dtype=np.uint64)) for s in q.shapes)
            out = np.zeros(max(N, 1), np.float32)
            rc = self.lib.dqo_dequantize(h, out.ctypes.data)
            if rc:
                raise OracleError(rc, "dequantize")
            return out[:N]
        finally:
            self.lib.dqo_q_free(h)

    def encode_record(self, target: QState, base: QState = None, quality=0.0) -> bytes:
        ht = self._handle(target)
        hb = self._handle(base) if base is not None else None
        try:
            p, n = C.c_void_p(), C.c_size_t()
            rc = self.lib.dqo_encode_record(hb, ht, quality, C.byref(p), C.byref(n))
            if rc:
                raise OracleError(rc, "encode")
            out = C.string_at(p, n.value)
            self.lib.dqo_free(p)
            return out
        finally:
            self.lib.dqo_q_free(ht)
            if hb:
                self.lib.dqo_q_free(hb)

    def decode_record(self, rec: bytes, base: QState = None) -> QState:
        hb = self._handle(base) if base is not None else None
        h = C.c_void_p()
        try:
            rc = self.lib.dqo_decode_record(rec, len(rec), hb, C.byref(h))
            if rc:
                raise OracleError(rc, "decode")
        finally:
            if hb:
                self.lib.dqo_q_free(hb)
        try:
            # read names/shapes back through a second decode-free path: the record itself
            names, types, shapes = _record_layout(rec)
            cbs, lv, pp, pv = self._to_qstate(h, (names, types, shapes))
            step, cfg = _record_step_cfg(rec)
        finally:
            self.lib.dqo_q_free(h)
        return QState(step, cfg, cbs, names, types, shapes, lv, pp, pv)

    def payload_bytes(self, base: QState, target: QState, variant: int):
        hb, ht = self._handle(base), self._handle(target)
        try:
            return self.lib.dqo_payload_bytes(hb, ht, variant)
        finally:
            self.lib.dqo_q_free(hb)
            self.lib.dqo_q_free(ht)

    # -- primitives ----------------------------------------------------------
    def crc32(self, b: bytes):
        return self.lib.dqo_crc32(b, len(b))

    def rle_encode(self, v):
        v = np.ascontiguousarray(v, np.uint16)
        out = np.zeros(2 * v.size + 1, np.int64)
        n = self.lib.dqo_rle_encode(v.ctypes.data, v.size, out.ctypes.data)
        return out[:n].copy()

    def huffman_encode(self, syms):
        s = np.ascontiguousarray(syms, np.int64)
        ts = np.zeros(s.size + 1, np.int64)
        tl = np.zeros(s.size + 1, np.uint8)
        tsize, p, nb = C.c_size_t(), C.c_void_p(), C.c_size_t()
        rc = self.lib.dqo_huffman_encode(s.ctypes.data, s.size, ts.ctypes.data, tl.ctypes.data,
                                         C.byref(tsize), C.byref(p), C.byref(nb))
        if rc:
            raise OracleError(rc, "huffman")
        data = C.string_at(p, nb.value) if nb.value else b""
        self.lib.dqo_free(p)
        return list(zip(ts[:tsize.value].tolist(), tl[:tsize.value].tolist())), data

    def delta_compute(self, prev, cur, B):
        prev = np.ascontiguousarray(prev, np.uint16)
        cur = np.ascontiguousarray(cur, np.uint16)
        out = np.zeros(max(prev.size, 1), np.uint16)
        rc = self.lib.dqo_delta_compute(prev.ctypes.data, cur.ctypes.data, prev.size, B,
                                        out.ctypes.data)
        if rc:
            raise OracleError(rc, "delta")
        return out[:prev.size]

    def rearrange(self, d, prev, B):
        d = np.ascontiguousarray(d, np.uint16)
        prev = np.ascontiguousarray(prev, np.uint16)
        out = np.zeros(max(d.size, 1), np.uint16)
        ids = np.zeros(B + 1, np.uint32)
        sizes = np.zeros(B + 1, np.uint64)
        ng = C.c_uint32()
        rc = self.lib.dqo_rearrange(d.ctypes.data, prev.ctypes.data, d.size, B, out.ctypes.data,
                                    ids.ctypes.data, sizes.ctypes.data, C.byref(ng))
        if rc:
            raise OracleError(rc, "rearrange")
        groups, o = [], 0
        for g in range(ng.value):
            groups.append(out[o:o + int(sizes[g])].copy())
            o += int(sizes[g])
        return ids[:ng.value].tolist(), groups

    # -- evaluation ------------------------------------------------------------
    def proxy_quality(self, tensors, recon):
        ck, keep = self._ckpt(tensors)
        r = np.ascontiguousarray(recon, np.float32)
        return self.lib.dqo_proxy_quality(C.byref(ck), r.ctypes.data)

    def estimate_compression(self, tensors, q: QState):
        ck, keep = self._ckpt(tensors)
        h = self._handle(q)
        try:
            return self.lib.dqo_estimate_compression(C.byref(ck), h)
        finally:
            self.lib.dqo_q_free(h)

    def config_hash(self, cfg: Config):
        return self.lib.dqo_config_hash(C.byref(cfg))

    def quantize_seed(self, seed, cfg: Config):
        return self.lib.dqo_quantize_seed(seed, C.byref(cfg))

    # -- ranker / trajectory -------------------------------------------------
    def ema_update(self, ema, g, beta=0.9):
        e = np.ascontiguousarray(ema, np.float32).copy()
        g = np.ascontiguousarray(g, np.float32)
        self.lib.dqo_ema_update(e.ctypes.data, g.ctypes.data, e.size, beta)
        return e

    def scores(self, w, ema=None):
        w = np.ascontiguousarray(w, np.float32)
        mag = np.zeros_like(w)
        sens = None if ema is None else np.zeros_like(w)
        e = None if ema is None else np.ascontiguousarray(ema, np.float32)
        self.lib.dqo_scores(w.ctypes.data, None if e is None else e.ctypes.data, w.size,
                            mag.ctypes.data, None if sens is None else sens.ctypes.data)
        return mag, sens

    def default_layout(self, params):
        numel = np.zeros(9, np.uint64)
        types = np.zeros(9, np.uint8)
        ranks = np.zeros(9, np.uint8)
        dims = np.zeros(18, np.uint64)
        self.lib.dqo_default_layout(params, numel.ctypes.data, types.ctypes.data,
                                    ranks.ctypes.data, dims.ctypes.data)
        names = ["model.embed.weight", "model.layer0.attn.qkv.weight",
                 "model.layer0.attn.out.weight", "model.layer0.mlp.fc1.weight",
                 "model.layer0.mlp.fc2.weight", "model.stem.conv.weight",
                 "model.layer0.norm.weight", "model.layer0.mlp.fc1.bias", "model.output.weight"]
        out = []
        for i in range(9):
            shape = tuple(int(d) for d in dims[2 * i:2 * i + int(ranks[i])])
            out.append((names[i], int(types[i]), shape))
        return out

    def generate_trajectory(self, layout, steps, seed, lr0=0.1, decay=0.9, noise=0.05):
        """layout: list of (name, type, shape). Returns list of (weights, grads) tensor lists."""
        numel = np.array([int(np.prod(s, dtype=np.uint64)) for _, _, s in layout], np.uint64)
        N = int(numel.sum())
        w = np.zeros((steps, N), np.float32)
        g = np.zeros((steps, N), np.float32)
        rc = self.lib.dqo_generate_trajectory(numel.ctypes.data, len(layout), steps, lr0, decay,
                                              noise, seed, w.ctypes.data, g.ctypes.data)
        if rc:
            raise OracleError(rc, "trajectory")
        out = []
        for s in range(steps):
            ws, gs, o = [], [], 0
            for (name, lt, shape), n in zip(layout, numel):
                n = int(n)
                ws.append(Tensor(name, lt, tuple(shape), w[s, o:o + n]))
                gs.append(Tensor(name, lt, tuple(shape), g[s, o:o + n]))
                o += n
            out.append((ws, gs))
        return out


def _record_layout(rec: bytes):
    """Walk a DQDR record header for tensor names/types/shapes (codec.cpp:462-511)."""
    import struct
    pos = 4 + 4 + 1 + 8 + 8 + 4 + (4 + 4 + 8 + 8 + 1 + 8 + 8) + 8
    nlt = rec[pos]
    pos += 1
    for _ in range(nlt):
        ln = struct.unpack_from("<I", rec, pos + 1)[0]
        pos += 5 + 4 * ln
    nt = struct.unpack_from("<I", rec, pos)[0]
    pos += 4

    def uv():
        nonlocal pos
        v = s = 0
        while True:
            b = rec[pos]
            pos += 1
            v |= (b & 0x7F) << s
            if not b & 0x80:
                return v
            s += 7

    names, types, shapes = [], [], []
    for _ in range(nt):
        nl = struct.unpack_from("<H", rec, pos)[0]
        pos += 2
        names.append(rec[pos:pos + nl].decode())
        pos += nl
        types.append(rec[pos])
        rank = rec[pos + 1]
        pos += 2
        shapes.append(tuple(struct.unpack_from("<%dQ" % rank, rec, pos)))
        pos += 8 * rank
        npro = uv()
        for _ in range(npro):
            uv()
            pos += 2
        ng = uv()
        for _ in range(ng):
            uv(), uv(), uv()
            ts = uv()
            for _ in range(ts):
                uv()
                pos += 1
            nb = uv()
            pos += nb
    return names, types, shapes


def _record_step_cfg(rec: bytes):
    import struct
    step = struct.unpack_from("<Q", rec, 17)[0]
    bins, eb, pf, tf, m, sg, al = struct.unpack_from("<IIddBdd", rec, 29)
    return step, (bins, eb, pf, tf, m, sg, al)


_ORACLE = None


def get() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = Oracle()
    return _ORACLE
