"""Helpers around the reference compiled from its own sources (oracle/_ref).

TEST INFRASTRUCTURE ONLY.  ``dqtref`` is the unmodified reference pybind module
(bindings/py_module.cpp) built by ``make -C oracle ref`` with the namespace
renamed (-Ddqt=dqtref) so it can share a process with the product module.
"""
from __future__ import annotations

import os
import sys

import numpy as np

from .oracle import QState, Tensor

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "dqtref"))


def load():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import dqtref  # noqa: E402

    return dqtref


def checkpoint(tensors, step=0):
    d = load()
    c = d.Checkpoint()
    c.step = step
    for t in tensors:
        c.add_tensor(t.name, np.ascontiguousarray(t.data, np.float32).reshape(t.shape),
                     d.LayerType(int(t.type)))
    return c


def config(cfg_tuple):
    d = load()
    b, eb, pf, tf, m, s, a = cfg_tuple
    return d.QuantConfig(bins=b, embed_bins=eb, prune_frac=pf, protect_frac=tf,
                         metric=d.PruneMetric(int(m)), sigma=s, alpha=a)


def qstate(q) -> QState:
    d = load()
    cfg = q.config
    cft = (cfg.bins, cfg.embed_bins, cfg.prune_frac, cfg.protect_frac, int(cfg.metric), cfg.sigma,
           cfg.alpha)
    cbs = [np.asarray(q.codebook(d.LayerType(lt)), np.float32) for lt in range(7)]
    names, types, shapes, levels, pp, pv = [], [], [], [], [], []
    for t in q.tensors:
        names.append(t.name)
        types.append(int(t.type))
        shapes.append(tuple(t.shape))
        levels.append(np.asarray(t.levels, np.uint16).ravel().copy())
        pp.append(np.array([e.pos for e in t.protected_values], np.uint64))
        # the binding exposes the bf16 value as a float; recover the bits
        vals = np.array([e.value for e in t.protected_values], np.float32)
        pv.append((vals.view(np.uint32) >> 16).astype(np.uint16))
    return QState(int(q.step), cft, cbs, names, types, shapes, levels, pp, pv)


def tensors_of(ck):
    return [Tensor(t.name, int(t.type), tuple(t.shape), np.asarray(t.data, np.float32).ravel())
            for t in ck.tensors]


def payload_bytes(base: QState, target: QState, variant: int) -> int:
    """payload_bytes_pe / _rle / _he of the reference (oracle/ref_extra.cpp)."""
    import ctypes as C

    lib = C.CDLL(os.path.join(REF_DIR, "libdqtref_extra.so"))
    fn = lib.ref_payload_bytes
    fn.restype = C.c_uint64
    nt = len(target.levels)
    types = np.array([int(t) for t in target.types] or [0], np.uint8)
    numel = np.array([np.asarray(lv).size for lv in target.levels] or [0], np.uint64)
    keep = []

    def ptrs(q):
        arr = [np.ascontiguousarray(np.asarray(lv).ravel(), np.uint16) for lv in q.levels]
        keep.append(arr)
        return (C.c_void_p * max(nt, 1))(*[a.ctypes.data for a in arr])

    def cbl(q):
        a = np.array([len(c) for c in q.codebooks], np.uint32)
        keep.append(a)
        return a.ctypes.data

    return int(fn(int(variant), nt, C.c_void_p(types.ctypes.data), C.c_void_p(numel.ctypes.data),
                  ptrs(base), C.c_void_p(cbl(base)), ptrs(target), C.c_void_p(cbl(target))))
