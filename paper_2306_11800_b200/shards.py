"""Tensor-sharded Chain::append on ONE engine, for checkpoints larger than one GPU's
working set (BASELINE.json configs[3..4]: GPT-2 XL sharded 2/4/8 ways, Llama-3-8B).

The multi-GPU path (distributed.py, comm.cu) splits the tensors into contiguous
shards (plan_shards) and has exactly two exchanges per step: the score histograms
after pass A and the QUANTIZE-value histograms after pass B are summed over the
ranks, so every rank derives the same thresholds and codebooks
(quantize.cpp:34-92, 256-325).  Here the shards are processed one after another on
one engine and the two exchanges become sums over the shards; each shard's data is
(re)loaded by a caller callback before each of its three stages, so only one
shard's inputs need to be resident at a time (C5: 32 GB of weights + 32 GB of EMA).

Every shard's record is a complete DQDR record of its tensors (global alphabet,
encode_record_shard with its own tensor count), so it is decoded on its own for the
round-trip check.  Patching the tensor count of shard 0's prefix and concatenating
the bodies with the CRC-32 combined (distributed.assemble_record) gives the record
of the whole checkpoint, byte-identical to the single-engine record
(codec.cpp:398-460) -- tests/test_c4c5_gpu.py checks this at GPT-2-XL size.
"""
from __future__ import annotations

import struct
import time

import numpy as np

from . import distributed as D
from . import engine as E


class LocalShardedChain:
    def __init__(self, engine, names, types, shapes, n_shards, cfg, seed=1, device=None,
                 release_inputs=True):
        import torch

        self.torch = torch
        self.eng = engine
        self.cfg = cfg
        self.seed = seed
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        numel = [int(np.prod(s, dtype=np.int64)) for s in shapes]
        self.plan = D.plan_shards(numel, n_shards)
        self.ck = [E.DevCheckpoint(engine, names[a:b], types[a:b], shapes[a:b])
                   for a, b in self.plan]
        self.nt = len(names)
        self.prev = [None] * len(self.plan)
        # free each shard's inputs after every stage: one shard's weights + EMA resident
        self.release_inputs = release_inputs
        self.t_engine = 0.0  # seconds spent in engine calls (loads excluded)

    def _timed(self, fn, *a):
        # the histogram sums (torch ops) are complete before the engine reads them,
        # whichever stream the engine runs on
        self.torch.cuda.current_stream(self.dev).synchronize()
        t = time.perf_counter()
        r = fn(*a)
        self.eng.sync()
        self.t_engine += time.perf_counter() - t
        return r

    def _done(self, ck):
        if self.release_inputs:
            ck.release()

    def step(self, step, load, quality=0.0, keep_records=True, check_roundtrip=True):
        """One Chain::append of the whole checkpoint.  ``load(s, ck)`` fills shard s's
        weights and EMA (``ck.set_weights`` / ``ck.set_ema``) for this step; it is called
        once per stage (three times per shard).  Returns (per-shard records or sizes,
        round-trip results)."""
        torch, eng, cfg = self.torch, self.eng, self.cfg
        n_s, n_v = eng.shard_hist_len(cfg, 0), eng.shard_hist_len(cfg, 1)
        score = torch.zeros(n_s, dtype=torch.int64, device=self.dev)
        value = torch.zeros(n_v, dtype=torch.int64, device=self.dev)
        tmp = torch.empty(max(n_s, n_v), dtype=torch.int64, device=self.dev)
        for s, ck in enumerate(self.ck):  # pass A; exchange 1: sum of score histograms
            load(s, ck)
            self._timed(eng.shard_stage1, ck, cfg, tmp.data_ptr())
            self._done(ck)
            score += tmp[:n_s]
        for s, ck in enumerate(self.ck):  # pass B; exchange 2: sum of value histograms
            load(s, ck)
            self._timed(eng.shard_stage2, ck, cfg, score.data_ptr(), tmp.data_ptr())
            self._done(ck)
            value += tmp[:n_v]
        states = []
        for s, ck in enumerate(self.ck):  # codebooks (identical for every shard) + pass C
            load(s, ck)
            states.append(self._timed(eng.shard_stage3, ck, cfg, self.seed, step, value.data_ptr()))
            self._done(ck)
        B = max(2, max(max(st.info().max_levels, 0 if p is None else p.info().max_levels)
                       for st, p in zip(states, self.prev)))
        records, roundtrip = [], []
        for s, st in enumerate(states):
            a, b = self.plan[s]
            rh, body_off = self._timed(eng.encode_record_shard, st, self.prev[s], quality, B, b - a)
            rec = E.Engine.record_bytes(rh)
            if check_roundtrip:
                t = time.perf_counter()
                dec = eng.decode_record(rec, base=self.prev[s])
                ok = eng.states_equal(dec, st)
                self.t_decode = getattr(self, "t_decode", 0.0) + time.perf_counter() - t
                roundtrip.append(ok)
                del dec
            records.append((rec, body_off) if keep_records else len(rec))
        self.prev = states
        return records, roundtrip

    def assemble(self, records):
        """The whole checkpoint's record from the shards' standalone records."""
        bodies, crcs, lens = [], [], []
        prefix = None
        for s, (rec, off) in enumerate(records):
            if prefix is None:  # shard 0's prefix with the global tensor count
                prefix = rec[:off - 4] + struct.pack("<I", self.nt)
            bodies.append(rec[off:len(rec) - 4])
            crcs.append(struct.unpack("<I", rec[-4:])[0])
            lens.append(2 * int(sum(np.prod(sh, dtype=np.int64) for sh in self.ck[s].meta.shapes)))
        return D.assemble_record(prefix, bodies, crcs, lens)
