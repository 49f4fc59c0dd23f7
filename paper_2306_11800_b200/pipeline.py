"""Pipelined delta chain: a pool of workers, one CUDA stream + engine each.

``Chain::append`` (chain.cpp:86-129) compresses a series of checkpoints where
each record depends on the previous quantized state.  Quantization of a
snapshot depends only on the snapshot (and the EMA), so every step's quantize
can run as soon as its weights are in HBM; only the encode of step k waits for
the quantized state of step k-1.  Step k runs on worker k mod W:

    worker 0:  [h2d 0] quantize 0 ......... encode 0|base   [h2d 3] quantize 3 ...
    worker 1:     [h2d 1] quantize 1 ...... wait q0 > encode 1|0     [h2d 4] ...
    worker 2:        [h2d 2] quantize 2 ... wait q1 > encode 2|1 ...

With W streams in flight the GPU always has queued work while a worker blocks
on a host read-back (record size, overflow counts) or a host->device copy, and
the few-CTA phases (k-means restarts, per-group Huffman) overlap the streaming
passes of the other workers.  Cross-stream order is explicit: encode(k) waits
on the CUDA event recorded after quantize(k-1); a state is released only after
both encodes that read it (as target and as base) have completed on the device.
Host calls into the engines release the GIL (ctypes).  Records are identical to
sequential ``compress_step``.
"""
from __future__ import annotations

import threading

from . import engine as E


class ChainCompressor:
    def __init__(self, device=0, workers=2):
        import torch

        self.torch = torch
        self.device = device
        self.nw = max(1, int(workers))
        self.streams = [torch.cuda.Stream(device) for _ in range(self.nw)]
        self.engines = [E.Engine(device, s.cuda_stream) for s in self.streams]
        self._host_ck = [None] * self.nw  # per-worker device checkpoint for host inputs

    # back-compat names: the first worker's engine / stream
    @property
    def eq(self):
        return self.engines[0]

    @property
    def launches(self):
        return sum(e.launches for e in self.engines)

    def checkpoint(self, names, types, shapes):
        """Device-resident checkpoints live on the first engine (any worker may read them)."""
        return E.DevCheckpoint(self.engines[0], names, types, shapes)

    def run(self, ckpts, cfg, seed, steps, base=None, quality=0.0, on_record=None,
            host=None):
        """Compress snapshot k (``ckpts[k]``, a DevCheckpoint, or with ``host`` =
        (names, types, shapes, ema_ptrs) a list of per-tensor host arrays) at
        ``steps[k]`` as a delta chain starting from ``base`` (None: the first record
        is FULL).  ``on_record(k, handle)`` runs on the worker thread with the record
        handle (valid during the call; calls may arrive out of step order).  Returns
        the last quantized state."""
        torch = self.torch
        n = len(ckpts)
        states = [None] * n
        q_ev = [None] * n
        q_ready = [threading.Event() for _ in range(n)]
        users = [0] * n  # encodes done that read state k (target + base)
        lock = threading.Lock()
        err = []

        def release(k):
            with lock:
                users[k] += 1
                if users[k] == 2 and k != n - 1:
                    states[k] = None

        def worker(w):
            eng, stream = self.engines[w], self.streams[w]
            try:
                for k in range(w, n, self.nw):
                    if err:
                        return
                    ck = ckpts[k]
                    if host is not None:  # host->device copy on this worker's stream
                        if self._host_ck[w] is None:
                            names, types, shapes, ema = host
                            c = E.DevCheckpoint(eng, names, types, shapes)
                            c.set_ema(ema)
                            self._host_ck[w] = c
                        self._host_ck[w].set_weights(ck)
                        ck = self._host_ck[w]
                    st = eng.quantize(ck, cfg, seed, steps[k])
                    ev = torch.cuda.Event()
                    ev.record(stream)
                    states[k], q_ev[k] = st, ev
                    q_ready[k].set()
                    if k > 0:
                        q_ready[k - 1].wait()
                        if err:
                            return
                        stream.wait_event(q_ev[k - 1])
                        prev = states[k - 1]
                    else:
                        prev = base
                    r = eng.encode_record_handle(st, prev, quality)
                    try:
                        if on_record is not None:
                            on_record(k, r)
                    finally:
                        E.LIB.dqtg_record_destroy(r)
                    eng.sync()  # encode(k) done on the device: its inputs may be released
                    release(k)
                    if k > 0:
                        release(k - 1)
            except BaseException as ex:  # surfaced to the caller
                err.append(ex)
                for ev in q_ready:
                    ev.set()

        ths = [threading.Thread(target=worker, args=(w,), daemon=True) for w in range(self.nw)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if err:
            raise err[0]
        return states[n - 1] if n else base

    def sync(self):
        for e in self.engines:
            e.sync()
