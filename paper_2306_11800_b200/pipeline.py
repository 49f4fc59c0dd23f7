"""Pipelined delta chain: quantize(snapshot i+1) overlaps encode(snapshot i).

``Chain::append`` (chain.cpp:86-129) compresses a series of checkpoints where
each record depends on the previous quantized state.  Quantization of the next
snapshot does not depend on the current record, so two engines on two CUDA
streams run the two halves concurrently:

    stream Q:  quantize(1)  quantize(2)  quantize(3) ...
    stream E:               encode(1|0)  encode(2|1)  encode(3|2) ...

The k-means of quantize (a latency-bound, few-CTA phase) then hides behind the
bandwidth-bound codec of the previous step.  Ordering is explicit: encode(i)
waits on the CUDA event recorded after quantize(i); a state is released on the
quantize stream only after the encode that reads it as a base has finished.
Host calls into the engines release the GIL (ctypes), so one thread per engine
keeps both streams fed.  Results are identical to sequential compress_step.
"""
from __future__ import annotations

import queue
import threading

from . import engine as E


class ChainCompressor:
    def __init__(self, device=0):
        import torch

        self.torch = torch
        self.device = device
        self.sq = torch.cuda.Stream(device)
        self.se = torch.cuda.Stream(device)
        self.eq = E.Engine(device, self.sq.cuda_stream)
        self.ee = E.Engine(device, self.se.cuda_stream)

    @property
    def launches(self):
        return self.eq.launches + self.ee.launches

    def checkpoint(self, names, types, shapes):
        """Checkpoints live on the quantize engine."""
        return E.DevCheckpoint(self.eq, names, types, shapes)

    def run(self, ckpts, cfg, seed, steps, base=None, quality=0.0, on_record=None):
        """Compress ckpts[k] at steps[k] as a delta chain starting from ``base``
        (None: the first record is FULL).  ``on_record(k, handle)`` is called on the
        encode thread with the record handle (valid during the call).  Returns the
        last quantized state."""
        torch = self.torch
        q = queue.Queue(maxsize=2)
        err = []

        def producer():
            try:
                for k, ck in enumerate(ckpts):
                    st = self.eq.quantize(ck, cfg, seed, steps[k])
                    ev = torch.cuda.Event()
                    ev.record(self.sq)
                    q.put((k, st, ev))
            except BaseException as ex:  # surfaced on the consumer side
                err.append(ex)
            finally:
                q.put(None)

        th = threading.Thread(target=producer, daemon=True)
        th.start()
        prev = base
        last = base
        try:
            while True:
                item = q.get()
                if item is None:
                    break
                k, st, ev = item
                self.se.wait_event(ev)
                r = self.ee.encode_record_handle(st, prev, quality)
                try:
                    if on_record is not None:
                        on_record(k, r)
                finally:
                    E.LIB.dqtg_record_destroy(r)
                done = torch.cuda.Event()
                done.record(self.se)
                self.sq.wait_event(done)  # prev may be freed (on stream Q) after this encode
                prev = st
                last = st
        finally:
            th.join()
        if err:
            raise err[0]
        return last

    def sync(self):
        self.eq.sync()
        self.ee.sync()
