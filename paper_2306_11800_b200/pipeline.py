"""Pipelined delta chain over the native worker pool (dqtg_pipe_*, csrc/engine/pipe.cu).

``Chain::append`` (chain.cpp:86-129) compresses a series of checkpoints where
each record depends on the previous quantized state.  Quantization of a
snapshot depends only on the snapshot (and the EMA), so every step's quantize
can run as soon as its weights are in HBM; only the encode of step k waits for
the quantized state of step k-1.  Step k runs on worker k mod W (one engine,
CUDA stream and C++ host thread each):

    worker 0:  [copy 0] quantize 0 ......... encode 0|base   [copy 2] quantize 2 ...
    worker 1:     [copy 1] quantize 1 ...... wait q0 > encode 1|0     [copy 3] ...

While one worker blocks on a host read-back or a host->device copy, the other
keeps the GPU fed, and the few-CTA phases (k-means restarts, per-group Huffman)
overlap the streaming passes of the other worker.  Records are identical to
sequential ``compress_step``.
"""
from __future__ import annotations

from . import engine as E


class ChainCompressor:
    def __init__(self, device=0, workers=2, stream=None, comms=None, n_tensors_total=0):
        """``stream`` (a cudaStream_t as int, optional): every run forks from and joins
        into it, so CUDA events recorded on it bracket the run's device work.
        ``comms`` (one engine Comm per worker, distributed.make_comm): every rank runs
        the chain over its tensor shard; records reach ``on_record`` on rank 0 only."""
        self.device = device
        self.nw = max(1, int(workers))
        self.pipe = E.Pipe(device, self.nw)
        if stream:
            self.pipe.set_stream(stream)
        if comms:
            self.pipe.set_comms(comms, n_tensors_total)
        self._eng = None

    @property
    def eq(self):
        """Engine owning checkpoints made by checkpoint() (and nominal owner of returned states)."""
        if self._eng is None:
            self._eng = E.Engine(self.device)
        return self._eng

    @property
    def launches(self):
        return self.pipe.launches

    def checkpoint(self, names, types, shapes):
        """A device-resident snapshot (any worker reads it)."""
        return E.DevCheckpoint(self.eq, names, types, shapes)

    def run(self, ckpts, cfg, seed, steps, base=None, quality=0.0, on_record=None,
            host=None):
        """Compress snapshot k at ``steps[k]`` as a delta chain from ``base`` (None:
        the first record is FULL).  ``ckpts[k]`` is a DevCheckpoint (device resident,
        read in place by the worker; its own EMA gives snapshot k's sensitivity
        scores, and either every checkpoint carries an EMA or none does), or with
        ``host`` = (names, types, shapes, ema) a list of per-tensor host arrays /
        pointers (copied into HBM by the worker; ``ema`` is shared by the series).  ``on_record(k, handle)`` runs on a worker thread with the record
        handle (valid during the call; calls may arrive out of step order).  Returns
        the last quantized state."""
        if not ckpts:
            return base
        if host is not None:
            names, types, shapes, ema = host
            snaps = ckpts
        else:
            c0 = ckpts[0]
            names, types, shapes = c0.meta.names, c0.meta.types, c0.meta.shapes
            nt = len(names)
            snaps = [[c.weights_dev + 4 * c.tensor_offset(i) for i in range(nt)] for c in ckpts]
            has = [bool(c.ema_dev) for c in ckpts]
            if any(has) and not all(has):
                raise ValueError("either every checkpoint of the series carries an EMA or none does")
            emas = None
            if all(has):
                emas = [[c.ema_dev + 4 * c.tensor_offset(i) for i in range(nt)] for c in ckpts]
            return self.pipe.run(names, types, shapes, snaps, cfg, seed, steps, None, base, quality,
                                 on_record, engine=self.eq, emas=emas)
        return self.pipe.run(names, types, shapes, snaps, cfg, seed, steps, ema, base, quality,
                             on_record, engine=self.eq)

