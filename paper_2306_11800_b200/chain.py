"""Device-resident record chain: ``Chain::append/restore`` (src/chain.cpp:86-154)
with the previous quantized state kept in HBM.

The drop-in ``dqt.Chain`` (csrc/host/chain.cpp) takes host ``QuantizedCheckpoint``
values, so every append uploads the base and target levels again.  ``DeviceChain``
takes the engine's device states (``Engine.quantize`` / ``compress_step`` /
``ChainCompressor`` outputs): the delta base is the state of the previous append,
already in HBM, and only the record bytes cross PCIe (D2H), once.  The directory
layout is the reference's, byte for byte: ``manifest.txt`` ("# dqt-chain <id>"
header, then "step,FULL|DELTA,file,base" lines) and one DQDR file
``rec-%012d.dqdr`` per step, FULL every ``full_every`` records — the reference
``Chain`` (and the drop-in) open, verify and restore it.  ``restore`` replays the
records on the device (``Engine.decode_record``).
"""
from __future__ import annotations

import os
import struct
import secrets
from dataclasses import dataclass
from typing import Optional

from . import engine as E

_MANIFEST = "manifest.txt"
_HEADER = "# dqt-chain "


class ChainError(E.EngineError):
    """dqt::Error family raised by the chain (status codes as include/dqtg.h)."""

    def __init__(self, status, msg):
        super().__init__(status, msg)


def _corrupt(msg):
    return ChainError(16, msg)  # ChainCorrupt


@dataclass
class ChainEntry:
    """include/dqt/chain.hpp:13-18"""
    step: int
    full: bool
    filename: str
    base_step: int = 0


class DeviceChain:
    def __init__(self, engine: E.Engine, directory: str, full_every: int = 50):
        """Chain::open (src/chain.cpp:22-70): creates the directory and manifest, or
        loads and validates an existing manifest."""
        if full_every == 0:
            raise ChainError(1, "full_every must be >= 1")
        self.engine = engine
        self.dir = directory
        self.full_every = int(full_every)
        self.entries: list[ChainEntry] = []
        self._prev: Optional[E.DevState] = None  # state of the last append (HBM)
        os.makedirs(directory, exist_ok=True)
        mp = os.path.join(directory, _MANIFEST)
        if not os.path.exists(mp):
            self.id = secrets.token_hex(8)
            with open(mp, "w") as f:
                f.write(_HEADER + self.id + "\n")
            return
        with open(mp) as f:
            lines = f.read().split("\n")
        if not lines or not lines[0].startswith(_HEADER):
            raise _corrupt("manifest missing chain header")
        self.id = lines[0][len(_HEADER):]
        for ln, line in enumerate(lines[1:], start=2):
            if not line:
                continue
            parts = line.split(",")
            if len(parts) < 3:
                raise _corrupt(f"manifest line {ln} malformed")
            step, kind, fname = int(parts[0]), parts[1], parts[2]
            base = parts[3] if len(parts) > 3 else ""
            if kind == "FULL":
                e = ChainEntry(step, True, fname)
            elif kind == "DELTA":
                if not base:
                    raise _corrupt(f"manifest line {ln} missing base")
                e = ChainEntry(step, False, fname, int(base))
            else:
                raise _corrupt(f"manifest line {ln} has kind {kind}")
            if self.entries and e.step <= self.entries[-1].step:
                raise _corrupt(f"manifest steps not strictly ascending at step {e.step}")
            if not self.entries and not e.full:
                raise _corrupt("first chain entry must be FULL")
            if not e.full and e.base_step != self.entries[-1].step:
                raise _corrupt(f"delta at step {e.step} does not chain from the preceding entry")
            self.entries.append(e)

    # -------------------------------------------------------------- queries
    def empty(self):
        return not self.entries

    def latest_step(self):
        if not self.entries:
            raise ChainError(1, "chain is empty")  # UnknownStep
        return self.entries[-1].step

    def record_path(self, e: ChainEntry):
        return os.path.join(self.dir, e.filename)

    # -------------------------------------------------------------- append
    def _next_is_full(self):
        since_full = 0
        for e in reversed(self.entries):
            if e.full:
                break
            since_full += 1
        return not self.entries or since_full + 1 >= self.full_every

    def _commit(self, step, full, rec: bytes):
        e = ChainEntry(step, full, f"rec-{step:012d}.dqdr",
                       0 if full else self.entries[-1].step)
        with open(self.record_path(e), "wb") as f:
            f.write(rec)
        with open(os.path.join(self.dir, _MANIFEST), "a") as f:
            f.write(f"{e.step},{'FULL' if e.full else 'DELTA'},{e.filename},"
                    f"{'' if e.full else e.base_step}\n")
        self.entries.append(e)
        return e

    def _base_state(self):
        base_step = self.entries[-1].step
        if self._prev is not None and int(self._prev.info().step) == base_step:
            return self._prev
        return self.restore(base_step)

    def append(self, state: E.DevState, quality_delta=0.0) -> ChainEntry:
        """Chain::append (src/chain.cpp:86-129) of a device state."""
        step = int(state.info().step)
        if self.entries and step <= self.entries[-1].step:
            raise ChainError(1, f"append step {step} not after {self.entries[-1].step}")
        full = self._next_is_full()
        rec = self.engine.encode_record(state, None if full else self._base_state(), quality_delta)
        e = self._commit(step, full, rec)
        self._prev = state
        return e

    def append_snapshots(self, compressor, ckpts, cfg, seed, steps, quality_delta=0.0, host=None):
        """Quantize + append a series of snapshots through the pipelined worker pool
        (pipeline.ChainCompressor): records stream back from the workers and are
        committed in step order; FULL records start a new pipelined segment."""
        steps = [int(s) for s in steps]
        if self.entries and steps and steps[0] <= self.entries[-1].step:
            raise ChainError(1, f"append step {steps[0]} not after {self.entries[-1].step}")
        k = 0
        while k < len(steps):
            full = self._next_is_full()
            since_full = 0
            for e in reversed(self.entries):
                if e.full:
                    break
                since_full += 1
            # records until (and excluding) the next FULL one
            room = self.full_every - since_full - 1 if not full else self.full_every
            n = max(1, min(len(steps) - k, room))
            base = None if full else self._base_state()
            recs = {}

            def grab(i, r):
                import numpy as np

                buf = np.empty(E.LIB.dqtg_record_size(r), np.uint8)
                E._check(E.LIB.dqtg_record_copy(r, buf.ctypes.data))
                recs[i] = buf.tobytes()

            seg = ckpts[k:k + n]
            last = compressor.run(seg, cfg, seed, steps[k:k + n], base=base, quality=quality_delta,
                                  on_record=grab, host=host)
            for i in range(n):
                self._commit(steps[k + i], full and i == 0, recs[i])
            self._prev = last
            k += n
        return self.entries[-1] if self.entries else None

    # -------------------------------------------------------------- restore
    def restore(self, step) -> E.DevState:
        """Chain::restore (src/chain.cpp:131-154): replay from the last FULL record
        on the device."""
        idx = next((i for i, e in enumerate(self.entries) if e.step == step), None)
        if idx is None:
            raise ChainError(1, f"step {step} not in chain")  # UnknownStep
        start = idx
        while not self.entries[start].full:
            if start == 0:
                raise _corrupt(f"no FULL record precedes step {step}")
            start -= 1
        ents = self.entries[start:idx + 1]
        recs = []
        for e in ents:
            with open(self.record_path(e), "rb") as f:
                recs.append(f.read())
        # the decoded step is the record header's target step (bytes 17..24): the first
        # record whose header disagrees with the manifest ends the replay there -- after
        # the records up to it decoded, as the reference's sequential restore checks it
        stop = None
        for k, (e, rec) in enumerate(zip(ents, recs)):
            if len(rec) >= 25 and struct.unpack_from("<Q", rec, 17)[0] != e.step:
                stop = k
                break
        last = len(recs) if stop is None else stop + 1
        # a manifest FULL entry restarts the chain with no base (chain.cpp:146)
        state, k0 = None, 0
        for k in range(1, last + 1):
            if k == last or ents[k].full:
                state = self.engine.decode_chain(recs[k0:k], base=None if ents[k0].full else state)
                k0 = k
        if stop is not None:
            raise _corrupt(f"record step {int(state.info().step)} disagrees with manifest "
                           f"step {ents[stop].step}")
        return state

    def restore_latest(self) -> E.DevState:
        return self.restore(self.latest_step())
