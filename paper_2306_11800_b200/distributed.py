"""Tensor-sharded compress + delta-encode across the GPUs of one box.

One process per GPU (torchrun), NCCL for the only two real exchanges of the path:
the score histograms (pass A) and the QUANTIZE-value histograms (pass B) must be
global so that every rank derives the same thresholds and codebooks
(``torch.distributed.all_reduce`` of u64 counts, exact and order independent).
After that each rank quantizes and encodes its own tensors; the record of the
whole checkpoint is the rank-0 prefix, the ranks' tensor blocks in tensor order,
and the CRC-32 combined from the per-rank CRCs (zlib ``crc32_combine`` rule) —
byte-identical to the single-GPU record.

The host-side pieces (``plan_shards``, ``crc32_combine``, ``assemble_record``)
are plain Python and are exercised with the gloo backend on CPU in
tests/test_distributed_cpu.py.
"""
from __future__ import annotations

import struct

import numpy as np

_POLY = 0xEDB88320


def _gf2_mult(a, b):
    p = 0
    m = 1 << 31
    while True:
        if a & m:
            p ^= b
            if (a & (m - 1)) == 0:
                break
        m >>= 1
        b = (b >> 1) ^ _POLY if b & 1 else b >> 1
    return p


_X2N = [1 << 30]
for _k in range(1, 32):
    _X2N.append(_gf2_mult(_X2N[-1], _X2N[-1]))


def _x2nmodp(n, k):
    p = 1 << 31
    while n:
        if n & 1:
            p = _gf2_mult(_X2N[k & 31], p)
        n >>= 1
        k += 1
    return p


def crc32_combine(crc1: int, crc2: int, len2: int) -> int:
    """CRC-32 of A||B from crc(A), crc(B), len(B) (GF(2) shift by 8*len2 bits)."""
    if len2 == 0:
        return crc1
    return _gf2_mult(_x2nmodp(len2, 3), crc1) ^ crc2


def plan_shards(numel, world):
    """Contiguous tensor ranges per rank, greedily balanced by element count.

    Contiguity keeps every rank's record blocks a contiguous slice of the record."""
    numel = [int(n) for n in numel]
    total = sum(numel)
    bounds, start, acc = [], 0, 0
    for r in range(world):
        target = total * (r + 1) / world
        end = start
        while end < len(numel) and (r == world - 1 or acc + numel[end] / 2 <= target):
            acc += numel[end]
            end += 1
        bounds.append((start, end))
        start = end
    return bounds


def assemble_record(prefix: bytes, bodies, crcs, stream_lens) -> bytes:
    """Full DQDR record from rank 0's prefix and every rank's (body, crc, level-stream bytes)."""
    crc = None
    for c, n in zip(crcs, stream_lens):
        crc = c if crc is None else crc32_combine(crc, c, n)
    return bytes(prefix) + b"".join(bytes(b) for b in bodies) + struct.pack("<I", crc or 0)


class RemoteRankError(RuntimeError):
    """Another rank failed in a sharded step; raised on every rank."""


def _agree(err, group, device):
    """Collective status check before a data collective: a rank whose local stage
    raised would otherwise leave the others blocked in the next all_reduce.  Every
    rank re-raises (its own error, or RemoteRankError naming the failed ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        if err is not None:
            raise err
        return
    flag = torch.tensor([0 if err is None else 1], dtype=torch.int64, device=device)
    flags = [torch.zeros_like(flag) for _ in range(dist.get_world_size(group))]
    dist.all_gather(flags, flag, group=group)
    if err is not None:
        raise err
    bad = [r for r, x in enumerate(flags) if int(x.item())]
    if bad:
        raise RemoteRankError(f"sharded step failed on rank(s) {bad}")


def make_comm(engine, group=None):
    """The engine library's own NCCL communicator over the ranks of ``group``: rank 0
    makes the id, torch.distributed broadcasts it (any backend)."""
    import torch.distributed as dist

    from . import engine as E

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    box = [E.Comm.unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(box, src=0, group=group)
    return E.Comm(engine, box[0], world, rank)


def compress_sharded(engine, ckpt, cfg, seed, step, base_state, *, group=None, device=None,
                     quality=0.0, n_tensors_total=None, gather_record=False, comm=None):
    """One compress+delta step of a tensor-sharded checkpoint.

    ``ckpt`` holds this rank's tensors.  Returns (state, record_bytes_or_None,
    stats): the state stays on this GPU for the next step; with
    ``gather_record`` rank 0 receives the assembled record.

    With ``comm`` (an engine Comm, see make_comm) the whole step runs in the engine
    library (dqtg_compress_sharded): NCCL all-reduces on the engine stream and the
    record gathered into rank 0's device memory.  Without it the exchanges go through
    torch.distributed (any backend; the CPU tests use gloo)."""
    import torch
    import torch.distributed as dist

    from . import engine as E

    if comm is not None:
        state, rec = engine.compress_sharded(comm, ckpt, cfg, seed, step, base_state, quality,
                                             n_tensors_total or 0)
        stats = {"record_bytes_local": None, "comm": "dqtg_comm (NCCL)"}
        out = None
        if rec is not None:
            size = E.LIB.dqtg_record_size(rec)
            stats["record_bytes"] = size
            if gather_record:
                buf = np.empty(size, np.uint8)
                E._check(E.LIB.dqtg_record_copy(rec, buf.ctypes.data))
                out = buf.tobytes()
            E.LIB.dqtg_record_destroy(rec)
        return state, out, stats

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = device or torch.device("cuda", torch.cuda.current_device())
    n_s = engine.shard_hist_len(cfg, 0)
    n_v = engine.shard_hist_len(cfg, 1)
    score = torch.empty(n_s, dtype=torch.int64, device=dev)
    value = torch.empty(n_v, dtype=torch.int64, device=dev)
    def local(fn):
        try:
            fn()
            engine.sync()
            return None
        except Exception as ex:  # noqa: BLE001 - re-raised on every rank by _agree
            return ex

    _agree(local(lambda: engine.shard_stage1(ckpt, cfg, score.data_ptr())), group, dev)
    if world > 1:
        dist.all_reduce(score, group=group)
    _agree(local(lambda: engine.shard_stage2(ckpt, cfg, score.data_ptr(), value.data_ptr())),
           group, dev)
    if world > 1:
        dist.all_reduce(value, group=group)
    box = []
    _agree(local(lambda: box.append(engine.shard_stage3(ckpt, cfg, seed, step,
                                                        value.data_ptr()))), group, dev)
    state = box[0]
    # global alphabet and tensor count
    info = state.info()
    lv = [info.max_levels, base_state.info().max_levels if base_state is not None else 0]
    meta = torch.tensor([max(lv), len(ckpt.meta.names)], dtype=torch.int64, device=dev)
    if world > 1:
        mx = meta[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        cnt = meta[1:].clone()
        dist.all_reduce(cnt, group=group)
        meta = torch.cat([mx, cnt])
    gB = max(2, int(meta[0]))
    gnt = int(meta[1]) if n_tensors_total is None else n_tensors_total
    rec, body_off = engine.encode_record_shard(state, base_state, quality, gB, gnt)
    size = E.LIB.dqtg_record_size(rec)
    stats = {"record_bytes_local": size, "body_offset": body_off, "B": gB}
    out = None
    if gather_record:
        buf = np.empty(size, np.uint8)
        E._check(E.LIB.dqtg_record_copy(rec, buf.ctypes.data))
        body = buf[body_off:size - 4].tobytes()
        crc = struct.unpack("<I", buf[size - 4:].tobytes())[0]
        stream = 2 * int(info.param_count)
        parts = [None] * world
        if world > 1:
            dist.all_gather_object(parts, (body, crc, stream), group=group)
        else:
            parts = [(body, crc, stream)]
        if not dist.is_initialized() or dist.get_rank(group) == 0:
            out = assemble_record(buf[:body_off].tobytes(), [p[0] for p in parts],
                                  [p[1] for p in parts], [p[2] for p in parts])
    E.LIB.dqtg_record_destroy(rec)
    return state, out, stats


def assign_configs(m, world):
    """Round-robin split of m candidate configs over the ranks (config i on rank
    i mod world): neighbouring configs of a guided-search batch (search.cpp:247-296,
    387-482) have similar cost, so round-robin balances the ranks."""
    return [list(range(r, m, world)) for r in range(world)]


def eval_batch_sharded(evaluate, cfgs, seeds, *, group=None):
    """Batched candidate evaluation (EvalCache::prefetch, search.cpp:174-204) spread
    over the ranks of one box: each rank evaluates its share with its own engine
    (``evaluate(cfgs, seeds) -> (quality[], est[])``, e.g. ``Engine.eval_batch``
    bound to the rank's copy of the checkpoint), and the results are all-gathered
    so every rank holds the whole batch in the original order (the search control
    then continues identically on every rank)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    mine = assign_configs(len(cfgs), world)[rank]
    err = None
    part = (mine, [], [])
    try:
        if mine:
            q, e = evaluate([cfgs[i] for i in mine], [seeds[i] for i in mine])
            part = (mine, [float(x) for x in q], [float(x) for x in e])
    except Exception as ex:  # noqa: BLE001 - every rank learns about it below
        err = ex
        part = (mine, None, f"{type(ex).__name__}: {ex}")
    parts = [None] * world
    if world > 1:
        dist.all_gather_object(parts, part, group=group)
    else:
        parts = [part]
    if err is not None:
        raise err
    bad = [(r, p[2]) for r, p in enumerate(parts) if p[1] is None]
    if bad:
        raise RemoteRankError(f"candidate evaluation failed on rank(s): {bad}")
    quality = [0.0] * len(cfgs)
    est = [0.0] * len(cfgs)
    for idx, q, e in parts:
        for j, i in enumerate(idx):
            quality[i], est[i] = q[j], e[j]
    return quality, est


def sharded_evaluator(inner=None, *, group=None):
    """Search control across the ranks: an Evaluator for the drop-in
    ``guided_exhaustive_search`` / ``delta_neighborhood_search`` (search.cpp:247-296,
    387-482) whose ``evaluate_batch`` -- called once per EvalCache::prefetch batch
    (search.cpp:174-204) -- evaluates this rank's round-robin share with ``inner``
    (default: the device ProxyEvaluator) and all-gathers the results.  Every rank runs
    the same search with the same inputs, so every rank sees identical batches,
    identical results and reaches the same outcome; the evaluation work is split
    ``world`` ways."""
    from . import dqt

    inner = inner if inner is not None else dqt.ProxyEvaluator()

    class ShardedEvaluator(dqt.Evaluator):
        def __init__(self):
            super().__init__()
            self.inner = inner

        def evaluate(self, checkpoint, scores, config, seed):
            return self.inner.evaluate(checkpoint, scores, config, seed)

        def evaluate_batch(self, checkpoint, scores, configs, seeds, parallelism=1):
            def run(cfgs, sds):
                res = self.inner.evaluate_batch(checkpoint, scores, cfgs, sds, parallelism)
                return [r.quality_delta for r in res], [r.est_compression for r in res]

            q, e = eval_batch_sharded(run, list(configs), list(seeds), group=group)
            return [dqt.EvalResult(a, b) for a, b in zip(q, e)]

    return ShardedEvaluator()
