"""Host logic of the tensor-sharded multi-GPU path on CPU (gloo, world size 2).

The device work of each rank is stood in for by the oracle; what is tested is
the product's distributed plumbing (paper_2306_11800_b200/distributed.py):
histogram all-reduce gives the whole-checkpoint histogram, contiguous tensor
shards, and the record assembled from per-rank tensor blocks + CRC combine is
byte-identical to the single-process record.
"""
import os
import socket
import struct
import zlib

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2306_11800_b200 import distributed as D
from tests.util import SMALL_LAYOUT, flat, make_tensors, perturb


def test_crc32_combine_matches_zlib():
    rng = np.random.default_rng(0)
    for n1, n2 in [(0, 5), (5, 0), (1, 1), (100, 3), (4096, 12345), (7, 100003)]:
        a = rng.integers(0, 256, n1, dtype=np.uint8).tobytes()
        b = rng.integers(0, 256, n2, dtype=np.uint8).tobytes()
        assert D.crc32_combine(zlib.crc32(a), zlib.crc32(b), len(b)) == zlib.crc32(a + b)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_shards_contiguous_and_balanced(world):
    numel = [38597376, 786432, 768, 768] + [2359296, 2304, 589824, 768, 768, 768, 2359296, 3072,
                                            2359296, 768] * 12
    b = D.plan_shards(numel, world)
    assert b[0][0] == 0 and b[-1][1] == len(numel)
    assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
    sizes = [sum(numel[s:e]) for s, e in b]
    assert sum(sizes) == sum(numel)
    if world > 1:
        assert max(sizes) <= max(max(numel), 2 * sum(numel) / world)


def _block_offsets(rec):
    """Byte range of every tensor block of a DQDR record (codec.cpp:440-456)."""
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

    out = []
    for _ in range(nt):
        start = pos
        nl = struct.unpack_from("<H", rec, pos)[0]
        pos += 2 + nl + 1
        rank = rec[pos]
        pos += 1 + 8 * rank
        for _ in range(uv()):
            uv()
            pos += 2
        for _ in range(uv()):
            uv(), uv(), uv()
            for _ in range(uv()):
                uv()
                pos += 1
            nb = uv()  # read before adding: uv() advances pos
            pos += nb
        out.append((start, pos))
    return out, out[0][0] if out else pos


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from oracle import oracle as orc

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = orc.get()
        t1 = make_tensors(seed=3)
        t2 = perturb(t1, seed=4)
        bounds = D.plan_shards([t.data.size for t in t1], world)
        s, e = bounds[rank]
        # (1) histogram all-reduce == whole-checkpoint histogram
        kmin, z, pos, neg = o.sketch_dense(flat(t1[s:e]) if e > s else np.zeros(0, np.float32), 0.01)
        h = torch.tensor(np.concatenate([[z], pos, neg]).astype(np.int64))
        dist.all_reduce(h)
        _, zf, posf, negf = o.sketch_dense(flat(t1), 0.01)
        ok_hist = np.array_equal(h.numpy(), np.concatenate([[zf], posf, negf]).astype(np.int64))
        # (2) record assembled from per-rank tensor blocks + CRC combine
        cfg = orc.Config()
        m1, _ = o.scores(flat(t1))
        m2, _ = o.scores(flat(t2))
        q1 = o.quantize(t1, 1, m1, None, cfg, 1)
        q2 = o.quantize(t2, 2, m2, None, cfg, 1)
        full = o.encode_record(q2, q1)
        blocks, prefix_end = _block_offsets(full)
        body = b"".join(full[a:b] for a, b in blocks[s:e])
        stream = b"".join(np.asarray(lv, np.uint16).astype("<u2").tobytes() for lv in q2.levels[s:e])
        parts = [None] * world
        dist.all_gather_object(parts, (body, zlib.crc32(stream), len(stream)))
        rec = D.assemble_record(full[:prefix_end], [p[0] for p in parts], [p[1] for p in parts],
                                [p[2] for p in parts])
        q.put((rank, ok_hist, rec == full))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_histograms_and_record_assembly_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    assert all(r[1] for r in res), "all-reduced shard histograms != whole-checkpoint histogram"
    assert all(r[2] for r in res), "assembled record != single-process record"


def _eval_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfgs = [(b, p) for b in (4, 8, 16, 32) for p in (0.0, 0.1, 0.5)]
        seeds = list(range(100, 100 + len(cfgs)))
        seen = []

        def evaluate(cs, ss):  # deterministic stand-in for Engine.eval_batch
            seen.extend(cs)
            return [b * 0.01 + p for b, p in cs], [s * 1.5 for s in ss]

        qual, est = D.eval_batch_sharded(evaluate, cfgs, seeds)
        ok = (qual == [b * 0.01 + p for b, p in cfgs] and est == [s * 1.5 for s in seeds]
              and seen == [cfgs[i] for i in D.assign_configs(len(cfgs), world)[rank]])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_assign_configs_round_robin():
    parts = D.assign_configs(10, 3)
    assert parts == [[0, 3, 6, 9], [1, 4, 7], [2, 5, 8]]
    assert sorted(i for p in parts for i in p) == list(range(10))


@pytest.mark.parametrize("world", [2])
def test_eval_batch_sharded_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_eval_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    assert all(r[1] for r in res), "sharded batch evaluation differs from the serial order"


def _sharded_evaluator_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2306_11800_b200 import dqt

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seen = []

        class Fake(dqt.Evaluator):  # stands in for the device ProxyEvaluator
            def evaluate(self, c, s, cfg, seed):
                return dqt.EvalResult(0.01 * cfg.bins + cfg.prune_frac, 1.5 * seed)

            def evaluate_batch(self, c, s, cfgs, seeds, parallelism=1):
                seen.extend(cfg.bins for cfg in cfgs)
                return [self.evaluate(c, s, cfg, sd) for cfg, sd in zip(cfgs, seeds)]

        ev = D.sharded_evaluator(Fake())
        cfgs = [dqt.QuantConfig(bins=b, prune_frac=p) for b in (4, 8, 16, 32) for p in (0.0, 0.1)]
        seeds = list(range(7, 7 + len(cfgs)))
        res = ev.evaluate_batch(None, None, cfgs, seeds, 2)
        ok = ([r.quality_delta for r in res] == [0.01 * c.bins + c.prune_frac for c in cfgs]
              and [r.est_compression for r in res] == [1.5 * s for s in seeds]
              and seen == [cfgs[i].bins for i in D.assign_configs(len(cfgs), world)[rank]])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_sharded_evaluator_gloo():
    """The Evaluator handed to the drop-in search splits each batch over the ranks
    and returns the whole batch, in order, on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_evaluator_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(2)]
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    assert all(r[1] for r in res)


def _fail_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []

        def evaluate(cs, ss):
            if rank == 1:
                raise ValueError("local evaluation failure")
            return [0.0] * len(cs), [1.0] * len(cs)

        try:
            D.eval_batch_sharded(evaluate, [(4, 0.0)] * 6, list(range(6)))
            out.append("no error")
        except D.RemoteRankError:
            out.append("remote")
        except ValueError:
            out.append("local")
        # the status exchange in front of a data collective (compress_sharded's stages)
        try:
            D._agree(RuntimeError("stage") if rank == 0 else None, None, torch.device("cpu"))
            out.append("no error")
        except D.RemoteRankError:
            out.append("remote")
        except RuntimeError:
            out.append("local")
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_rank_failure_raises_on_every_rank():
    """a rank failing before a collective must not leave the others blocked
    in it -- every rank raises (its own error or RemoteRankError)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(60)
    assert res[0] == ["remote", "local"] and res[1] == ["local", "remote"], res
