"""distributed.compress_sharded itself across two processes (world size 2, gloo,
both ranks on cuda:0): each rank holds a contiguous shard of the tensors
(plan_shards), the score and value histograms are all-reduced, each rank encodes
its blocks with the global alphabet and rank 0 assembles the record.  The FULL and
DELTA records must equal the oracle's for the whole checkpoint, for every config."""
import os
import pickle
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path, cfg_tuples):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2306_11800_b200 import distributed as D
    from paper_2306_11800_b200 import engine as E
    from tests.util import flat, make_tensors, perturb

    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = E.Engine(0)
    t1 = make_tensors(seed=41)
    t2 = perturb(t1, seed=42, frac=0.1)
    ema = np.random.default_rng(5).normal(0, 0.1, flat(t1).size).astype(np.float32)
    offs = np.cumsum([0] + [t.data.size for t in t1])
    lo, hi = D.plan_shards([t.data.size for t in t1], world)[rank]
    recs = []
    for cfg_t in cfg_tuples:
        prev = None
        for step, ts in ((1, t1), (2, t2)):
            mine = ts[lo:hi]
            ck = eng.checkpoint([t.name for t in mine], [t.type for t in mine],
                                [t.shape for t in mine], weights=[t.data for t in mine],
                                ema=[ema[offs[i]:offs[i + 1]] for i in range(lo, hi)])
            st, rec, _ = D.compress_sharded(eng, ck, E.Config(*cfg_t), 1, step, prev,
                                            n_tensors_total=len(ts), gather_record=True)
            recs.append(rec)
            prev = st
    if rank == 0:
        with open(out_path, "wb") as f:
            pickle.dump(recs, f)
    dist.destroy_process_group()


def test_two_process_sharded_records(oracle, tmp_path):
    import torch.multiprocessing as mp

    from tests.util import CONFIGS, flat, make_tensors, perturb

    out = str(tmp_path / "recs.pkl")
    cfgs = [CONFIGS[0], CONFIGS[1], CONFIGS[2]]
    mp.spawn(_worker, args=(2, _free_port(), out, [c.astuple() for c in cfgs]), nprocs=2, join=True)
    with open(out, "rb") as f:
        recs = pickle.load(f)
    t1 = make_tensors(seed=41)
    t2 = perturb(t1, seed=42, frac=0.1)
    ema = np.random.default_rng(5).normal(0, 0.1, flat(t1).size).astype(np.float32)
    want = []
    for cfg in cfgs:
        prev = None
        for step, ts in ((1, t1), (2, t2)):
            m, s = oracle.scores(flat(ts), ema)
            q = oracle.quantize(ts, step, m, s, cfg, 1)
            want.append(oracle.encode_record(q, prev))
            prev = q
    assert len(recs) == len(want)
    for i, (a, b) in enumerate(zip(recs, want)):
        assert a == b, i
