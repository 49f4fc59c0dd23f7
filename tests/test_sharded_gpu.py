"""Tensor-sharded quantize + encode on the device (the multi-GPU path of §8e),
simulated with several shards on one GPU: stage histograms summed across
shards, per-shard tensor blocks assembled into one record.  Must be
byte-identical to the single-shard record and to the oracle."""
import struct

import numpy as np
import pytest

from paper_2306_11800_b200 import distributed as D
from tests.util import CONFIGS, flat, make_tensors, perturb

pytestmark = pytest.mark.gpu


def _sharded_records(eng, shards_w, shards_prev_state, cfg, seed, step, ema_parts, nt_total):
    import torch

    from paper_2306_11800_b200 import engine as E

    ns, nv = eng.shard_hist_len(cfg, 0), eng.shard_hist_len(cfg, 1)
    scores = [torch.zeros(ns, dtype=torch.int64, device="cuda") for _ in shards_w]
    values = [torch.zeros(nv, dtype=torch.int64, device="cuda") for _ in shards_w]
    for ck, sc in zip(shards_w, scores):
        eng.shard_stage1(ck, cfg, sc.data_ptr())
    eng.sync()
    tot = sum(scores)
    for ck, v in zip(shards_w, values):
        eng.shard_stage2(ck, cfg, tot.data_ptr(), v.data_ptr())
        eng.sync()
    vtot = sum(values)
    states = [eng.shard_stage3(ck, cfg, seed, step, vtot.data_ptr()) for ck in shards_w]
    gB = max([s.info().max_levels for s in states] +
             [p.info().max_levels for p in shards_prev_state if p is not None] + [2])
    prefix, bodies, crcs, lens = None, [], [], []
    for st, prev in zip(states, shards_prev_state):
        r, off = eng.encode_record_shard(st, prev, 0.0, gB, nt_total)
        n = E.LIB.dqtg_record_size(r)
        buf = np.empty(n, np.uint8)
        E._check(E.LIB.dqtg_record_copy(r, buf.ctypes.data))
        E.LIB.dqtg_record_destroy(r)
        if prefix is None:
            prefix = buf[:off].tobytes()
        bodies.append(buf[off:n - 4].tobytes())
        crcs.append(struct.unpack("<I", buf[n - 4:].tobytes())[0])
        lens.append(2 * int(st.info().param_count))
    return states, D.assemble_record(prefix, bodies, crcs, lens)


@pytest.mark.parametrize("ci", [0, 1, 2])
@pytest.mark.parametrize("nshards", [2, 3])
def test_sharded_equals_single(oracle, ci, nshards):
    from paper_2306_11800_b200 import engine as E

    eng = E.Engine(0)
    cfg = CONFIGS[ci]
    if ci == 2:  # sensitivity metric needs the EMA
        pass
    t1 = make_tensors(seed=10 + ci)
    t2 = perturb(t1, seed=20 + ci)
    rng = np.random.default_rng(ci)
    ema = rng.normal(0, 0.1, flat(t1).size).astype(np.float32)
    sizes = [t.data.size for t in t1]
    bounds = D.plan_shards(sizes, nshards)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    ecfg = E.Config(*cfg.astuple())

    def ck_for(ts, s, e):
        c = eng.checkpoint([t.name for t in ts[s:e]], [t.type for t in ts[s:e]],
                           [t.shape for t in ts[s:e]], weights=[t.data for t in ts[s:e]],
                           ema=[ema[offs[i]:offs[i + 1]] for i in range(s, e)])
        return c

    prev_states = [None] * nshards
    recs = []
    for step, ts in ((1, t1), (2, t2)):
        shards = [ck_for(ts, s, e) for s, e in bounds]
        states, rec = _sharded_records(eng, shards, prev_states, ecfg, 5, step, None, len(ts))
        recs.append(rec)
        prev_states = states
    # single checkpoint through the oracle
    o_states = []
    for step, ts in ((1, t1), (2, t2)):
        m, s = oracle.scores(flat(ts), ema)
        o_states.append(oracle.quantize(ts, step, m, s, cfg, 5))
    assert recs[0] == oracle.encode_record(o_states[0])
    assert recs[1] == oracle.encode_record(o_states[1], o_states[0])
