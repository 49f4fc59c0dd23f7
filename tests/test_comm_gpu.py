"""The engine library's NCCL data plane (comm.cu): a one-rank communicator runs the
whole sharded step through dqtg_compress_sharded (histogram all-reduces, the
global alphabet, the body gather and the CRC combine on rank 0) and must write the
single-GPU record byte for byte, FULL and DELTA, equal to the oracle's.  (Several
ranks need several GPUs: NCCL refuses two ranks on one device; the host logic of
the multi-rank exchange is covered with gloo in test_distributed_cpu.py and
test_sharded_mp_gpu.py.)"""
import numpy as np
import pytest

from tests.util import CONFIGS, flat, make_tensors, perturb

pytestmark = pytest.mark.gpu


def test_one_rank_sharded_step_equals_single_gpu(oracle):
    from paper_2306_11800_b200 import distributed as D
    from paper_2306_11800_b200 import engine as E

    eng = E.Engine(0)
    comm = D.make_comm(eng)
    assert (comm.rank, comm.size) == (0, 1)
    t1 = make_tensors(seed=31)
    t2 = perturb(t1, seed=32, frac=0.1)
    ema = np.random.default_rng(4).normal(0, 0.1, flat(t1).size).astype(np.float32)
    sizes = np.cumsum([t.data.size for t in t1])[:-1]
    for cfg in CONFIGS[:3]:
        prev = prev_q = None
        for step, ts in ((1, t1), (2, t2)):
            ck = eng.checkpoint([t.name for t in ts], [t.type for t in ts], [t.shape for t in ts],
                                weights=[t.data for t in ts], ema=np.split(ema, sizes))
            st, rec, stats = D.compress_sharded(eng, ck, E.Config(*cfg.astuple()), 1, step, prev,
                                                comm=comm, gather_record=True)
            m, s = oracle.scores(flat(ts), ema)
            q = oracle.quantize(ts, step, m, s, cfg, 1)
            assert rec == oracle.encode_record(q, prev_q)
            ref_st, ref_r = eng.compress_step(ck, E.Config(*cfg.astuple()), 1, step, prev)
            n = E.LIB.dqtg_record_size(ref_r)
            buf = np.empty(n, np.uint8)
            E._check(E.LIB.dqtg_record_copy(ref_r, buf.ctypes.data))
            E.LIB.dqtg_record_destroy(ref_r)
            assert rec == buf.tobytes()
            prev, prev_q = st, q


def test_comm_allreduce_one_rank():
    import torch

    from paper_2306_11800_b200 import distributed as D
    from paper_2306_11800_b200 import engine as E

    eng = E.Engine(0)
    comm = D.make_comm(eng)
    x = torch.arange(1000, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    comm.allreduce_u64(x.data_ptr(), x.numel())
    eng.sync()
    assert torch.equal(x.cpu(), torch.arange(1000, dtype=torch.int64))


def test_pipe_with_one_rank_comms_matches_plain_pipe():
    """The worker pool on communicators (dqtg_pipe_set_comms): worker w runs the
    sharded step of snapshots w mod W on its own communicator; with one rank the
    records equal the plain worker pool's."""
    from paper_2306_11800_b200 import distributed as D
    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200.pipeline import ChainCompressor

    series = [make_tensors(seed=7)]
    for k in range(5):
        series.append(perturb(series[-1], seed=70 + k))
    ema = np.random.default_rng(6).normal(0, 0.1, flat(series[0]).size).astype(np.float32)
    sizes = np.cumsum([t.data.size for t in series[0]])[:-1]
    names = [t.name for t in series[0]]
    types = [t.type for t in series[0]]
    shapes = [t.shape for t in series[0]]
    out = []
    for use_comms in (False, True):
        eng = E.Engine(0)
        comms = [D.make_comm(eng) for _ in range(3)] if use_comms else None
        cc = ChainCompressor(0, workers=3, comms=comms)
        cks = []
        for ts in series:
            c = cc.checkpoint(names, types, shapes)
            c.set_weights([t.data for t in ts])
            c.set_ema(np.split(ema, sizes))
            cks.append(c)
        recs = {}

        def grab(k, r):
            n = E.LIB.dqtg_record_size(r)
            buf = np.empty(n, np.uint8)
            E._check(E.LIB.dqtg_record_copy(r, buf.ctypes.data))
            recs[k] = buf.tobytes()

        cc.run(cks, E.Config(), 1, list(range(len(cks))), on_record=grab)
        out.append(recs)
    assert sorted(out[0]) == list(range(6))
    assert out[0] == out[1]
