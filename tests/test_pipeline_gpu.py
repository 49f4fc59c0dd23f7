"""The pipelined chain (worker-pool streams, encode(k) waits on quantize(k-1))
produces the same records as the oracle, for device-resident and host inputs.
Device-resident snapshots carry their own gradient EMA each (the sensitivity
scores of step k come from snapshot k's EMA); host inputs share one."""
import numpy as np
import pytest

from tests.util import flat, make_tensors, perturb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("workers,host_inputs", [(1, False), (2, False), (3, False), (3, True)])
def test_pipelined_chain_matches_oracle(oracle, workers, host_inputs):
    from oracle.oracle import Config as OC
    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200.pipeline import ChainCompressor

    series = [make_tensors(seed=5)]
    for k in range(4):
        series.append(perturb(series[-1], seed=50 + k))
    rng = np.random.default_rng(1)
    n_el = flat(series[0]).size
    emas = [rng.normal(0, 0.1 * (1 + k), n_el).astype(np.float32) for k in range(len(series))]
    ema = emas[0]
    names = [t.name for t in series[0]]
    types = [t.type for t in series[0]]
    shapes = [t.shape for t in series[0]]
    sizes = np.cumsum([t.data.size for t in series[0]])[:-1]
    cfg = E.Config()
    cc = ChainCompressor(0, workers=workers)
    cks = []
    for k, ts in enumerate(series):
        if host_inputs:
            cks.append([np.ascontiguousarray(t.data, np.float32) for t in ts])
            continue
        c = cc.checkpoint(names, types, shapes)
        c.set_weights([t.data for t in ts])
        c.set_ema(np.split(emas[k], sizes))
        cks.append(c)
    host = (names, types, shapes, np.split(ema, sizes)) if host_inputs else None
    recs = {}

    def grab(k, r):
        n = E.LIB.dqtg_record_size(r)
        buf = np.empty(n, np.uint8)
        E._check(E.LIB.dqtg_record_copy(r, buf.ctypes.data))
        recs[k] = buf.tobytes()

    cc.run(cks, cfg, 3, list(range(len(cks))), on_record=grab, host=host)
    prev = None
    for k, ts in enumerate(series):
        m, s = oracle.scores(flat(ts), ema if host_inputs else emas[k])
        q = oracle.quantize(ts, k, m, s, OC(), 3)
        assert recs[k] == oracle.encode_record(q, prev), k
        prev = q
