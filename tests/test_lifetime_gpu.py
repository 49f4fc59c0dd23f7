"""Handle lifetimes: checkpoints, states and records keep their engine alive, so an
engine (or pipe) handle may be destroyed before the objects it made, in any order
(Python's cycle collector finalises in arbitrary order)."""
import gc

import numpy as np
import pytest

from tests.util import make_tensors

pytestmark = pytest.mark.gpu


def _layout(ts):
    return [t.name for t in ts], [t.type for t in ts], [t.shape for t in ts]


def test_engine_destroyed_before_its_objects():
    from paper_2306_11800_b200 import engine as E

    ts = make_tensors(seed=1)
    names, types, shapes = _layout(ts)
    eng = E.Engine(0)
    ck = eng.checkpoint(names, types, shapes, weights=[t.data for t in ts])
    st = eng.quantize(ck, E.Config(), 1, 1)
    ref = st.download()
    rec = eng.encode_record_handle(st)
    E.LIB.dqtg_engine_destroy(eng.h)  # the owner lets go first
    eng.h = None
    # the objects still work (their engine is alive until the last one goes)
    h = st.download()
    for a, b in zip(h.levels, ref.levels):
        np.testing.assert_array_equal(a, b)
    assert E.LIB.dqtg_record_size(rec) > 0
    E.LIB.dqtg_record_destroy(rec)
    del ck, st
    gc.collect()


def test_cycle_collected_in_any_order():
    from paper_2306_11800_b200 import engine as E

    ts = make_tensors(seed=2)
    names, types, shapes = _layout(ts)
    for _ in range(3):
        eng = E.Engine(0)
        ck = eng.checkpoint(names, types, shapes, weights=[t.data for t in ts])
        st = eng.quantize(ck, E.Config(), 1, 1)
        cyc = {"eng": eng, "ck": ck, "st": st}
        cyc["self"] = cyc
        eng.cycle = cyc  # engine <-> objects reference cycle
        del eng, ck, st, cyc
        gc.collect()


def test_pipe_state_outlives_pipe():
    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200.pipeline import ChainCompressor

    ts = make_tensors(seed=3)
    names, types, shapes = _layout(ts)
    cc = ChainCompressor(0, workers=2)
    cks = []
    for k in range(3):
        c = cc.checkpoint(names, types, shapes)
        c.set_weights([t.data * np.float32(1 + 0.01 * k) for t in ts])
        cks.append(c)
    last = cc.run(cks, E.Config(), 1, [0, 1, 2])
    want = last.download()
    del cc, cks
    gc.collect()
    got = last.download()  # made by a worker engine of the destroyed pipe
    for a, b in zip(got.levels, want.levels):
        np.testing.assert_array_equal(a, b)
    del last
    gc.collect()
