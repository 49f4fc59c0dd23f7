"""The fused score/partition pass (opt-in: DQTG_FUSED_AB=1) (quantize.cu pass_ab_kernel) guesses the protect
thresholds from a tile sample, partitions with the guess, lists the elements near
the guessed thresholds and corrects them once the exact quantiles are known
(falling back to pass B when a threshold lands outside the listed band).  Here the
guess is pushed off by a few buckets on purpose (test hook DQTG_FUSED_GUESS_SHIFT):
inside the band the corrections must reproduce the oracle's states and records
exactly; outside it the pass B fallback must."""
import os

import numpy as np
import pytest

from tests.util import CONFIGS, flat, make_tensors, perturb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shift", [0, 2, -3, 4, 9, -40])
@pytest.mark.parametrize("cfg_i", [0, 1, 5])
def test_guessed_thresholds_corrected(oracle, shift, cfg_i):
    from oracle.oracle import Config as OC  # noqa: F401
    from paper_2306_11800_b200 import engine as E

    eng = E.Engine(0)
    t1 = make_tensors(seed=21)
    t2 = perturb(t1, seed=22, frac=0.3)
    ema = np.random.default_rng(3).normal(0, 0.1, flat(t1).size).astype(np.float32)
    sizes = np.cumsum([t.data.size for t in t1])[:-1]
    cfg = CONFIGS[cfg_i]
    os.environ["DQTG_FUSED_GUESS_SHIFT"] = str(shift)
    os.environ["DQTG_FUSED_AB"] = "1"
    try:
        prev_dev = prev_ref = None
        for step, ts in ((1, t1), (2, t2)):
            ck = eng.checkpoint([t.name for t in ts], [t.type for t in ts], [t.shape for t in ts],
                                weights=[t.data for t in ts], ema=np.split(ema, sizes))
            st = eng.quantize(ck, E.Config(*cfg.astuple()), 1, step)
            m, s = oracle.scores(flat(ts), ema)
            q = oracle.quantize(ts, step, m, s, cfg, 1)
            got = st.download()
            for a, b in zip(got.levels, q.levels):
                np.testing.assert_array_equal(a, b)
            for a, b in zip(got.prot_pos, q.prot_pos):
                np.testing.assert_array_equal(a, b)
            assert eng.encode_record(st, prev_dev) == oracle.encode_record(q, prev_ref)
            prev_dev, prev_ref = st, q
    finally:
        del os.environ["DQTG_FUSED_GUESS_SHIFT"]
        del os.environ["DQTG_FUSED_AB"]
