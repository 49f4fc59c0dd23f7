"""Pass C fused into the DELTA encoder (codec.cu enc_tile_delta_kernel<true>,
reached through dqtg_compress_step = Chain::append, chain.cpp:86-129).

The target levels are computed from w and the partition (pass B's 2-bit codes, or
the protected bitmap of pass A2's candidate list) inside the encoder's tile pass
(quantize.cpp:396-423) instead of being written by pass C and read back.  Asserted against the oracle, bit for bit: the DELTA record
(codec.cpp:398-460), the state's levels, protected (pos, bf16) entries and
codebooks, for every test config (prune / protect / metric / alpha), explicit and
EMA-derived scores, ragged tensors (sizes that are not multiples of 4, 16 or 64)
and delta densities from 0 to 100 %; and that fused and unfused runs agree.
"""
import os

import numpy as np
import pytest

from oracle.oracle import QState, Tensor
from tests.util import CONFIGS, SMALL_LAYOUT, flat, make_tensors, perturb

pytestmark = pytest.mark.gpu

RAGGED = [
    ("tok_embed.weight", 4, (333, 7)),
    ("blk.attn.qkv", 2, (4097,)),
    ("blk.fc1.weight", 1, (65, 63)),
    ("blk.norm.weight", 3, (1,)),
    ("blk.fc1.bias", 5, (17,)),
    ("stem.conv.weight", 0, (8191,)),
    ("head.weight", 6, (3, 5, 7)),
]


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine

    return engine.Engine(0)


def _qs(h) -> QState:
    return QState(h.step, h.config, h.codebooks, h.names, h.types, h.shapes, h.levels, h.prot_pos,
                  h.prot_val)


def _ckpt(eng, ts, ema, derived, oracle):
    names = [t.name for t in ts]
    types = [t.type for t in ts]
    shapes = [t.shape for t in ts]
    sizes = np.cumsum([t.data.size for t in ts])[:-1]
    w = [t.data for t in ts]
    if derived:
        return eng.checkpoint(names, types, shapes, weights=w,
                              ema=None if ema is None else np.split(ema, sizes))
    m, s = oracle.scores(flat(ts), ema)
    return eng.checkpoint(names, types, shapes, weights=w, mag=np.split(m, sizes),
                          sens=None if s is None else np.split(s, sizes))


def _step(eng, oracle, cfg, t0, t1, ema, derived, seed=7):
    from paper_2306_11800_b200.engine import Config

    dcfg = Config(*cfg.astuple())
    base = eng.quantize(_ckpt(eng, t0, ema, derived, oracle), dcfg, seed, 3)
    m0, s0 = oracle.scores(flat(t0), ema)
    m1, s1 = oracle.scores(flat(t1), ema)
    o0 = oracle.quantize(t0, 3, m0, s0, cfg, seed)
    o1 = oracle.quantize(t1, 4, m1, s1, cfg, seed)
    out = {}
    # fused with pass A2 + candidates (default), fused with pass B, unfused
    for mode, env in (("fused", {}), ("fused_passb", {"DQTG_NO_PASS_A2": "1"}),
                      ("fused_a2_fallback", {"DQTG_A2_BOUND_SHIFT": "40"}),
                      # bounds next to the thresholds: the sensitivity threshold in the
                      # lumped bound bucket must fall back, one bucket above must not
                      ("fused_a2_edge3", {"DQTG_A2_BOUND_SHIFT": "3"}),
                      ("fused_a2_edge4", {"DQTG_A2_BOUND_SHIFT": "4"}),
                      ("fused_a2_edge5", {"DQTG_A2_BOUND_SHIFT": "5"}),
                      ("unfused", {"DQTG_NO_FUSED_C": "1"})):
        os.environ.update(env)
        try:
            st, rh = eng.compress_step(_ckpt(eng, t1, ema, derived, oracle), dcfg, seed, 4,
                                       base=base, quality=0.5)
        finally:
            for k in env:
                os.environ.pop(k, None)
        out[mode] = (st.download(), eng.record_bytes(rh))
    want_rec = oracle.encode_record(o1, o0, 0.5)
    for fused, (got, rec) in out.items():
        assert _qs(got) == o1, ("state", fused)
        assert rec == want_rec, ("record", fused, len(rec), len(want_rec))


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
@pytest.mark.parametrize("derived", [False, True])
def test_fused_compress_step_matches_oracle(eng, oracle, ci, derived):
    cfg = CONFIGS[ci]
    t0 = make_tensors(seed=ci)
    t1 = perturb(t0, seed=200 + ci)
    rng = np.random.default_rng(ci)
    ema = rng.normal(0, 0.1, flat(t0).size).astype(np.float32) if (cfg.metric or ci % 2 == 0) else None
    _step(eng, oracle, cfg, t0, t1, ema, derived)


@pytest.mark.parametrize("frac", [0.0, 0.02, 0.3, 1.0])
def test_fused_ragged_and_dense(eng, oracle, frac):
    cfg = CONFIGS[1]
    t0 = make_tensors(RAGGED, seed=5)
    # frac of the elements moved far enough to change level: 0 (all-zero deltas) to
    # 1 (a fresh draw: dense deltas, the Z list in global memory)
    rng = np.random.default_rng(9)
    t1 = []
    for t in t0:
        x = t.data.copy()
        msk = rng.random(x.size) < frac
        x[msk] = rng.normal(0.0, 0.08, int(msk.sum())).astype(np.float32)
        t1.append(Tensor(t.name, t.type, t.shape, x))
    ema = rng.normal(0, 0.1, flat(t0).size).astype(np.float32)
    _step(eng, oracle, cfg, t0, t1, ema, True)


def test_fused_large_tensor(eng, oracle):
    """Tensors of many tiles (runs crossing tiles, per-tensor symbol flush)."""
    cfg = CONFIGS[0]
    lay = [("tok_embed.weight", 4, (3000, 97)), ("blk.fc1.weight", 1, (700, 300)),
           ("blk.norm.weight", 3, (777,))]
    t0 = make_tensors(lay, seed=1)
    t1 = perturb(t0, seed=2, frac=0.03, scale=0.02)
    ema = np.random.default_rng(3).normal(0, 0.1, flat(t0).size).astype(np.float32)
    _step(eng, oracle, cfg, t0, t1, ema, True)


@pytest.mark.parametrize("where", ["ema_nan", "ema_inf", "w_inf"])
def test_fused_step_non_finite(eng, oracle, where):
    """NaN / Inf scores or weights raise NonFiniteData on the fused step -- also where pass
    A2 builds no sensitivity histogram (it checks the sensitivities itself) -- as the
    unfused path and the reference's sketch do."""
    from paper_2306_11800_b200.engine import Config, EngineError

    cfg = CONFIGS[0]
    lay = [("tok_embed.weight", 4, (3000, 97)), ("blk.fc1.weight", 1, (700, 300))]
    t0 = make_tensors(lay, seed=1)
    t1 = perturb(t0, seed=2, frac=0.03, scale=0.02)
    ema = np.random.default_rng(3).normal(0, 0.1, flat(t0).size).astype(np.float32)
    dcfg = Config(*cfg.astuple())
    base = eng.quantize(_ckpt(eng, t0, ema, True, oracle), dcfg, 7, 3)
    bad_ema, bad_t1 = ema.copy(), [Tensor(t.name, t.type, t.shape, t.data.copy()) for t in t1]
    at = 200_000 + 123  # inside the second tensor, a full half tile
    if where == "ema_nan":
        bad_ema[at] = np.nan
    elif where == "ema_inf":
        bad_ema[at] = np.inf
    else:
        bad_t1[1].data.reshape(-1)[at - t1[0].data.size] = np.inf
    for env in ({}, {"DQTG_NO_PASS_A2": "1"}, {"DQTG_NO_FUSED_C": "1"}):
        os.environ.update(env)
        try:
            with pytest.raises(EngineError) as ei:
                eng.compress_step(_ckpt(eng, bad_t1, bad_ema, True, oracle), dcfg, 7, 4, base=base)
            assert ei.value.status == 5, (where, env, ei.value)
        finally:
            for k in env:
                os.environ.pop(k, None)
