"""BASELINE.json configs[3] and [4] on one B200.

C4 (GPT-2 XL, 1,557,611,200 fp32 params): the whole-checkpoint chain (FULL, then
DELTA against it) on one engine, and the same snapshots as 2, 4 and 8 tensor
shards (paper_2306_11800_b200/shards.py: the multi-GPU path's two histogram
exchanges as sums over the shards).  Asserted: every shard's record decodes back to
its state (decode_delta_record, codec.cpp:513-597), and the records assembled from
the shards are byte-identical to the whole-checkpoint records -- the sharded
quantize + encode reproduces the single-GPU result at full C4 size.

C5 (Llama-3-8B, 8,030,261,248 params, bf16 draws upcast to fp32: 32 GB of weights +
32 GB of EMA): 8 shards regenerated on demand from per-shard seeds; FULL + DELTA,
every shard record round-trips through the device decoder.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c4_sharded_records_equal_whole():
    import torch

    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200 import shards as S
    from paper_2306_11800_b200 import workloads as W

    dev = torch.device("cuda", 0)
    eng = E.Engine(0, torch.cuda.current_stream(dev).cuda_stream)
    lay = W.gpt2_xl_layout()
    assert W.layout_params(lay) == 1_557_611_200
    names = [n for n, _, _ in lay]
    types = [t for _, t, _ in lay]
    shapes = [s for _, _, s in lay]
    snaps, ema = W.series(torch, lay, 2, 77, dev)
    cfg = E.Config()
    whole, prev = [], None
    for k, w in enumerate(snaps):
        ck = E.DevCheckpoint(eng, names, types, shapes)
        ck.set_weights(W.tensor_ptrs(w.data_ptr(), lay))
        ck.set_ema(W.tensor_ptrs(ema.data_ptr(), lay))
        st = eng.quantize(ck, cfg, 1, k)
        whole.append(eng.encode_record(st, prev))
        prev = st
        del ck
    del prev
    offs = np.concatenate([[0], np.cumsum([W.numel(s) for s in shapes])])

    for n in (2, 4, 8):
        ch = S.LocalShardedChain(eng, names, types, shapes, n, cfg, seed=1, device=dev)

        def load(s, ck, k):
            a, b = ch.plan[s]
            base = snaps[k].data_ptr() + 4 * int(offs[a])
            ck.set_weights(W.tensor_ptrs(base, lay[a:b]))
            ck.set_ema(W.tensor_ptrs(ema.data_ptr() + 4 * int(offs[a]), lay[a:b]))

        for k in range(2):
            recs, rt = ch.step(k, lambda s, ck: load(s, ck, k))
            assert all(rt), (n, k, rt)
            assert ch.assemble(recs) == whole[k], (n, k)
        del ch


def test_c5_sharded_roundtrip():
    import torch

    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200 import shards as S
    from paper_2306_11800_b200 import workloads as W

    import gc

    gc.collect()
    torch.cuda.empty_cache()  # the C4 test's snapshots
    dev = torch.device("cuda", 0)
    eng = E.Engine(0, torch.cuda.current_stream(dev).cuda_stream)
    lay = W.llama3_8b_layout()
    assert W.layout_params(lay) == 8_030_261_248
    names = [n for n, _, _ in lay]
    ch = S.LocalShardedChain(eng, names, [t for _, t, _ in lay], [s for _, _, s in lay], 8,
                             E.Config(), seed=1, device=dev)
    gen = W.ShardSeries(torch, lay, ch.plan, 5, dev, bf16=True)
    sizes = []
    for k in range(2):
        recs, rt = ch.step(k, lambda s, ck: gen.load(s, k, ck), keep_records=False)
        assert len(rt) == 8 and all(rt), (k, rt)
        sizes.append(sum(recs))
    # FULL then DELTA: the delta record is much smaller than the full one
    assert sizes[1] < sizes[0]
