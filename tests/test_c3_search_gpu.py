"""Config search at the C3 shape (BASELINE configs[2]: a BERT checkpoint searched
over bin counts / prune / protect fractions with batched candidate evaluation),
at reduced width: the drop-in guided_exhaustive_search with the device
ProxyEvaluator (one dqtg_eval_batch per EvalCache::prefetch batch) must reach the
reference's outcome (oracle/_ref, parallelism = nproc, same bytes): the same
config, the same number of evaluations, est_compression exactly and the quality
delta within the reference's own rounding bound (search.cpp:247-296, 380-385).

proxy_quality_delta sums N squared differences sequentially in double
(search.cpp:35-46): that sum is within (N-1) u of the exact one (u = 2^-53), which
at N = 4.4 M is ~5e-10 relative -- larger than 1e-12.  The device sums in a fixed
tree order (error ~log2(N) u), so the two agree to the reference's bound, not to
1e-12; measured: 1.3e-12 relative here."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c3_shaped_search_matches_reference(ref):
    import torch

    from paper_2306_11800_b200 import dqt
    from paper_2306_11800_b200 import workloads as W

    d = ref.load()
    layout = W.bert_large_layout(n_layer=2, d=128, ffn=512)
    N = W.layout_params(layout)
    tr = W.Trajectory(torch, N, 77, torch.device("cuda", 0))
    w = tr.next().cpu().numpy()
    tr.next()
    ema = tr.ema().cpu().numpy()
    nproc = os.cpu_count() or 1

    def run(m):
        c = m.Checkpoint()
        c.step = 1
        e = m.Checkpoint()
        for (name, lt, shape), x, g in zip(layout, W.split(w, layout), W.split(ema, layout)):
            c.add_tensor(name, x.reshape(shape), m.LayerType(lt))
            e.add_tensor(name, g.reshape(shape), m.LayerType(lt))
        st = m.ema_init(0.9)
        m.ema_update(st, e)
        s = m.compute_scores(c, st)
        for thr in (0.1, 0.03):
            out = m.guided_exhaustive_search(c, s, m.ConfigCube(), m.ProxyEvaluator(),
                                             m.SearchParams(threshold=thr, parallelism=nproc, seed=3))
            yield out

    for o1, o2 in zip(run(dqt), run(d)):
        key = lambda o: (o.config.bins, o.config.embed_bins, o.config.prune_frac,  # noqa: E731
                         o.config.protect_frac, int(o.config.metric), o.feasible, o.evaluations_used)
        assert key(o1) == key(o2)
        assert o1.est_compression == o2.est_compression
        tol = max(1e-12, N * 2.0 ** -53)  # sequential-sum bound of the reference
        assert abs(o1.quality_delta - o2.quality_delta) <= tol * max(abs(o2.quality_delta), 1e-300)
