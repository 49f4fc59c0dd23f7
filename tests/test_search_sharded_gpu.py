"""Search control across ranks: guided_exhaustive_search and
delta_neighborhood_search with distributed.sharded_evaluator on two ranks (gloo,
both on cuda:0) reach exactly the outcome of the single-process search with the
device ProxyEvaluator, while each rank evaluates only its share of every batch --
and that outcome is the reference's own (oracle/_ref: the same configs, evaluation
counts and compression estimates; quality deltas within the reference's sequential
sum bound, search.cpp:35-46)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(dqt):
    rng = np.random.default_rng(3)
    c = dqt.Checkpoint()
    c.add_tensor("tok_embed.weight", rng.normal(0, 0.05, (300, 64)).astype(np.float32),
                 dqt.LayerType.EMBEDDING)
    c.add_tensor("h.0.attn.weight", rng.normal(0, 0.05, (128, 128)).astype(np.float32),
                 dqt.LayerType.ATTENTION)
    c.add_tensor("h.0.mlp.weight", rng.normal(0, 0.05, (128, 256)).astype(np.float32),
                 dqt.LayerType.LINEAR)
    c.add_tensor("h.0.ln.weight", (1 + rng.normal(0, 0.01, 128)).astype(np.float32),
                 dqt.LayerType.NORM)
    return c, dqt.compute_scores(c)


def _outcome(o):
    c = o.config
    return (c.bins, c.embed_bins, c.prune_frac, c.protect_frac, int(c.metric), o.quality_delta,
            o.est_compression, o.evaluations_used, o.feasible)


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2306_11800_b200 import distributed as D
    from paper_2306_11800_b200 import dqt

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, s = _problem(dqt)
        calls = []

        class Counting(dqt.ProxyEvaluator):
            def evaluate_batch(self, checkpoint, scores, configs, seeds, parallelism=1):
                calls.append(len(configs))
                return dqt.ProxyEvaluator.evaluate_batch(self, checkpoint, scores, configs, seeds,
                                                         parallelism)

        ev = D.sharded_evaluator(Counting())
        params = dqt.SearchParams(threshold=0.1, seed=4)
        g = dqt.guided_exhaustive_search(c, s, dqt.ConfigCube(), ev, params)
        d = dqt.delta_neighborhood_search(c, s, dqt.ConfigCube(), ev, g.config, 1, params)
        q.put((rank, _outcome(g), _outcome(d), sum(calls)))
    finally:
        dist.destroy_process_group()


def _search(m):
    c, s = _problem(m)
    params = m.SearchParams(threshold=0.1, seed=4)
    ev = m.ProxyEvaluator()
    g = m.guided_exhaustive_search(c, s, m.ConfigCube(), ev, params)
    d = m.delta_neighborhood_search(c, s, m.ConfigCube(), ev, g.config, 1, params)
    return g, d


def test_sharded_search_matches_single_process(ref):
    from paper_2306_11800_b200 import dqt

    g, d = _search(dqt)
    want = (_outcome(g), _outcome(d))
    # the single-process device search is the reference's search
    n = 300 * 64 + 128 * 128 + 128 * 256 + 128  # elements of _problem
    tol = max(1e-12, n * 2.0 ** -53)
    for mine, theirs in zip((g, d), _search(ref.load())):
        a, b = _outcome(mine), _outcome(theirs)
        assert a[:5] == b[:5] and a[6:] == b[6:], (a, b)
        assert abs(a[5] - b[5]) <= tol * max(abs(b[5]), 1e-300), (a, b)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, go, do, n_eval in res:
        assert (go, do) == want, rank
    # the two ranks split the evaluations (round robin per batch)
    total = g.evaluations_used + d.evaluations_used
    assert res[0][3] + res[1][3] <= total and max(res[0][3], res[1][3]) < total
