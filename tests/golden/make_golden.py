"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref = the
reference library compiled from /root/reference/proj sources).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures (golden_*.npz) are committed; the tests that read them never touch
/root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402

LAYOUT = [("tok_embed.weight", 4, (40, 16)), ("blk.attn.qkv", 2, (48, 16)),
          ("blk.fc1.weight", 1, (64, 12)), ("blk.norm.weight", 3, (200,)),
          ("blk.fc1.bias", 5, (120,)), ("stem.conv.weight", 0, (24, 9)), ("head.weight", 6, (30, 5))]
CASES = [  # (bins, embed, prune, protect, metric, sigma, alpha, seed, with_ema)
    (16, 32, 0.0, 0.005, 0, 0.2, 0.01, 1, True),
    (8, 16, 0.2, 0.01, 1, 0.2, 0.01, 7, True),
    (4, 16, 0.5, 0.0005, 0, 0.5, 0.02, 3, False),
]


def main():
    d = R.load()
    rng = np.random.default_rng(2306)
    for ci, (b, eb, pf, tf, m, sg, al, seed, with_ema) in enumerate(CASES):
        w1 = [(0.05 * rng.standard_normal(s)).astype(np.float32) for _, _, s in LAYOUT]
        w1[3] = (1.0 + 0.05 * rng.standard_normal(LAYOUT[3][2])).astype(np.float32)
        w2 = [(x + (rng.random(x.shape) < 0.1) * 0.004 * rng.standard_normal(x.shape)).astype(np.float32)
              for x in w1]
        g = [[(0.1 * rng.standard_normal(s)).astype(np.float32) for _, _, s in LAYOUT] for _ in range(2)]

        def ck(arrs, step):
            c = d.Checkpoint()
            c.step = step
            for (n, lt, _), a in zip(LAYOUT, arrs):
                c.add_tensor(n, a, d.LayerType(lt))
            return c

        ema = None
        if with_ema:
            ema = d.ema_init(0.9)
            for k in range(2):
                d.ema_update(ema, ck(g[k], k + 1))
        cfg = d.QuantConfig(bins=b, embed_bins=eb, prune_frac=pf, protect_frac=tf,
                            metric=d.PruneMetric(m), sigma=sg, alpha=al)
        c1, c2 = ck(w1, 10), ck(w2, 11)
        q1 = d.quantize_checkpoint(c1, d.compute_scores(c1, ema), cfg, seed)
        q2 = d.quantize_checkpoint(c2, d.compute_scores(c2, ema), cfg, seed)
        full = bytes(d.encode_delta_record(q1, None, 0.125))
        delta = bytes(d.encode_delta_record(q2, q1, 0.25))
        out = {
            "w1": np.concatenate([x.ravel() for x in w1]),
            "w2": np.concatenate([x.ravel() for x in w2]),
            "g0": np.concatenate([x.ravel() for x in g[0]]),
            "g1": np.concatenate([x.ravel() for x in g[1]]),
            "config": np.array([b, eb, pf, tf, m, sg, al], np.float64),
            "seed": np.array([seed]), "with_ema": np.array([with_ema]),
            "full": np.frombuffer(full, np.uint8), "delta": np.frombuffer(delta, np.uint8),
            "levels2": np.concatenate([np.asarray(t.levels, np.uint16).ravel() for t in q2.tensors]),
            "cb2": np.concatenate([np.asarray(q2.codebook(d.LayerType(lt)), np.float32) for lt in range(7)]),
            "cb2_len": np.array([len(q2.codebook(d.LayerType(lt))) for lt in range(7)], np.int64),
        }
        np.savez_compressed(os.path.join(HERE, f"golden_case{ci}.npz"), **out)
        print(f"case {ci}: FULL {len(full)} B, DELTA {len(delta)} B")
    # sketch known answers
    x = np.concatenate([rng.normal(0, 0.05, 3000), [0.0, -0.0, 1e-13, 5.0, -5.0, 3.4e38]]).astype(np.float32)
    s = d.sketch_build(x, 0.01)
    h = s.histogram()
    np.savez_compressed(os.path.join(HERE, "golden_sketch.npz"), x=x,
                        keys=np.asarray(h.keys), counts=np.asarray(h.counts, np.uint64),
                        q=np.array([s.quantile(q) for q in (0.0, 0.01, 0.5, 0.9975, 1.0)]))


if __name__ == "__main__":
    main()
