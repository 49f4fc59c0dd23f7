"""Shared test inputs (seeded numpy generators; never /root/reference at run time)."""
import numpy as np

from oracle.oracle import Config, Tensor

# (name, layer type, shape) like tests/helpers.hpp small_checkpoint in the reference
SMALL_LAYOUT = [
    ("tok_embed.weight", 4, (100, 20)),
    ("blk.attn.qkv", 2, (100, 20)),
    ("blk.fc1.weight", 1, (100, 20)),
    ("blk.norm.weight", 3, (500,)),
    ("blk.fc1.bias", 5, (500,)),
    ("stem.conv.weight", 0, (30, 7)),
    ("head.weight", 6, (64, 3)),
]

CONFIGS = [
    Config(),
    Config(bins=8, embed_bins=16, prune_frac=0.1, protect_frac=0.01),
    Config(bins=4, embed_bins=16, prune_frac=0.5, protect_frac=0.0005, metric=1),
    Config(bins=32, embed_bins=32, prune_frac=0.0, protect_frac=0.0),
    Config(bins=6, embed_bins=32, prune_frac=0.3, protect_frac=0.9),   # protect/prune overlap
    Config(bins=12, embed_bins=16, prune_frac=0.2, protect_frac=0.005, metric=1, sigma=0.7,
           alpha=0.02),
]


def make_tensors(layout=SMALL_LAYOUT, seed=0, scale=0.05):
    rng = np.random.default_rng(seed)
    out = []
    for i, (name, lt, shape) in enumerate(layout):
        n = int(np.prod(shape))
        x = rng.normal(0.0, scale * (1 + 0.3 * i), n).astype(np.float32)
        if lt == 3:  # LayerNorm-like weights around 1
            x = (1.0 + 0.1 * rng.normal(size=n)).astype(np.float32)
        out.append(Tensor(name, lt, tuple(shape), x))
    return out


def flat(tensors):
    return np.concatenate([np.ascontiguousarray(t.data, np.float32).ravel() for t in tensors])


def perturb(tensors, seed, frac=0.05, scale=0.01):
    rng = np.random.default_rng(seed)
    out = []
    for t in tensors:
        x = t.data.copy()
        m = rng.random(x.size) < frac
        x[m] += (scale * rng.normal(size=int(m.sum()))).astype(np.float32)
        out.append(Tensor(t.name, t.type, t.shape, x))
    return out
