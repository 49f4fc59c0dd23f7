"""Synthetic checkpoint series for the BASELINE.json configurations (input
synthesis for bench.py and the full-size parity tests; not part of the
compression path).

Layouts follow SURVEY.md §8d (GPT-2 small C2, BERT-large C3, GPT-2 XL C4,
Llama-3-8B C5) with the reference's layer types (include/dqt/tensor.hpp:12-21).
The trajectory follows the reference generator's dynamics
(/root/reference/proj/src/trajectory.cpp:75-113): w0 = 0.05 N(0,1); per step
g = w + 0.05 * noise * N(0,1); w -= float(lr) * g (two float roundings, no FMA);
lr *= decay.  The normal draws come from torch's Philox generator on the GPU
(the reference's serial mt19937_64 Box-Muller would take minutes per GB), so
both bench arms and the parity tests get identical bytes from the same seed.
The gradient EMA is the reference's ema_update (ranker.cpp:21-37) in float,
b * g + (1 - b) * e with b = float(beta), every product and sum rounded
separately — bit-identical to what the reference's own ema_update produces
from the same gradients.
"""
from __future__ import annotations

import numpy as np

CONV, LIN, ATT, NORM, EMB, BIAS, OTHER = range(7)


def numel(shape):
    return int(np.prod(shape, dtype=np.int64))


def gpt2_layout(n_layer=12, d=768, vocab=50257, ctx=1024, blocks=None, with_embed=True,
                with_lnf=True):
    """GPT-2 (HF transformers naming; Conv1D weights are [in, out])."""
    L = []
    if with_embed:
        L += [("transformer.wte.weight", EMB, (vocab, d)), ("transformer.wpe.weight", EMB, (ctx, d))]
    for i in (range(n_layer) if blocks is None else blocks):
        p = f"transformer.h.{i}."
        L += [(p + "ln_1.weight", NORM, (d,)), (p + "ln_1.bias", BIAS, (d,)),
              (p + "attn.c_attn.weight", ATT, (d, 3 * d)), (p + "attn.c_attn.bias", BIAS, (3 * d,)),
              (p + "attn.c_proj.weight", ATT, (d, d)), (p + "attn.c_proj.bias", BIAS, (d,)),
              (p + "ln_2.weight", NORM, (d,)), (p + "ln_2.bias", BIAS, (d,)),
              (p + "mlp.c_fc.weight", LIN, (d, 4 * d)), (p + "mlp.c_fc.bias", BIAS, (4 * d,)),
              (p + "mlp.c_proj.weight", LIN, (4 * d, d)), (p + "mlp.c_proj.bias", BIAS, (d,))]
    if with_lnf:
        L += [("transformer.ln_f.weight", NORM, (d,)), ("transformer.ln_f.bias", BIAS, (d,))]
    return L


def gpt2_small_layout(**kw):
    """C2: 124,439,808 params, 148 tensors."""
    return gpt2_layout(12, 768, **kw)


def gpt2_xl_layout(**kw):
    """C4: 48 layers, d = 1600 (1,557,611,200 params)."""
    return gpt2_layout(48, 1600, **kw)


def bert_large_layout(n_layer=24, d=1024, ffn=4096, vocab=30522, ctx=512):
    """C3: BERT-large (HF naming), 335,141,888 params."""
    L = [("bert.embeddings.word_embeddings.weight", EMB, (vocab, d)),
         ("bert.embeddings.position_embeddings.weight", EMB, (ctx, d)),
         ("bert.embeddings.token_type_embeddings.weight", EMB, (2, d)),
         ("bert.embeddings.LayerNorm.weight", NORM, (d,)),
         ("bert.embeddings.LayerNorm.bias", BIAS, (d,))]
    for i in range(n_layer):
        p = f"bert.encoder.layer.{i}."
        for m in ("query", "key", "value"):
            L += [(p + f"attention.self.{m}.weight", ATT, (d, d)),
                  (p + f"attention.self.{m}.bias", BIAS, (d,))]
        L += [(p + "attention.output.dense.weight", ATT, (d, d)),
              (p + "attention.output.dense.bias", BIAS, (d,)),
              (p + "attention.output.LayerNorm.weight", NORM, (d,)),
              (p + "attention.output.LayerNorm.bias", BIAS, (d,)),
              (p + "intermediate.dense.weight", LIN, (ffn, d)),
              (p + "intermediate.dense.bias", BIAS, (ffn,)),
              (p + "output.dense.weight", LIN, (d, ffn)), (p + "output.dense.bias", BIAS, (d,)),
              (p + "output.LayerNorm.weight", NORM, (d,)), (p + "output.LayerNorm.bias", BIAS, (d,))]
    L += [("bert.pooler.dense.weight", LIN, (d, d)), ("bert.pooler.dense.bias", BIAS, (d,))]
    return L


def llama3_8b_layout(n_layer=32, d=4096, ffn=14336, kv=1024, vocab=128256):
    """C5: Llama-3-8B (HF naming), 8,030,261,248 params."""
    L = [("model.embed_tokens.weight", EMB, (vocab, d))]
    for i in range(n_layer):
        p = f"model.layers.{i}."
        L += [(p + "input_layernorm.weight", NORM, (d,)),
              (p + "self_attn.q_proj.weight", ATT, (d, d)),
              (p + "self_attn.k_proj.weight", ATT, (kv, d)),
              (p + "self_attn.v_proj.weight", ATT, (kv, d)),
              (p + "self_attn.o_proj.weight", ATT, (d, d)),
              (p + "post_attention_layernorm.weight", NORM, (d,)),
              (p + "mlp.gate_proj.weight", LIN, (ffn, d)),
              (p + "mlp.up_proj.weight", LIN, (ffn, d)),
              (p + "mlp.down_proj.weight", LIN, (d, ffn))]
    L += [("model.norm.weight", NORM, (d,)), ("lm_head.weight", OTHER, (vocab, d))]
    return L


LAYOUTS = {"C2": gpt2_small_layout, "C3": bert_large_layout, "C4": gpt2_xl_layout,
           "C5": llama3_8b_layout}


def layout_params(layout):
    return sum(numel(s) for _, _, s in layout)


def ema_of(torch, grads, beta=0.9):
    """ema_update (ranker.cpp:21-37) over `grads` in order: the first copies, later
    ones e = b * g + (1 - b) * e in float with separately rounded operations."""
    b = torch.tensor(beta, dtype=torch.float32, device=grads[0].device)
    omb = torch.tensor(1.0, dtype=torch.float32, device=b.device) - b  # 1.0f - b
    e = grads[0].clone()
    for g in grads[1:]:
        e = torch.add(torch.mul(g, b), torch.mul(e, omb))
    return e


class Trajectory:
    """Snapshot series w_0, w_1, ... of one flat fp32 checkpoint on `device`
    (reference dynamics, see module doc).  ``bf16`` draws every normal as bf16 and
    upcasts (C5's "bf16-to-fp32" checkpoints: the low 16 mantissa bits of w0 are 0).
    Iterate with ``next()``; ``grads`` holds the first ``n_grads`` gradients."""

    def __init__(self, torch, n, seed, device, lr0=0.1, decay=0.9, noise=0.05, bf16=False,
                 n_grads=2):
        self.torch = torch
        self.n = int(n)
        self.g = torch.Generator(device=device).manual_seed(int(seed))
        self.device = device
        self.lr = float(lr0)
        self.decay = float(decay)
        self.sigma = float(noise) * 0.05
        self.bf16 = bf16
        self.n_grads = n_grads
        self.grads = []
        self.w = torch.mul(self._randn(), torch.tensor(0.05, dtype=torch.float32, device=device))
        if bf16:
            self.w = self.w.to(torch.bfloat16).to(torch.float32)
        self.k = 0

    def _randn(self):
        t = self.torch
        dt = t.bfloat16 if self.bf16 else t.float32
        return t.randn(self.n, generator=self.g, device=self.device, dtype=dt).to(t.float32)

    def next(self):
        """Returns snapshot k (a fresh tensor) and advances to k + 1."""
        t = self.torch
        w = self.w
        sig = t.tensor(self.sigma, dtype=t.float32, device=self.device)
        g = t.add(w, t.mul(self._randn(), sig))
        if len(self.grads) < self.n_grads:
            self.grads.append(g)
        lr = t.tensor(self.lr, dtype=t.float32, device=self.device)  # float(lr)
        self.w = t.sub(w, t.mul(g, lr))
        self.lr *= self.decay
        self.k += 1
        return w

    def ema(self, beta=0.9):
        return ema_of(self.torch, self.grads, beta)


def series(torch, layout, n_snap, seed, device, **kw):
    """n_snap flat snapshots and the EMA of the first two gradients."""
    tr = Trajectory(torch, layout_params(layout), seed, device, **kw)
    snaps = [tr.next() for _ in range(n_snap)]
    if len(tr.grads) < 2:
        tr.next()
    return snaps, tr.ema()


def tensor_ptrs(base_ptr, layout, elem_bytes=4):
    ptrs, o = [], 0
    for _, _, s in layout:
        ptrs.append(base_ptr + elem_bytes * o)
        o += numel(s)
    return ptrs


def split(flat, layout):
    """Per-tensor views of a flat numpy array."""
    out, o = [], 0
    for _, _, s in layout:
        n = numel(s)
        out.append(flat[o:o + n])
        o += n
    return out


class ShardSeries:
    """Per-shard regeneration of a trajectory too large for one GPU's working set
    (C5): shard s of the tensor plan gets its own generator (seed * 1009 + s), so any
    snapshot of any shard can be rebuilt on demand from its seed (the reference
    dynamics above, bf16 draws for C5).  ``load(s, k, ck)`` writes snapshot k of shard s
    and the EMA of its first two gradients into the device checkpoint ``ck``."""

    def __init__(self, torch, layout, plan, seed, device, bf16=False):
        self.torch, self.layout, self.plan = torch, layout, plan
        self.seed, self.device, self.bf16 = int(seed), device, bf16

    def shard_layout(self, s):
        a, b = self.plan[s]
        return self.layout[a:b]

    def load(self, s, k, ck):
        torch = self.torch
        lay = self.shard_layout(s)
        tr = Trajectory(torch, layout_params(lay), self.seed * 1009 + s, self.device,
                        bf16=self.bf16)
        w = None
        for _ in range(k + 1):
            w = tr.next()
        if len(tr.grads) < 2:
            tr.next()
        ema = tr.ema()
        ck.set_weights(tensor_ptrs(w.data_ptr(), lay))
        ck.set_ema(tensor_ptrs(ema.data_ptr(), lay))
        del tr, w, ema
