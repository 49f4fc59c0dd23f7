"""Restore-path driver: C2 records (GPT-2-small layout), then decode_delta_record +
dequantize with per-kernel timing.  DQTG_TIMELINE=1 adds the launch timeline."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_11800_b200 import workloads as W  # noqa: E402


def main():
    import torch

    from paper_2306_11800_b200 import engine as E

    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    dev = torch.device("cuda", 0)
    eng = E.Engine(0, torch.cuda.current_stream(dev).cuda_stream)
    layout = W.gpt2_small_layout()
    names = [n for n, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    N = sum(W.numel(s) for s in shapes)
    snaps, ema = W.series(torch, layout, steps + 2, 1234, dev)
    cfg = E.Config()
    recs, prev = [], None
    for i, s in enumerate(snaps):
        c = E.DevCheckpoint(eng, names, types, shapes)
        c.set_weights(W.tensor_ptrs(s.data_ptr(), layout))
        c.set_ema(W.tensor_ptrs(ema.data_ptr(), layout))
        st = eng.quantize(c, cfg, 1, i)
        recs.append(eng.encode_record(st, prev))
        prev = st
    out = torch.empty(N, dtype=torch.float32, device=dev)
    optr = E._ptr_array(W.tensor_ptrs(out.data_ptr(), layout))
    dec = eng.decode_record(recs[0])
    dec = eng.decode_record(recs[1], base=dec)
    if os.environ.get("DQTG_CHAIN"):  # Chain::restore timing through decode_chain
        def deq(k, h):
            E._check(E.LIB.dqtg_dequantize(eng.h, h, optr))
        for rep in range(3):
            t = time.perf_counter()
            d = eng.decode_chain(recs[2:], base=dec, on_state=deq)
            eng.sync()
            dt = time.perf_counter() - t
            print(f"chain pass {rep}: {1e3 * dt / len(recs[2:]):.2f} ms/record, "
                  f"{4.0 * N * len(recs[2:]) / dt / 1e9:.1f} GB/s fp32 out", flush=True)
        return
    eng.profile(True)
    for rec in recs[2:]:
        t = time.perf_counter()
        dec = eng.decode_record(rec, base=dec)
        t1 = time.perf_counter()
        E._check(E.LIB.dqtg_dequantize(eng.h, dec.h, optr))
        eng.sync()
        print(f"decode {1e3 * (t1 - t):.2f} ms + dequantize {1e3 * (time.perf_counter() - t1):.2f} ms, "
              f"record {len(rec)} B")
    for k, v in sorted(eng.profile_report().items(), key=lambda kv: -kv[1][1]):
        print(f"  {k}: {v[0]} launches {v[1]:.3f} ms")


if __name__ == "__main__":
    main()
