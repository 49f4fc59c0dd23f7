#!/usr/bin/env python3
"""Benchmark: checkpoint compress + delta-encode throughput (fp32-in GB/s) on B200.

Workload (BASELINE.json configs[1], "C2"): GPT-2-small layout (124,439,808 fp32
params, 148 tensors, layer types per SURVEY.md §8d), a synthetic training
trajectory generated on the GPU with the reference generator's dynamics
(paper_2306_11800_b200/workloads.py: w0 = 0.05 N(0,1); g = w + 0.0025 N(0,1);
w -= lr g; lr = 0.1 * 0.9^t, trajectory.cpp:75-113), gradient EMA over the first
two gradients (the reference's ema_update arithmetic), default QuantConfig (bins 16, embed 32, prune 0, protect 0.005, MAGNITUDE, sigma 0.2,
alpha 0.01).  One step = compute_scores (fused) + quantize_checkpoint +
encode_delta_record against the previous snapshot's quantized state — the
Chain::append path — for the next snapshot of the series.

value: device-resident (weights + EMA in HBM, previous levels in HBM, record
produced in HBM), CUDA events on the engine stream, max over ranks.
e2e:   same step through the C ABI with HOST buffers: pinned weights H2D, the
step, record D2H, every step.
Inputs per step (1 GB of weights+EMA) exceed the 126 MB L2, so no flush is needed.

--impl reference: the unmodified reference library (oracle/_ref, compiled from
/root/reference/proj sources) on the host cores, on the SAME workload and the
SAME input bytes (the series is generated with the same seed by the same torch
generator on the GPU and copied to the host): compute_scores + quantize_checkpoint
+ encode_delta_record per step, W warm-up then K timed steps, same metric.  The
reference's compress path is single-threaded, so it uses one core.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "checkpoint compress+delta GB/s (fp32 in)"

# ---------------------------------------------------------------------------- workload
from paper_2306_11800_b200 import workloads as W  # noqa: E402

gpt2_small_layout = W.gpt2_small_layout
numel = W.numel
SEED = 1234  # rank r generates its shard's series with seed SEED + r


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def read_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []
        self.cpu = [0, 0]  # host CPU jiffies: steal, total (hypervisor steal of the VM)

    @staticmethod
    def _cpu_stat():
        try:
            with open("/proc/stat") as f:
                v = [int(x) for x in f.readline().split()[1:]]
            return v[7] if len(v) > 7 else 0, sum(v)
        except Exception:
            return 0, 0

    def merge(self, other):
        self.lines += other.lines
        self.cpu = [a + b for a, b in zip(self.cpu, other.cpu)]
        return self

    def __enter__(self):
        self._c0 = self._cpu_stat()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        c1 = self._cpu_stat()
        self.cpu = [self.cpu[0] + c1[0] - self._c0[0], self.cpu[1] + c1[1] - self._c0[1]]
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        steal = self.cpu[0] / self.cpu[1] if self.cpu[1] else None
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "host_cpu_steal_frac": steal}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm), "host_cpu_steal_frac": steal}


# ---------------------------------------------------------------------------- reference arm
def reference_chain(n_timed, n_warm, seed=SEED, cpu_seconds=None):
    """The reference (oracle/_ref) on the C2 chain of the GPU arm, same bytes.

    Snapshot 0 is quantized untimed (the chain's FULL base, as in our arm); step i
    (i = 1 ...) = compute_scores + quantize_checkpoint + encode_delta_record(q_i,
    q_{i-1}) of snapshot i, timed from the reference's Python API.  Returns
    (per-step seconds of the timed steps, params, mean record bytes, same_bytes)."""
    import torch

    from oracle import ref as R

    if not R.available():
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    d = R.load()
    layout = gpt2_small_layout()
    N = W.layout_params(layout)
    gpu = torch.cuda.is_available()
    dev = torch.device("cuda", 0) if gpu else torch.device("cpu")
    tr = W.Trajectory(torch, N, seed, dev)

    def host_ckpt(x, step):
        host = x.cpu().numpy()
        c = d.Checkpoint()
        c.step = step
        for (name, lt, shape), v in zip(layout, W.split(host, layout)):
            c.add_tensor(name, v.reshape(shape), d.LayerType(lt))
        return c

    s0, s1 = tr.next(), tr.next()
    ema = d.ema_init(0.9)
    for k, g in enumerate(tr.grads):
        d.ema_update(ema, host_ckpt(g, k + 1))
    tr.grads = []
    cfg = d.QuantConfig()
    c = host_ckpt(s0, 0)
    q_prev = d.quantize_checkpoint(c, d.compute_scores(c, ema), cfg, 1)
    ts, rec = [], []
    pending = s1
    t_end = None if cpu_seconds is None else time.perf_counter() + cpu_seconds
    i = 0
    while True:
        i += 1
        if i > n_warm + n_timed and (t_end is None or time.perf_counter() >= t_end):
            break
        snap = pending if pending is not None else tr.next()
        pending = None
        c = host_ckpt(snap, i)
        del snap
        t = time.perf_counter()
        q = d.quantize_checkpoint(c, d.compute_scores(c, ema), cfg, 1)
        r = d.encode_delta_record(q, q_prev)
        dt = time.perf_counter() - t
        if i > n_warm:
            ts.append(dt)
            rec.append(len(r))
        q_prev = q
        del c
    return ts, N, float(np.mean(rec)), gpu


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ts, N, rec_mean, same = reference_chain(args.steps, args.warmup)
    t = sum(ts)
    value = 4.0 * N * len(ts) / t / 1e9
    sample = (f"C2 full ({N} params), {args.warmup} warm-up + {len(ts)} timed steps of "
              f"compute_scores+quantize_checkpoint+encode_delta_record, oracle/_ref, 1 thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / len(ts),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (GPU trajectory with the reference generator dynamics)",
        "config": {"workload": "C2: GPT-2-small layout 124.4M fp32 params, delta chain",
                   "params_per_gpu": N, "quant_config": "default (bins16/embed32/"
                   "protect0.005/MAGNITUDE/sigma0.2/alpha0.01), EMA sensitivity",
                   "same_config": True, "same_bytes": same, "seed": SEED,
                   "record_bytes": rec_mean, "compression_ratio": 4.0 * N / rec_mean},
        "cpu_baseline": dict({"value": value, "unit": "GB/s", "cores": 1, "kind": "reference",
                              "sample": sample}, **cpu_info()),
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
ALGO_BYTES = {  # algorithmic HBM bytes per parameter per launch
    # fused pass C + sparse DELTA tile pass (compress_step): read w, the protected
    # bitmap (1/8 B) and the previous levels, write the target levels once
    "quant_delta_kernel": 4.0 + 0.125 + 2.0 + 2.0,
    "pass_a2_kernel": 8.0,  # read w + EMA (score histograms + protected candidates)
    "pass_b_kernel": 8.25,  # read w + EMA, write 2-bit partition codes
    "pass_c_kernel": 6.25,  # read w + partition codes, write levels
    "enc_tile_delta_kernel": 4.0,  # read levels + previous levels
    "enc_tile_kernel": 4.0,  # read levels + previous levels
}
# span name -> kernel name in the ncu report (profiles/ncu_traffic.json)
NCU_NAME = {"quant_delta_kernel": "enc_tile_delta_kernel"}


def write_dqt1(path, layout, flat, step=0):
    """write_checkpoint (src/tensor.cpp:77-98) of one flat snapshot."""
    import struct

    with open(path, "wb") as f:
        f.write(b"DQT1" + struct.pack("<IQI", 1, step, 0) + struct.pack("<I", len(layout)))
        o = 0
        for name, lt, shape in layout:
            nb = name.encode()
            f.write(struct.pack("<H", len(nb)) + nb + struct.pack("<BB", lt, len(shape)))
            f.write(b"".join(struct.pack("<Q", d) for d in shape))
            n = numel(shape)
            f.write(memoryview(np.ascontiguousarray(flat[o:o + n], np.float32)).cast("B"))
            o += n


def measure_ingest(eng, layout, flat, cpu=True, reps=3):
    import tempfile

    fd, path = tempfile.mkstemp(suffix=".dqt")
    os.close(fd)
    try:
        write_dqt1(path, layout, flat, step=1)
        size = os.path.getsize(path)
        ck, _, _ = eng.read_dqt1(path)  # warm: pinned staging, page cache
        got = ck.download()
        ok = all(np.array_equal(g.view(np.uint32), flat[o:o + g.size].view(np.uint32))
                 for g, o in zip(got, np.cumsum([0] + [g.size for g in got])[:-1]))
        del ck, got
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            ck, _, _ = eng.read_dqt1(path)
            ts.append(time.perf_counter() - t)
            del ck
        out = {"value": size / min(ts) / 1e9, "unit": "GB/s (DQT1 file -> HBM)",
               "file_bytes": size, "ms": 1e3 * min(ts), "bit_exact": bool(ok),
               "timing": f"best of {reps} reads, host wall clock, page cache warm",
               "path": "Engine.read_dqt1: host header parse, 8 reader threads, pinned 4 MiB "
                       "chunks -> cudaMemcpyAsync, device NaN/Inf check; page cache warm"}
        if cpu:
            from oracle import ref as R

            if R.available():
                d = R.load()
                t = time.perf_counter()
                d.read_checkpoint(path)
                tr = time.perf_counter() - t
                out["cpu_reference"] = {"value": size / tr / 1e9, "unit": "GB/s",
                                        "kind": "reference", "cores": 1,
                                        "sample": "oracle/_ref read_checkpoint of the same file"}
        return out
    finally:
        os.unlink(path)


tensor_ptrs = W.tensor_ptrs


def host_checkpoint(d, layout, flat, step=0):
    """A Checkpoint of the given module (ours: dqt; the reference: dqtref) from one
    flat host array."""
    c = d.Checkpoint()
    c.step = step
    for (name, lt, shape), v in zip(layout, W.split(flat, layout)):
        c.add_tensor(name, v.reshape(shape), d.LayerType(lt))
    return c


def measure_c3(torch, dev, cpu_ref=True, ref_layers=1):
    """BASELINE configs[2] (C3): guided_exhaustive_search (search.cpp:380-385) over the
    default ConfigCube on a BERT-large checkpoint (335,141,888 params, synthetic, EMA
    sensitivity), threshold 0.1, parallelism = nproc, through the drop-in module with
    the device ProxyEvaluator (batched candidate evaluation).  The reference's
    ProxyEvaluator::evaluate (search.cpp:107-112) is timed on a bounded sample of the
    same bytes (embeddings + ref_layers encoder layers)."""
    from paper_2306_11800_b200 import dqt

    layout = W.bert_large_layout()
    N = W.layout_params(layout)
    tr = W.Trajectory(torch, N, SEED + 100, dev)
    w = tr.next()
    tr.next()
    ema = tr.ema().cpu().numpy()
    wh = w.cpu().numpy()
    del w, tr
    nproc = os.cpu_count() or 1
    c = host_checkpoint(dqt, layout, wh, 1)
    e = dqt.ema_init(0.9)
    dqt.ema_update(e, host_checkpoint(dqt, layout, ema, 1))  # first update copies
    scores = dqt.compute_scores(c, e)
    ev = dqt.ProxyEvaluator()
    params = dqt.SearchParams(threshold=0.1, parallelism=nproc, seed=1)
    t = time.perf_counter()
    out = dqt.guided_exhaustive_search(c, scores, dqt.ConfigCube(), ev, params)
    dt = time.perf_counter() - t
    res = {"workload": "C3: BERT-large 335.1M fp32 params, guided_exhaustive_search threshold 0.1, "
                       f"parallelism {nproc}, default ConfigCube",
           "params": N, "search_s": dt, "evaluations": out.evaluations_used,
           "evals_per_s": out.evaluations_used / dt,
           "eval_gbs": 4.0 * N * out.evaluations_used / dt / 1e9,
           "chosen": {"bins": out.config.bins, "embed_bins": out.config.embed_bins,
                      "prune_frac": out.config.prune_frac, "protect_frac": out.config.protect_frac,
                      "metric": int(out.config.metric)},
           "quality_delta": out.quality_delta, "est_compression": out.est_compression,
           "feasible": out.feasible,
           "path": "dqt.guided_exhaustive_search + dqt.ProxyEvaluator: every EvalCache::prefetch "
                   "batch is one dqtg_eval_batch (shared pass B per partition, 8 candidates per "
                   "read of w); checkpoint resident in HBM across batches; host wall clock"}
    del c, scores, ev
    if cpu_ref:
        from oracle import ref as R

        d = R.load()
        sub = [x for x in layout if x[0].startswith("bert.embeddings")]
        for i in range(ref_layers):
            sub += [x for x in layout if x[0].startswith(f"bert.encoder.layer.{i}.")]
        names = {x[0] for x in sub}
        pick = [v for (n, _, _), v in zip(layout, W.split(wh, layout)) if n in names]
        pick_e = [v for (n, _, _), v in zip(layout, W.split(ema, layout)) if n in names]
        Ns = sum(int(v.size) for v in pick)
        rc = host_checkpoint(d, sub, np.concatenate(pick), 1)
        re_ = d.ema_init(0.9)
        d.ema_update(re_, host_checkpoint(d, sub, np.concatenate(pick_e), 1))
        rs = d.compute_scores(rc, re_)
        cfg = d.QuantConfig()
        t = time.perf_counter()  # ProxyEvaluator::evaluate (search.cpp:107-112), step by step
        q = d.quantize_checkpoint(rc, rs, cfg, 1)
        d.proxy_quality_delta(rc, d.dequantize_checkpoint(q))
        d.estimate_compression(rc, q)
        tr_ = time.perf_counter() - t
        one = 4.0 * Ns / tr_ / 1e9
        res["cpu_reference"] = {
            "value": one, "unit": "GB/s per evaluation, 1 thread", "kind": "reference", "cores": 1,
            "ideal_parallel_gbs": one * nproc, "nproc": nproc, "eval_s": tr_,
            "sample": f"ProxyEvaluator::evaluate (quantize + dequantize + proxy_quality_delta + "
                      f"estimate_compression), default QuantConfig, BERT-large embeddings + "
                      f"{ref_layers} encoder layer(s) ({Ns} params) of the same bytes"}
        res["speedup_vs_reference_ideal_parallel"] = res["eval_gbs"] / (one * nproc)
    return res


def measure_big(torch, dev, steps=2):
    """BASELINE configs[3] / [4] on ONE B200 (the driver's GPUs are single).
    C4 (GPT-2 XL, 1.56 B params): the whole-checkpoint chain (FULL, then DELTA steps)
    on one engine, CUDA-synchronised wall time of quantize + encode per DELTA step; the
    same snapshots as 8 tensor shards (shards.LocalShardedChain, the 8-GPU split)
    give byte-identical records.  C5 (Llama-3-8B, 8.03 B params, bf16 draws upcast):
    8 tensor shards on one engine, inputs regenerated per stage (excluded from the
    time), FULL + DELTA, every shard record decoded back on the device."""
    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200 import shards as S

    out = {}
    eng = E.Engine(0, torch.cuda.current_stream(dev).cuda_stream)
    cfg = E.Config()
    lay = W.gpt2_xl_layout()
    names, types, shapes = ([x[i] for x in lay] for i in range(3))
    N = W.layout_params(lay)
    snaps, ema = W.series(torch, lay, steps + 1, SEED + 4, dev)
    offs = np.concatenate([[0], np.cumsum([W.numel(s) for s in shapes])])
    whole, prev, ts = [], None, []
    for k, w in enumerate(snaps):
        ck = E.DevCheckpoint(eng, names, types, shapes)
        ck.set_weights(W.tensor_ptrs(w.data_ptr(), lay))
        ck.set_ema(W.tensor_ptrs(ema.data_ptr(), lay))
        torch.cuda.synchronize()
        t = time.perf_counter()
        st, rh = eng.compress_step(ck, cfg, 1, k, base=prev)
        eng.sync()
        if k:
            ts.append(time.perf_counter() - t)
        whole.append(E.Engine.record_bytes(rh))
        prev = st
        del ck
    del prev
    ch = S.LocalShardedChain(eng, names, types, shapes, 8, cfg, seed=1, device=dev)
    same = True
    for k in range(len(snaps)):
        def load(s, ck, k=k):
            a, b = ch.plan[s]
            ck.set_weights(W.tensor_ptrs(snaps[k].data_ptr() + 4 * int(offs[a]), lay[a:b]))
            ck.set_ema(W.tensor_ptrs(ema.data_ptr() + 4 * int(offs[a]), lay[a:b]))
        recs, rt = ch.step(k, load)
        same &= ch.assemble(recs) == whole[k] and all(rt)
    out["c4"] = {"workload": "C4: GPT-2 XL 1,557,611,200 fp32 params, delta chain, 1 GPU",
                 "params": N, "value": 4.0 * N / float(np.median(ts)) / 1e9, "unit": "GB/s",
                 "ms_per_step": 1e3 * float(np.median(ts)), "steps": len(ts),
                 "record_bytes_full": len(whole[0]), "record_bytes_delta": len(whole[-1]),
                 "sharded_8_records_identical_and_roundtrip": bool(same),
                 "timing": "compress_step (quantize + encode_delta_record) wall time, device synced"}
    del snaps, ema, ch, whole
    gc.collect()
    eng.trim()
    torch.cuda.empty_cache()
    lay = W.llama3_8b_layout()
    names, types, shapes = ([x[i] for x in lay] for i in range(3))
    N = W.layout_params(lay)
    if os.environ.get("DQTG_C5_OWN_STREAM"):  # diagnostics: the engine on a private stream
        eng = E.Engine(0)
    ch = S.LocalShardedChain(eng, names, types, shapes, 8, cfg, seed=1, device=dev)
    gen = W.ShardSeries(torch, lay, ch.plan, SEED + 5, dev, bf16=True)
    sizes, rts, tq, td = [], [], [], []
    for k in range(2):
        ch.t_engine, ch.t_decode = 0.0, 0.0
        recs, rt = ch.step(k, lambda s, ck, k=k: gen.load(s, k, ck), keep_records=False)
        sizes.append(int(sum(recs)))
        rts.append(bool(all(rt)))
        tq.append(ch.t_engine)
        td.append(ch.t_decode)
    out["c5"] = {"workload": "C5: Llama-3-8B 8,030,261,248 params (bf16 draws upcast to fp32), "
                             "8 tensor shards on 1 GPU",
                 "params": N, "compress_gbs_delta": 4.0 * N / tq[1] / 1e9,
                 "compress_s": tq, "decompress_gbs_delta": 4.0 * N / td[1] / 1e9,
                 "decompress_s": td, "record_bytes": sizes, "roundtrip_identical": rts,
                 "timing": "engine calls only (per-stage input regeneration excluded), FULL "
                           "then DELTA; decompress = decode_delta_record on the device + "
                           "state comparison"}
    del ch, gen
    gc.collect()
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # --share-gpu (testing the N>1 path on one GPU): every rank on device 0, gloo
    gpu = 0 if args.share_gpu else local
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    local = gpu

    from paper_2306_11800_b200 import engine as E

    stream = torch.cuda.current_stream(dev)
    eng = E.Engine(local, stream.cuda_stream)
    layout = gpt2_small_layout()
    if world > 1:  # one GPT-2-small-sized shard per rank of one sharded checkpoint
        layout = [(f"shard{rank}.{n}", t, s) for n, t, s in layout]
    names = [n for n, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    N = sum(numel(s) for s in shapes)
    cfg = E.Config()
    n_snap = args.warmup + args.steps + 1

    snaps, ema = W.series(torch, layout, n_snap, SEED + rank, dev)
    torch.cuda.synchronize()
    ckpts = []
    for s in snaps:
        c = E.DevCheckpoint(eng, names, types, shapes)
        c.set_weights(tensor_ptrs(s.data_ptr(), layout))
        c.set_ema(tensor_ptrs(ema.data_ptr(), layout))
        ckpts.append(c)
    host_snaps = [s.cpu().numpy() for s in snaps[:3]]
    del snaps
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # FULL record for snapshot 0, then a chain of DELTA records.  N=1: the fused
    # C-ABI step; N>1: the tensor-sharded path (score/value histograms all-reduced
    # over NCCL, each rank encodes its own tensor blocks).
    rec_bytes = []
    comm = None
    if world > 1:
        from paper_2306_11800_b200 import distributed as DIST

        # the engine library's own NCCL communicator (dqtg_comm_*): histogram
        # all-reduces and the record gather on the engine stream; --share-gpu (all
        # ranks on one GPU, where NCCL refuses duplicate devices) uses torch/gloo
        if not args.share_gpu:
            comm = DIST.make_comm(eng)
        state, _, _ = DIST.compress_sharded(eng, ckpts[0], cfg, 1, 0, None, device=dev,
                                            n_tensors_total=len(names) * world, comm=comm)

        def step(i, prev):
            st, _, stats = DIST.compress_sharded(eng, ckpts[i], cfg, 1, i, prev, device=dev,
                                                 n_tensors_total=len(names) * world, comm=comm)
            # record bytes per rank's share: the whole record (rank 0) / world
            n = stats.get("record_bytes") or stats.get("record_bytes_local") or 0
            rec_bytes.append(n / world if comm is not None else n)
            return st
    else:
        state = eng.quantize(ckpts[0], cfg, 1, 0)

        def step(i, prev):
            st, r = eng.compress_step(ckpts[i], cfg, 1, i, prev)
            rec_bytes.append(E.LIB.dqtg_record_size(r))
            E.LIB.dqtg_record_destroy(r)
            return st

    for i in range(1, args.warmup + 1):
        state = step(i, state)
    barrier()
    launches0 = eng.launches
    syncs0 = eng.sync_stats()[0]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    mark = (lambda m: print(m, file=sys.stderr, flush=True)) if os.environ.get("DQTG_SYNC_TRACE") \
        else (lambda m: None)
    # no Python garbage collection pauses inside the timed regions (the host thread
    # drives the sequential chain between C calls)
    gc.collect()
    gc.disable()
    with ClockSampler(local) as clocks:
        mark("MARK sequential begin")
        t0.record(stream)
        for i in range(args.warmup + 1, args.warmup + 1 + args.steps):
            state = step(i, state)
        t1.record(stream)
        barrier()
        mark("MARK sequential end")
    ms = t0.elapsed_time(t1)
    gc.enable()
    launches = eng.launches - launches0
    syncs_per_step = (eng.sync_stats()[0] - syncs0) / args.steps
    ms_sequential = ms

    # pipelined chain (N=1): a pool of worker streams, step k on worker k mod W;
    # encode(k) waits on quantize(k-1) (paper_2306_11800_b200/pipeline.py)
    pipelined = None
    pipe_comms = None
    if (world == 1 or comm is not None) and not args.no_pipeline:
        from paper_2306_11800_b200.pipeline import ChainCompressor

        if comm is not None:  # one communicator per worker (dqtg_pipe_set_comms)
            pipe_comms = [DIST.make_comm(eng) for _ in range(args.workers)]
        # every run forks from / joins into `stream`: CUDA events on it time the chain
        cc = ChainCompressor(local, workers=args.workers, stream=stream.cuda_stream,
                             comms=pipe_comms, n_tensors_total=len(names) * world)
        torch.cuda.synchronize()
        # warm-up: at least two steps per worker (scratch and pool sizes settle)
        n_warm = max(args.warmup + 1, 2 * args.workers + 2)
        warm = [ckpts[j % (args.warmup + 1)] for j in range(n_warm - 1)] + [ckpts[args.warmup]]
        base = cc.run(warm, cfg, 1, list(range(n_warm)))
        # one untimed pass over the timed snapshots (first-pass pool/scheduling effects)
        cc.run(ckpts[args.warmup + 1:], cfg, 1, list(range(args.warmup + 1, n_snap)), base=base)
        torch.cuda.synchronize()
        # three timed passes of exactly K steps each; the median is reported (the
        # worker threads share the host CPU with the rest of the VM)
        pipe_reps, pipe_wall = [], []
        gc.collect()
        gc.disable()
        clocks_p = ClockSampler(local)
        clocks_p.__enter__()
        for _ in range(3):
            l0 = cc.launches
            torch.cuda.synchronize()
            tp0 = time.perf_counter()
            t0.record(stream)
            cc.run(ckpts[args.warmup + 1:], cfg, 1, list(range(args.warmup + 1, n_snap)), base=base)
            t1.record(stream)
            torch.cuda.synchronize()
            pipe_wall.append((time.perf_counter() - tp0) * 1e3)
            pipe_reps.append(t0.elapsed_time(t1))
            launches_p = cc.launches - l0
        clocks_p.__exit__(None, None, None)
        gc.enable()
        clocks.merge(clocks_p)
        pipelined = sorted(pipe_reps)[1]
        del base, cc
    if pipelined is not None and pipelined < ms:
        ms = pipelined
        launches = launches_p
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    value = 4.0 * N * world * args.steps / (ms / 1e3) / 1e9
    rec_mean = float(np.mean(rec_bytes[-args.steps:]))
    cr = 4.0 * N / rec_mean if rec_mean else None  # per-rank share of the record vs per-rank fp32 bytes

    # live per-kernel timing (CUDA events on the engine stream) for the roofline
    eng.profile(True)
    prof_steps = min(3, args.steps)
    for i in range(prof_steps):
        state = step(args.warmup + 1 + (i % args.steps), state)
    eng.sync()
    prof = eng.profile_report()
    eng.profile(False)
    peak, peak_kind = read_peak()
    tot_ms = sum(v[1] for v in prof.values())
    dom = max((k for k in prof if k in ALGO_BYTES), key=lambda k: prof[k][1])
    n_l, dom_ms = prof[dom]
    dom_avg_s = dom_ms / n_l / 1e3
    achieved = ALGO_BYTES[dom] * N / dom_avg_s / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(NCU_NAME.get(dom, dom))
    except Exception:
        pass
    step_algo = (12.0 + 4.0 / cr) * N  # SURVEY.md §8d, sensitivity present
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                "kernel_share_of_step": dom_ms / tot_ms if tot_ms else None,
                "step_algorithmic_gbs": step_algo / (ms_step / 1e3) / 1e9,
                "step_frac": step_algo / (ms_step / 1e3) / 1e9 / peak,
                "kernels_ms_per_step": {k: round(v[1] / prof_steps, 4) for k, v in
                                        sorted(prof.items(), key=lambda kv: -kv[1][1])}}

    # e2e through the public API with HOST buffers: every step copies that step's
    # weights from pinned host memory (H2D) and reads its record back into pinned
    # host memory (D2H).  N=1: the worker-pool chain compressor (copies overlap the
    # other workers' kernels); N>1: the tensor-sharded path.
    pinned = [torch.from_numpy(h).pin_memory() for h in host_snaps]
    e2e_steps = max(6, min(args.steps, 12))
    h2d = d2h = 0
    if world == 1:
        from paper_2306_11800_b200.pipeline import ChainCompressor

        cc = ChainCompressor(local, workers=args.workers)
        host = (names, types, shapes, tensor_ptrs(ema.data_ptr(), layout))
        rec_host = [torch.empty(int(4 * N), dtype=torch.uint8).pin_memory()
                    for _ in range(cc.nw)]
        d2h_l = []

        def grab(k, r):
            n = E.LIB.dqtg_record_size(r)
            E._check(E.LIB.dqtg_record_copy(r, rec_host[k % cc.nw].data_ptr()))
            d2h_l.append(n)

        def host_series(k0, n):
            return [tensor_ptrs(pinned[(k0 + j) % len(pinned)].data_ptr(), layout)
                    for j in range(n)]

        e2e_base = cc.run(host_series(0, 2 * cc.nw + 2), cfg, 1, list(range(2 * cc.nw + 2)),
                          host=host)
        # one untimed pass over the timed series (first-pass pool/scheduling effects)
        e2e_base = cc.run(host_series(0, e2e_steps), cfg, 1, list(range(2 * cc.nw + 2,
                          2 * cc.nw + 2 + e2e_steps)), base=e2e_base, on_record=grab, host=host)
        # three timed passes of e2e_steps steps; the median is reported
        e2e_reps = []
        gc.collect()
        gc.disable()
        for _ in range(3):
            d2h_l.clear()
            torch.cuda.synchronize()
            te = time.perf_counter()
            cc.run(host_series(2 * cc.nw + 2, e2e_steps), cfg, 1,
                   list(range(2 * cc.nw + 2, 2 * cc.nw + 2 + e2e_steps)), base=e2e_base,
                   on_record=grab, host=host)
            torch.cuda.synchronize()
            e2e_reps.append(time.perf_counter() - te)
        gc.enable()
        e2e_s = sorted(e2e_reps)[1]
        h2d = 4 * N * e2e_steps
        d2h = sum(d2h_l)
        e2e_path = ("ChainCompressor.run(host weights): per step H2D of the pinned snapshot + "
                    "quantize + encode_delta_record + record D2H, worker-pool streams")
        del cc, e2e_base
    else:
        e2e_ck = E.DevCheckpoint(eng, names, types, shapes)
        e2e_ck.set_ema(tensor_ptrs(ema.data_ptr(), layout))
        e2e_ck.set_weights(tensor_ptrs(pinned[0].data_ptr(), layout))
        e2e_state, _, _ = DIST.compress_sharded(eng, e2e_ck, cfg, 1, 0, None, device=dev,
                                                n_tensors_total=len(names) * world, comm=comm)

        def e2e_step(i, prev):
            nonlocal h2d, d2h
            e2e_ck.set_weights(tensor_ptrs(pinned[i % len(pinned)].data_ptr(), layout))
            h2d += 4 * N
            st, rec, stats = DIST.compress_sharded(eng, e2e_ck, cfg, 1, i, prev, device=dev,
                                                   n_tensors_total=len(names) * world,
                                                   gather_record=True, comm=comm)
            # D2H: the whole record on rank 0 (comm), each rank's blocks otherwise
            d2h += (len(rec) // world if rec is not None else 0) if comm is not None \
                else stats["record_bytes_local"]
            return st

        e2e_state = e2e_step(1, e2e_state)
        barrier()
        h2d = d2h = 0
        te = time.perf_counter()
        for i in range(2, 2 + e2e_steps):
            e2e_state = e2e_step(i, e2e_state)
        barrier()
        e2e_s = time.perf_counter() - te
        e2e_path = "dqtg_ckpt_set_weights(pinned host) + sharded compress + record gather"
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e = {"value": 4.0 * N * world * e2e_steps / e2e_s / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps,
           "path": e2e_path}
    if world == 1:
        e2e["reps_gbs"] = [round(4.0 * N * e2e_steps / x / 1e9, 2) for x in e2e_reps]
        e2e["timing"] = f"median of 3 passes of {e2e_steps} steps (host wall clock, device synced)"

    # restore: decode_delta_record + dequantize_checkpoint on the device (the other
    # half of the round trip, Chain::restore replay), records read from host memory
    restore = None
    if world == 1:
        r_steps = min(args.steps, 6)
        st_prev = eng.quantize(ckpts[0], cfg, 1, 0)
        recs = [eng.encode_record(st_prev)]
        for i in range(1, r_steps + 2):
            st_i, r = eng.compress_step(ckpts[i], cfg, 1, i, st_prev)
            buf = np.empty(E.LIB.dqtg_record_size(r), np.uint8)
            E._check(E.LIB.dqtg_record_copy(r, buf.ctypes.data))
            E.LIB.dqtg_record_destroy(r)
            recs.append(buf.tobytes())
            st_prev = st_i
        last_levels = torch.empty(0)
        out = torch.empty(N, dtype=torch.float32, device=dev)
        optr = E._ptr_array(tensor_ptrs(out.data_ptr(), layout))
        dec = eng.decode_record(recs[0])
        dec = eng.decode_record(recs[1], base=dec)  # warm-up
        E._check(E.LIB.dqtg_dequantize(eng.h, dec.h, optr))
        eng.sync()
        dec1 = dec
        restore_reps = []
        gc.collect()
        gc.disable()
        def deq(k, h):  # dequantize_checkpoint of every restored state into HBM
            E._check(E.LIB.dqtg_dequantize(eng.h, h, optr))

        for _ in range(2):  # untimed passes (pinned staging pool, walk threads)
            dec = eng.decode_chain(recs[2:], base=dec1, on_state=deq)
            eng.sync()
        for _ in range(3):  # median of three passes over the same records
            tr = time.perf_counter()
            dec = eng.decode_chain(recs[2:], base=dec1, on_state=deq)
            eng.sync()
            restore_reps.append(time.perf_counter() - tr)
        gc.enable()
        tr = sorted(restore_reps)[1]
        ok = eng.states_equal(dec, st_prev)
        nrec = len(recs) - 2
        restore = {"value": 4.0 * N * nrec / tr / 1e9, "unit": "GB/s (fp32 out)",
                   "reps_gbs": [round(4.0 * N * nrec / x / 1e9, 2) for x in restore_reps],
                   "ms_per_step": 1e3 * tr / nrec, "steps": nrec,
                   "record_bytes": float(np.mean([len(x) for x in recs[2:]])),
                   "levels_match_encoder": ok,
                   "path": "Engine.decode_chain(host DQDR bytes, base) = Chain::restore: the "
                           "host walk of record k+1 overlaps the device decode of record k; "
                           "dqtg_dequantize of every state into HBM"}
        del last_levels

    # ingest: a DQT1 file (read_checkpoint, src/tensor.cpp:110-149) streamed into a device
    # checkpoint through pinned staging (dqtg_ckpt_read_dqt1); page cache warm
    ingest = None
    if world == 1:
        ingest = measure_ingest(eng, layout, host_snaps[0], cpu=not args.no_cpu_baseline)

    c3 = None
    if world == 1 and not args.no_c3:
        del ckpts
        ckpts = None
        torch.cuda.empty_cache()
        c3 = measure_c3(torch, dev, cpu_ref=not args.no_cpu_baseline)

    big = None
    if world == 1 and args.big:
        ckpts = None
        snaps = host_snaps = None
        gc.collect()
        eng.trim()
        torch.cuda.empty_cache()
        big = measure_big(torch, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference on the same C2 chain and bytes, a bounded number of steps
        ckpts = None
        torch.cuda.empty_cache()
        ts, Ns, rec_ref, same = reference_chain(args.cpu_steps, 0)
        v = 4.0 * Ns * len(ts) / sum(ts) / 1e9
        cpu = dict({"value": v, "unit": "GB/s", "cores": 1, "kind": "reference",
                    "sample": f"C2 full ({Ns} params), steps 1..{len(ts)} of the same chain and "
                              f"bytes (compute_scores+quantize_checkpoint+encode_delta_record, "
                              f"oracle/_ref, 1 thread)",
                    "same_bytes": same, "record_bytes": rec_ref,
                    "record_bytes_match_gpu_arm": bool(rec_ref == float(np.mean(rec_bytes[:len(ts)])))
                    if len(rec_bytes) >= len(ts) else None}, **cpu_info())

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (GPU trajectory with the reference generator dynamics)",
            "nccl": None if world == 1 else {
                "nranks": world, "comm": "dqtg_comm (engine-owned NCCL communicator)"
                if comm is not None else "torch.distributed gloo (--share-gpu)",
                "pipeline_comms": len(pipe_comms) if pipe_comms else 0},
            "config": {"workload": "C2: GPT-2-small layout 124.4M fp32 params, delta chain",
                       "params_per_gpu": N, "quant_config": "default (bins16/embed32/"
                       "protect0.005/MAGNITUDE/sigma0.2/alpha0.01), EMA sensitivity",
                       "parallelism": (f"tensor-sharded x{world}, score/value histograms "
                                       f"all-reduced over NCCL" if world > 1 else "1 GPU"),
                       "l2": "inputs (1 GB/step) larger than L2; no flush",
                       "record_bytes": rec_mean, "compression_ratio": cr,
                       "ms_per_step_sequential": ms_sequential / args.steps,
                       "ms_per_step_pipelined": None if pipelined is None else pipelined / args.steps,
                       "ms_per_step_pipelined_reps": None if pipelined is None else
                       [round(x / args.steps, 4) for x in pipe_reps],
                       "host_syncs_per_step": syncs_per_step,
                       "ms_per_step_pipelined_wall": None if pipelined is None else
                       [round(x / args.steps, 4) for x in pipe_wall],
                       "timing": (f"pipelined chain: {args.workers} worker streams (step k on "
                                  f"worker k mod {args.workers}) forked from and joined into the "
                                  f"timing stream, CUDA events on it, median of 3 passes"
                                  if pipelined is not None and ms == pipelined else
                                  "CUDA events on the engine stream")},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "restore": restore,
            "ingest": ingest, "c3_search": c3, "c4_c5": big,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=2,
                    help="timed reference steps of the cpu_baseline leg (~10 s each at C2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 (BERT-large search) leg")
    ap.add_argument("--big", action="store_true",
                    help="add the C4 (GPT-2 XL) and C5 (Llama-3-8B, 8 shards) legs on this GPU")
    ap.add_argument("--workers", type=int, default=4, help="worker streams of the chain pipeline")
    ap.add_argument("--share-gpu", action="store_true",
                    help="test mode for N>1 on one GPU: all ranks on device 0 with gloo")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
