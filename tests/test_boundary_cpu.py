"""CPU-side checks of the drop-in boundary (no GPU needed).

* libdqtg.so exports every entry point include/dqtg.h declares;
* the C++ drop-in library and the Python module load and expose the reference
  module's names (bindings/py_module.cpp:50-391);
* without a GPU the product fails loudly instead of falling back to the CPU.
"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dqtg.h")

REFERENCE_MODULE_NAMES = """Error ChainCorrupt ChecksumMismatch UnknownStep ExternalEvaluatorFailed
TooFewDistinctPoints LayerType PruneMetric NamedTensor Checkpoint write_checkpoint read_checkpoint
LayerRule default_layer_rules load_layer_rules classify_layer_type apply_layer_rules Histogram Sketch
sketch_build sketch_merge sketch_quantile EmaState ema_init ema_update ema_save ema_load ScoreSet
compute_scores QuantConfig approx_kmeans ProtectedEntry QuantizedTensor QuantizedCheckpoint
quantize_checkpoint dequantize_checkpoint encode_delta_record decode_delta_record ChainEntry Chain
TrajectorySpec TrajectoryStep generate_trajectory default_layout ConfigCube SearchParams SearchOutcome
Evaluator ProxyEvaluator ExternalEvaluator guided_exhaustive_search delta_neighborhood_search
estimate_compression proxy_quality_delta""".split()


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dqtg_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2306_11800_b200 import engine

    lib = ctypes.CDLL(engine.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_module_surface():
    from paper_2306_11800_b200 import dqt

    missing = [n for n in REFERENCE_MODULE_NAMES if not hasattr(dqt, n)]
    assert not missing, missing
    cfg = dqt.QuantConfig(bins=8, embed_bins=16, prune_frac=0.1, protect_frac=0.01)
    assert (cfg.bins, cfg.embed_bins, cfg.prune_frac, cfg.protect_frac) == (8, 16, 0.1, 0.01)
    assert cfg.metric == dqt.PruneMetric.MAGNITUDE and cfg.sigma == 0.2 and cfg.alpha == 0.01
    assert dqt.SearchParams().threshold == 0.05 and dqt.ConfigCube().grid_size() == 108


def test_host_only_pieces_work_on_cpu(tmp_path):
    """Container I/O, layer rules and sketch bookkeeping are host code."""
    import numpy as np

    from paper_2306_11800_b200 import dqt

    c = dqt.Checkpoint()
    c.step = 3
    c.add_tensor("enc.attn.weight", np.arange(6, dtype=np.float32).reshape(2, 3),
                 dqt.LayerType.ATTENTION)
    c.meta = {"run": "x"}
    p = str(tmp_path / "c.dqt")
    dqt.write_checkpoint(p, c)
    assert dqt.read_checkpoint(p) == c
    rules = dqt.default_layer_rules()
    assert dqt.classify_layer_type("block0.conv1.weight", rules) == dqt.LayerType.CONV
    s = dqt.Sketch(0.01)
    s.add(1.0)
    s.add(-2.0)
    assert s.total() == 2 and s.bucket_count() == 2
    with pytest.raises(dqt.Error):
        dqt.Sketch(0.0)


def test_no_silent_cpu_fallback():
    """Without a B200 every device entry point raises instead of computing on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2306_11800_b200 import engine

    with pytest.raises(engine.EngineError):
        engine.Engine(0)
