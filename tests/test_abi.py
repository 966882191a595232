"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/taichi_b200.h declares, and its host-side pieces (presets, the
deterministic weight hash) agree with the oracle's restatement."""
import ctypes
import pathlib
import re

import numpy as np
import pytest

from oracle import model_ref as mr

REPO = pathlib.Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (REPO / "include" / "taichi_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:tc_status|const char\*|uint16_t)\s+(tc_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["tc_instance_create", "tc_step_launch", "tc_step_wait", "tc_kv_migrate", "tc_kv_release",
              "tc_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(str(built / "libtaichi_b200.so"))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing


def test_runtime_binding_covers_header(built):
    from paper_2508_01989_b200 import runtime
    assert set(declared_symbols()) == set(runtime.EXPORTED)


@pytest.mark.parametrize("name", ["tiny", "llama3_8b", "qwen2_5_14b", "llama3_8b:L2"])
def test_presets_match_oracle(built, name):
    from paper_2508_01989_b200 import runtime
    d = runtime.model_preset(name).as_dict()
    ref = mr.preset(name).__dict__
    for k, v in ref.items():
        assert d[k] == pytest.approx(v, rel=0, abs=0), k


def test_unknown_preset_reports_error(built):
    from paper_2508_01989_b200 import runtime
    with pytest.raises(runtime.TaichiError, match="unknown model preset"):
        runtime.model_preset("gpt2")


@pytest.mark.parametrize("tid,scale,offset", [(1, 1.0, 0.0), (2, float(mr.LIN_SCALE), 0.0),
                                              (mr.tid_layer(3, 5), float(mr.NORM_SCALE), 1.0),
                                              (mr.tid_layer(0, 7), float(mr.BIAS_SCALE), 0.0)])
def test_weight_hash_matches_oracle(built, tid, scale, offset):
    from paper_2508_01989_b200 import runtime
    lib = runtime.load_library()
    seed = 1234
    ref = mr.gen_bits(seed, tid, 8, 257, np.float32(scale), np.float32(offset)).ravel()
    for i in list(range(0, 2056, 37)) + [2055]:
        assert lib.tc_weight_value(seed, tid, i, scale, offset) == ref[i]


def test_create_without_gpu_fails_loudly(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2508_01989_b200 import runtime
    with pytest.raises(runtime.TaichiError):
        runtime.Instance("tiny")
