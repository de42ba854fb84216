"""C-ABI tests that need no GPU: the library loads, exports every symbol
include/dvw.h declares, and rejects bad configurations before touching CUDA."""
import ctypes
import os
import re

import pytest

from paper_1702_07825_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1702_07825_b200 import build
    build.build()
    from paper_1702_07825_b200 import _lib
    return _lib


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "dvw.h")).read()
    return sorted(set(re.findall(r"DVW_API\s+[\w\s\*]+?\b(dvwc?_\w+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert len(names) == 26, names
    raw = ctypes.CDLL(lib.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), n
    assert sorted(lib.EXPORTS) == names


def test_weights_numel_matches_roster(lib):
    for cfg in (synth.C1, synth.C2, synth.C3, synth.C4, synth.Config(3, 32, 128)):
        assert lib.weights_numel(cfg.n_layers, cfg.residual, cfg.skip) == synth.weights_numel(cfg)
    assert lib.weights_numel(0, 64, 128) == -1
    assert lib.weights_numel(2, 64, 128, levels=128) == -1


@pytest.mark.parametrize("kw,status", [
    (dict(n_layers=0, residual=64, skip=128), "DVW_E_SHAPE"),
    (dict(n_layers=2, residual=48, skip=128), "DVW_E_UNSUPPORTED"),
    (dict(n_layers=2, residual=64, skip=100), "DVW_E_UNSUPPORTED"),
    (dict(n_layers=2, residual=64, skip=128, levels=128), "DVW_E_UNSUPPORTED"),
    (dict(n_layers=2, residual=64, skip=128, dilations=[1, 0]), "DVW_E_SHAPE"),
])
def test_create_rejects_bad_config(lib, kw, status):
    with pytest.raises(lib.DvwError) as ei:
        lib.Model(**kw)
    assert ei.value.name == status
    assert lib.last_error()


def test_null_arguments(lib):
    assert lib.raw_call("dvw_create", None, None) == 1
    assert lib.raw_call("dvw_sync", None) == 1
    assert lib.raw_call("dvw_load_weights", None, None, 0, 0) == 1
    assert lib.raw_call("dvw_generate", None, None, 0, 1, None, 1, 1, None, None) == 1
    assert lib.raw_call("dvw_set_kernel", None, 0) == 1
    assert lib.raw_call("dvw_set_precision", None, 0) == 1
    assert lib.raw_call("dvw_set_weight_bits", None, 16) == 1
    assert lib.raw_call("dvw_set_weight_quant", None, 16, 1) == 1
    assert lib.raw_call("dvw_set_sampler", None, 0, ctypes.c_float(1.0), 1) == 1
    lib._lib.dvw_destroy(None)  # no-op
    assert "NULL" in lib.last_error()


def test_product_path_has_no_oracle_dependency():
    """The product package must not import or link anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_1702_07825_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", text, re.M), f
                assert not re.search(r'#include\s*[<"][^>"]*oracle', text), f
                assert "liboracle" not in text, f


def test_conditioner_abi_without_gpu(lib):
    assert lib.conditioner_numel(227, 64, 20, 64) > 0
    assert lib.raw_call("dvwc_create", None, None) == 1
    assert lib.raw_call("dvwc_load_weights", None, None, 0, 0) == 1
    assert lib.raw_call("dvwc_run", None, None, 1, 1, None, None) == 1
    lib._lib.dvwc_destroy(None)
    assert lib.raw_call("dvw_session_create", None, 1, None) == 1
    assert lib.raw_call("dvw_session_generate", None, None, None, 0, 1, None, 0, None, None) == 1
    assert lib.raw_call("dvw_session_position", None) == -1
    lib._lib.dvw_session_destroy(None)
