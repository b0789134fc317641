"""The C-ABI library: every entry point declared in include/knnm.h is
exported by libknnm.so and bound in _lib.SIGNATURES; without a GPU the
engine fails loudly instead of falling back to the CPU."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "knnm.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(knnm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_api():
    names = declared()
    for must in ("knnm_create", "knnm_set_dataset", "knnm_begin", "knnm_load_graph",
                 "knnm_insert_rows", "knnm_round", "knnm_phi", "knnm_export"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1908_00814_b200 import _lib

    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (knnm_[a-z_0-9]+)", out))
    for name in declared():
        assert name in exported, f"{name} declared in knnm.h but not exported"
        assert hasattr(lib, name)
    assert set(_lib.SIGNATURES) == set(declared())


def test_library_is_sm100a():
    from paper_1908_00814_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_string():
    from paper_1908_00814_b200 import _lib

    lib = _lib.load()
    assert lib.knnm_version() >= 1
    assert isinstance(lib.knnm_last_error(), bytes)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1908_00814_b200 import _lib
    from paper_1908_00814_b200.engine import Engine

    with pytest.raises((_lib.KnnmError, ValueError)):
        Engine(0)
