"""CPU checks of the C-ABI library: it loads without a GPU, exports every symbol include/fpdt.h declares,
and its host-only helpers agree with the layout contract.  No compute calls (there is no GPU here)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header="fpdt.h"):
    with open(os.path.join(ROOT, "include", header)) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(fpdt_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2408_16978_b200 import build
    build.build_all()
    from paper_2408_16978_b200 import _lib
    return _lib.load()


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("fpdt_attn_fwd", "fpdt_attn_bwd", "fpdt_ctx_create", "fpdt_ctx_destroy", "fpdt_last_error",
              "fpdt_get_unique_id", "fpdt_global_token"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_lists_every_symbol():
    from paper_2408_16978_b200 import fpdt
    assert sorted(fpdt.EXPORTED) == _declared()


def test_diag_library_is_separate(lib):
    """Diagnostics (micro-benchmarks, direct kernel launches) live in libfpdt_diag.so, not in the product library;
    the product library has no cuBLAS dependency (the projection GEMMs are the library's own kernels)."""
    from paper_2408_16978_b200 import _lib, fpdt
    diag = _lib.load_diag()
    assert sorted(fpdt.DIAG_EXPORTED) == _declared("fpdt_diag.h")
    assert not [n for n in fpdt.DIAG_EXPORTED if not hasattr(diag, n)]
    import subprocess
    so = os.path.join(ROOT, "paper_2408_16978_b200", "libfpdt.so")
    syms = subprocess.run(["nm", "-D", so], capture_output=True, text=True, check=True).stdout
    assert "fpdt_selftest" not in syms and "fpdt_debug" not in syms
    deps = subprocess.run(["readelf", "-d", so], capture_output=True, text=True, check=True).stdout
    assert "cublas" not in deps.lower() and "cublas" not in syms.lower()


def test_global_token_matches_layout_contract(lib):
    import fpdt_inputs as gen
    for p, C, s_local in ((1, 256, 1024), (2, 512, 1024), (4, 1024, 2048), (8, 2048, 2048)):
        for r in range(p):
            ref = gen.global_tokens_of_rank(r, p, s_local, C)
            got = np.array([lib.fpdt_global_token(t, C, p, r) for t in range(0, s_local, 37)])
            assert np.array_equal(got, ref[::37])


def test_no_gpu_fails_loudly(lib):
    """Without a usable GPU, context creation must return an error status (never a silent fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2408_16978_b200 import fpdt
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.FPDTContext()
    assert e.value.code == fpdt.FPDT_ERR_CUDA
    assert lib.fpdt_last_error()


def test_missing_library_raises(tmp_path, monkeypatch):
    from paper_2408_16978_b200 import _lib
    monkeypatch.setattr(_lib, "PKG", str(tmp_path))
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(_lib.FpdtLibraryMissing):
        _lib.load()
