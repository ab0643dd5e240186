"""C-ABI library checks that need no GPU: it builds for sm_100a, loads, exports every
symbol include/ganq.h declares, and rejects invalid arguments before touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2501_12956_b200 import _lib
from paper_2501_12956_b200 import build as gbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ganq.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ganq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    gbuild.build()
    return _lib.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("ganq_hessian", "ganq_quantize_layer", "ganq_objective", "ganq_workspace_size",
              "ganq_last_error"):
        assert s in syms


def test_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(_lib.SIG), "binding signatures must cover the header exactly"


def test_sm100a_code_in_library(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_tensor_core_and_tma_instructions_present(lib):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                          capture_output=True, text=True, check=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass or "UTCMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA tile loads
    assert "LDTM" in sass  # tcgen05.ld


def test_workspace_size(lib):
    assert lib.ganq_workspace_size(0, 10, 4) == 0
    assert lib.ganq_workspace_size(10, 10, 9) == 0
    a = lib.ganq_workspace_size(64, 128, 3)
    b = lib.ganq_workspace_size(128, 128, 3)
    assert 0 < a < b
    assert lib.ganq_workspace_size(4096, 4096, 4) > 4096 * 4096 * (8 + 4 + 4)


def test_argument_errors_without_gpu(lib):
    P = ctypes.c_void_p(1)
    st = lib.ganq_quantize_layer(P, 0, 4, P, 4, 10, None, P, P, P, 10, None)
    assert st == _lib.ERR_INVALID_ARG and b"must be >= 1" in lib.ganq_last_error()
    st = lib.ganq_quantize_layer(P, 4, 4, P, 0, 10, None, P, P, P, 10, None)
    assert st == _lib.ERR_INVALID_ARG
    st = lib.ganq_quantize_layer(P, 4, 4, P, 6, 10, None, P, P, P, 10, None)
    assert st == _lib.ERR_UNSUPPORTED
    st = lib.ganq_quantize_layer(P, 4, 4, P, 4, 0, None, P, P, P, 10, None)
    assert st == _lib.ERR_INVALID_ARG
    o = _lib.Opts()
    lib.ganq_default_opts(ctypes.byref(o))
    assert o.precond == 0 and o.tau == pytest.approx(1e-7)
    o.precond = 1
    o.lam = 0.0
    st = lib.ganq_quantize_layer(P, 4, 4, P, 2, 1, ctypes.byref(o), P, P, P, 10, None)
    assert st == _lib.ERR_INVALID_ARG and b"lambda" in lib.ganq_last_error()
    o.precond = 0
    st = lib.ganq_quantize_layer(P, 4, 4, P, 2, 1, ctypes.byref(o), P, P, None, 0, None)
    assert st == _lib.ERR_WORKSPACE
    st = lib.ganq_hessian(P, 0, 8, P, 0, None)
    assert st == _lib.ERR_INVALID_ARG
    assert lib.ganq_kmeans_codebook(P, 4, 8, 2, -1, P, None) == _lib.ERR_INVALID_ARG
    assert lib.ganq_kmeans_codebook(P, 4, 8, 5, 3, P, None) == _lib.ERR_UNSUPPORTED
    assert lib.ganq_kmeans_codebook(None, 4, 8, 2, 3, P, None) == _lib.ERR_INVALID_ARG


def test_binding_rejects_cpu_tensors():
    import torch
    import paper_2501_12956_b200 as g
    with pytest.raises(ValueError, match="CUDA"):
        g.hessian(torch.zeros((4, 8), dtype=torch.bfloat16))
    with pytest.raises(ValueError, match="CUDA"):
        g.quantize_layer(torch.zeros((4, 8)), torch.zeros((8, 8), dtype=torch.float64), 2, 1)


def test_lut_binding_rejects_host_tensors():
    import torch
    import paper_2501_12956_b200 as g
    with pytest.raises(ValueError, match="CUDA"):
        g.pack_codes(torch.zeros((2, 8), dtype=torch.uint8), 4)
    with pytest.raises(ValueError, match="CUDA"):
        g.kmeans_codebook(torch.zeros((2, 8)), 2)


def test_packed_row_bytes(lib):
    assert lib.ganq_packed_row_bytes(4096, 4) == 2048
    assert lib.ganq_packed_row_bytes(7, 3) == 3
    assert lib.ganq_packed_row_bytes(0, 4) == 0 and lib.ganq_packed_row_bytes(5, 9) == 0


def test_pipeline_module_imports():
    from paper_2501_12956_b200 import pipeline
    assert hasattr(pipeline, "LayerPipeline") and hasattr(pipeline, "quantize_layers")


def test_checkpoint_plan_and_files(tmp_path):
    import torch
    from paper_2501_12956_b200 import pipeline as pl
    assert pl.checkpoint_plan(3, None) == ([], [0, 1, 2])
    meta = {"m": 2, "n": 4, "n_bits": 2, "iters": 1}
    pl.save_checkpoint(str(tmp_path), 1, torch.zeros((2, 4), dtype=torch.uint8), torch.ones((2, 4)), meta)
    assert pl.checkpoint_plan(3, str(tmp_path)) == ([1], [0, 2])
    Q, T = pl.load_checkpoint(str(tmp_path), 1, meta)
    assert Q.dtype == torch.uint8 and torch.equal(T, torch.ones((2, 4)))
    with pytest.raises(ValueError):
        pl.load_checkpoint(str(tmp_path), 1, {**meta, "iters": 2})
    assert not any(f.name.endswith(".tmp") for f in tmp_path.iterdir())


def test_quantize_stacked_validates_without_gpu():
    import torch
    import paper_2501_12956_b200 as g
    with pytest.raises(ValueError):
        g.quantize_stacked([], torch.zeros((4, 4), dtype=torch.float64), 2)
    with pytest.raises(ValueError, match="CUDA"):
        g.quantize_stacked([torch.zeros((2, 4))], torch.zeros((4, 4), dtype=torch.float64), 2)
