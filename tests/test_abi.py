"""CPU: the C-ABI library loads, exports exactly what include/ggb.h declares,
the Python binding covers it, and without a GPU the product fails loudly
(no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    txt = open(os.path.join(ROOT, "include", "ggb.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ggb_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_surface():
    names = declared()
    for must in ["ggb_sample_vertices", "ggb_build_step_batch", "ggb_train_step", "ggb_dp_sync",
                 "ggb_optimizer_step", "ggb_graph_create", "ggb_state_create", "ggb_gemm_bf16", "ggb_spmm_csr"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2604_02651_b200 import _lib
    L = ctypes.CDLL(_lib.LIBPATH)
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED) == declared()


def test_symbols_in_dynamic_table():
    from paper_2604_02651_b200 import _lib
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIBPATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ggb_\w+)", out))
    assert set(declared()) <= exported


def test_library_is_sm100a():
    from paper_2604_02651_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIBPATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2604_02651_b200 import gridgnn as gg
    with pytest.raises(gg.GgbError) as e:
        gg.Context()
    assert e.value.code == 4  # GGB_ECUDA


def test_errors_map_to_reference_exceptions():
    from paper_2604_02651_b200 import _lib
    assert issubclass(_lib.InvalidArgument, ValueError)
    for code, cls in [(1, _lib.InvalidArgument), (2, _lib.CommContract), (3, _lib.CommTimeout)]:
        assert issubclass(cls, _lib.GgbError)
