"""CPU: libocgpu.so loads without a GPU and exports every symbol that
include/octgpu.h declares (no compute calls here)."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

from paper_2510_03932_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "octgpu.h"


def declared() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ocg_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = C.CDLL(str(_lib.LIB_PATH))
    names = declared()
    assert len(names) > 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert sorted(_lib.EXPORTS) == declared()


def test_model_api_without_gpu():
    from paper_2510_03932_b200 import MODELS, Model
    m = Model(MODELS["goddard"], 10)
    assert m.nvar == 4 * 10 + 5
    x, lam = m.synth_acceptance(1)
    assert x.shape == (m.nvar,) and lam.shape == (m.m_con,)
    assert "ocg_cjh" in m.generated_source()
    assert _lib.LIB.ocg_version().decode().startswith("octgpu")


def test_no_cpu_fallback():
    """The evaluation path refuses to run without a device instead of falling back."""
    import pytest
    import torch
    from paper_2510_03932_b200 import MODELS, EvalContext, Model
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        EvalContext(Model(MODELS["goddard"], 10))
