"""The C-ABI boundary (CPU-only checks: no kernel launches)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tsom_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsom_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2604_26555_b200 import _lib
    L = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), f"{n} declared in tsom_b200.h but not exported"
    assert sorted(_lib.EXPORTS) == names


def test_library_is_sm100a_only():
    from paper_2604_26555_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", "")), out


def test_version_string():
    import paper_2604_26555_b200 as pkg
    assert "sm_100a" in pkg.version()


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and
                    __import__("torch").cuda.is_available(), reason="GPU present")
def test_create_fails_loudly_without_a_b200():
    """No CPU fallback: without an sm_100 device the engine refuses to exist."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_26555_b200 import Engine, TsomError
    with pytest.raises(TsomError):
        Engine(16, 4)


def test_dropin_and_oracle_config_layouts_agree():
    import oracle
    from paper_2604_26555_b200 import dropin
    assert C.sizeof(dropin._Cfg) == C.sizeof(oracle._Cfg)
    if dropin.available():
        assert dropin.load().tsom_dropin_config_sizeof() == C.sizeof(dropin._Cfg)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2604_26555_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".hpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt, f
                assert "libtoposom_ref" not in txt, f
