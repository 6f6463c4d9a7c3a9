"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/pentab.h declares, and refuses to compute without a
device (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import paper_2101_06550_b200 as pb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pentab.h")).read()
    return set(re.findall(r"^PB_API\s+[a-z0-9_]+\s+\**([a-z0-9_]+)\(", src, flags=re.M))


def test_header_and_binding_agree():
    assert declared_symbols() == set(pb.EXPORTS)


def test_library_exports_every_symbol():
    L = pb.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    assert not pb.device_ok()
    n = 16
    z = np.zeros(n)
    with pytest.raises(pb.PentabError) as ei:
        pb.pent_factor(z, z, np.ones(n), z, z, batch=2, n=n)
    assert ei.value.code == pb.PB_ECUDA


def test_argument_validation():
    n = 4  # too small for a pentadiagonal system
    z = np.zeros(n)
    with pytest.raises(pb.PentabError) as ei:
        pb.pent_factor(z, z, np.ones(n), z, z, batch=2, n=n)
    assert ei.value.code == pb.PB_EINVAL
