"""The C-ABI library loads and exports every symbol include/sc.h declares (CPU, no GPU).

Only host-side validation paths are exercised here (they return before any CUDA
call); every compute call is a -m gpu test."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "sc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:sc_status|const char\*|uint64_t|size_t)\s+(sc_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_survey_boundary():
    names = declared_functions()
    for n in ("sc_context_load", "sc_context_free", "sc_decide", "sc_decision_hist", "sc_weights_from_hist",
              "sc_loss_fwd_bwd", "sc_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2310_07240_b200 as sc
    lib = ctypes.CDLL(sc.library_path())
    for n in declared_functions():
        assert hasattr(lib, n), n


def test_host_validation_without_gpu():
    import paper_2310_07240_b200 as sc
    with pytest.raises(sc.ScError) as e:
        sc.Context(10, [[1, 10]])
    assert e.value.status == sc.SC_ERR_INVALID_ARG and "not in [0, C)" in str(e.value)
    with pytest.raises(sc.ScError) as e:
        sc.Context(10, [[1]] * 9)
    assert e.value.status == sc.SC_ERR_INVALID_ARG
    with pytest.raises(sc.ScError) as e:
        sc.Context(10, [[1]], k=0.0)
    assert e.value.status == sc.SC_ERR_INVALID_ARG
    with pytest.raises(sc.ScError) as e:
        sc.Context(10, [[1]], order=7)
    assert e.value.status == sc.SC_ERR_INVALID_ARG
    assert "order" in sc.sc_last_error()


def test_no_cpu_fallback():
    """Product calls refuse host tensors instead of computing on the CPU."""
    import torch
    import paper_2310_07240_b200 as sc
    with pytest.raises(ValueError):
        sc.Batch(logits=torch.zeros(4, 12))._c()


def test_product_package_does_not_reference_the_oracle():
    pkg = os.path.join(ROOT, "paper_2310_07240_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for needle in ("import oracle", "from oracle", "liboracle", "sc_oracle", "orc_"):
                    assert needle not in txt, (f, needle)
