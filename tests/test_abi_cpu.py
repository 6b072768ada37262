"""CPU-side checks of the C ABI: the library loads without a GPU, exports every symbol
include/tcbf.h declares, and host-only validation / layout arithmetic behave as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tcbf():
    from paper_2505_03269_b200 import build
    build.build_tcbf()
    import paper_2505_03269_b200 as m
    return m


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "tcbf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tcbf_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(tcbf):
    L = tcbf.lib()
    names = _declared_symbols()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), f"{n} declared in tcbf.h but not exported"


def test_layout_sizes(tcbf):
    # F16: Kp = round_up(K, 64); bytes = B*2*rows*Kp*2; out = B*2*M*N*4
    w, x, o, k = tcbf.layout_sizes(1024, 1024, 256, 256, "f16")
    assert k == 256 and w == 256 * 2 * 1024 * 256 * 2 and x == w and o == 256 * 2 * 1024 * 1024 * 4
    w, x, o, k = tcbf.layout_sizes(3, 5, 65, 2, "f16")   # data is [B][2][K][round_up(N, 8)]
    assert k == 128 and w == 2 * 2 * 3 * 128 * 2 and x == 2 * 2 * 65 * 8 * 2 and o == 2 * 2 * 3 * 5 * 4
    # B1: Kw = round_up(ceil(K/32), 8) words
    w, x, o, k = tcbf.layout_sizes(1024, 4096, 512, 256, "b1")
    assert k == 16 and w == 256 * 2 * 1024 * 16 * 4 and x == 256 * 2 * 4096 * 16 * 4
    _, _, _, k = tcbf.layout_sizes(1, 1, 1, 1, "b1")
    assert k == 8
    _, _, _, k = tcbf.layout_sizes(1, 1, 257, 1, "b1")
    assert k == 16


@pytest.mark.parametrize("args", [(0, 1, 1, 1), (1, 0, 1, 1), (1, 1, 0, 1), (1, 1, 1, 0), (-5, 1, 1, 1),
                                  (1 << 40, 1 << 40, 1 << 20, 1 << 20)])
def test_invalid_sizes(tcbf, args):
    with pytest.raises(tcbf.TcbfError) as e:
        tcbf.layout_sizes(*args, "f16")
    assert e.value.status == 1


def test_b1_k_limit(tcbf):
    with pytest.raises(tcbf.TcbfError):
        tcbf.layout_sizes(1, 1, 1 << 30, 1, "b1")
    tcbf.layout_sizes(1, 1, (1 << 30) - 1, 1, "b1")


def test_plan_create_without_device(tcbf):
    L = tcbf.lib()
    h = ctypes.c_void_p()
    assert L.tcbf_plan_create(ctypes.byref(h), 0, 1, 1, 1, 0) == 1          # validation first
    assert h.value is None
    import torch
    if not torch.cuda.is_available():
        assert L.tcbf_plan_create(ctypes.byref(h), 8, 64, 32, 2, 0) == 2     # UNSUPPORTED_DEVICE
        assert h.value is None
        assert b"device" in L.tcbf_last_error()
    assert L.tcbf_plan_create(None, 8, 64, 32, 2, 0) == 1
    assert L.tcbf_plan_destroy(None) == 0


def test_status_strings(tcbf):
    names = [tcbf.status_string(i) for i in range(6)]
    assert names == ["TCBF_OK", "TCBF_ERR_INVALID_ARG", "TCBF_ERR_UNSUPPORTED_DEVICE",
                     "TCBF_ERR_DEVICE_MISMATCH", "TCBF_ERR_ALLOC", "TCBF_ERR_CUDA"]


def test_null_plan_arguments(tcbf):
    L = tcbf.lib()
    sz = ctypes.c_size_t()
    assert L.tcbf_packed_bytes(None, 0, ctypes.byref(sz)) == 1
    assert L.tcbf_output_bytes(None, ctypes.byref(sz)) == 1
    assert L.tcbf_pack(None, 0, None, 0, None, None) == 1
    assert L.tcbf_beamform(None, None, None, None, None) == 1
    assert L.tcbf_beamform_host(None, None, None, 0, None) == 1


def test_product_library_has_no_dev_switches(tcbf):
    """The ablation / trace switches of the DESIGN.md §4 studies exist only in TCBF_DEV builds:
    the product library cannot be put into a wrong-result mode by the environment."""
    data = open(tcbf.library_path, "rb").read()
    for s in (b"TCBF_DEBUG", b"TCBF_TRACE"):
        assert s not in data, s


def test_binding_validates_tensors_before_the_abi():
    """Raw pointers cross the ABI only for contiguous CUDA tensors of the right dtype and size."""
    import torch
    from paper_2505_03269_b200 import _need
    with pytest.raises(ValueError, match="CUDA"):
        _need(torch.zeros(4), "x", ("f32",), 16)
    with pytest.raises(TypeError):
        _need(np.zeros(4, np.float32), "x", ("f32",), 16)
