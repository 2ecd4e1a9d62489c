"""CPU-side checks of the native boundary: the C-ABI library loads, exports every
symbol include/gavis_b200.h declares, and fails loudly (status 5, DEVICE) when no
CUDA device exists -- there is no CPU fallback. No compute calls run here."""
import ctypes as C
import os
import re

import pytest

from paper_2605_30342_b200 import _native as N
from paper_2605_30342_b200.model import DeviceError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gavis_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gavis_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_30342_b200 import build
    build.build()
    return N.load()


def test_header_declares_binding_exports():
    assert declared_symbols() == sorted(N.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.gavis_abi_version() == 1


def test_struct_layouts_match_header():
    # sizes of the POD structs as laid out by a C compiler for the header
    assert C.sizeof(N.Camera) == 128
    assert C.sizeof(N.RasterConfigC) == 32
    assert C.sizeof(N.UncertaintyConfigC) == 112
    assert C.sizeof(N.SceneDesc) == 64
    assert C.sizeof(N.RenderOutputs) == 80


def test_no_cpu_fallback_without_device(lib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    h = C.c_void_p()
    status = lib.gavis_ctx_create(0, None, C.byref(h))
    assert status == 5
    with pytest.raises(DeviceError):
        N.check(status)


def test_comm_unique_id_without_device(lib):
    """The library's NCCL is loaded at run time (dlopen libnccl.so.2); a unique id
    needs no device (rank 0 makes it, the host ships the 128 bytes)."""
    from paper_2605_30342_b200 import api
    a, b = api.Comm.unique_id(), api.Comm.unique_id()
    assert len(a) == N.COMM_ID_BYTES == 128 and a != b


def test_comm_create_fails_loudly_without_device(lib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    h = C.c_void_p()
    assert lib.gavis_ctx_create(0, None, C.byref(h)) == 5  # no context, hence no communicator
