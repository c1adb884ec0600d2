"""The C-ABI library loads without a GPU and exports every symbol declared in include/hetgpu.h."""
import ctypes
import os
import re

from paper_1402_6601_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "hetgpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    decl = declared_functions()
    assert set(_native.EXPORTS) == set(decl)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_cpu_only_host_calls():
    L = _native.lib()
    assert L.hg_abi_version() == 3
    assert L.hg_device_count() >= 0
    assert isinstance(_native.last_error(), str)


def test_online_executor_data_path_is_the_c_abi():
    """online.py moves tiles and times kernels through libhetgpu (hg_copy_async, hg_event_*),
    not through torch."""
    src = open(os.path.join(ROOT, "paper_1402_6601_b200", "online.py")).read()
    assert "torch" not in src
    for sym in ("hg_copy_async", "hg_event_record", "hg_stream_wait_event", "hg_dev_alloc"):
        assert sym in src or sym.replace("hg_", "") in src
