"""CPU checks of the C-ABI library: it loads without a GPU and exports every symbol that
include/lmc.h declares (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "lmc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lmc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2202_12567_b200.build as b
    path = b.build()
    lib = ctypes.CDLL(path)
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_2202_12567_b200 import lmc
    assert sorted(lmc.EXPORTS) == declared()


def test_status_strings_without_gpu():
    from paper_2202_12567_b200 import lmc
    assert lmc.lib.lmc_status_str(0) == b"LMC_OK"
    assert lmc.lib.lmc_status_str(5) == b"LMC_EOVERFLOW"
    # a NULL config is rejected before any CUDA call
    assert lmc.lib.lmc_create(None, None, None, None, None, None) == lmc.LMC_EINVAL


def test_struct_layouts_match_the_library():
    from paper_2202_12567_b200 import lmc
    for k, cls in enumerate((lmc.Gbuffer, lmc.Vpls, lmc.LightTree, lmc.Scene, lmc.Config, lmc.Stats)):
        assert ctypes.sizeof(cls) == lmc.lib.lmc_sizeof_struct(k), cls.__name__


def test_oracle_struct_layouts_match():
    import oracle
    L = oracle.lib()
    L.orc_sizeof_inputs.restype = ctypes.c_int64
    L.orc_sizeof_result.restype = ctypes.c_int64
    assert ctypes.sizeof(oracle._Inputs) == L.orc_sizeof_inputs()
    assert ctypes.sizeof(oracle._Result) == L.orc_sizeof_result()


def test_library_loaded_before_torch_keeps_torch_importable():
    """liblmc.so links the NCCL that PyTorch ships: loading it first (as a C caller or the driver's
    build() would) must not put an older libnccl.so.2 in the process ahead of libtorch_cuda"""
    import subprocess
    import sys
    import paper_2202_12567_b200.build as b
    path = b.build()
    code = f"import ctypes; ctypes.CDLL({path!r}); import torch; print('ok')"
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
