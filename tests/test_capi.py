"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/tpf.h declares, validates arguments like the reference, and the
data path fails loudly (no CPU fallback) when there is no device."""
import ctypes as C
import os
import re

import pytest

import paper_2604_24013_b200 as tpf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "tpf.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(tpf_\w+)\s*\(", src, re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "tpf_ag_gemm" in syms and "tpf_gemm_rs" in syms and "tpf_schedule_build" in syms
    assert set(syms) == set(tpf.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(tpf.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_library_is_sm100a_only():
    # the fatbin carries sm_100a SASS (cuobjdump is part of the CUDA toolkit here)
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", tpf.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", tpf.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_version_and_error_string():
    assert tpf.lib().tpf_version() == 1
    with pytest.raises(ValueError):
        tpf.build_schedule(tpf.PAIRWISE, 5)
    assert b"even rank count" in tpf.lib().tpf_last_error()


def test_sym_bytes_sizing():
    # cfg2 T=8 GEMM-RS, bf16 wire: 7 slots x (8 m-blocks x 16 n-tiles x 64 KiB) per parity
    need = tpf.sym_bytes_rs(8, 1, 8192, 1792, 4096, 1, tpf.BF16)
    assert need == 2 * (1 << 20) + 2 * 7 * (8 * 16 * 128 * 256 * 2)
    assert tpf.sym_bytes_ag(1, 1, 8192, 4096, 3584) == 0


def test_no_device_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    h = C.c_void_p()
    rc = tpf.lib().tpf_comm_create_local_group(2, 1 << 22, C.byref(h))
    assert rc == tpf.E_CUDA
    assert tpf.lib().tpf_gemm(None, None, None, 128, 64, 64, 0, None) in (tpf.E_CUDA, tpf.E_SHAPE)
