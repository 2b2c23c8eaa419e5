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


def _fake_comm(world, local_group):
    """A Communicator shell (no device handle) for exercising the Python argument checks,
    which run before any C call."""
    import torch
    c = tpf.Communicator.__new__(tpf.Communicator)
    c._h = C.c_void_p()
    # host tensors stand in for device tensors: the shell's "device" is the CPU
    c.rank, c.world, c.is_local_group, c.device = 0, world, local_group, torch.device("cpu")
    return c


@pytest.mark.parametrize("local_group", [False, True])
def test_python_wrappers_validate_shapes_dtypes_layout(local_group):
    """Every wrapper checks the tensors before passing raw pointers to the C ABI and raises
    ShapeError naming both shapes (tensor.cpp:68-85): mismatched weight rows, undersized
    outputs, fp32 inputs, transposed (non-contiguous) inputs and host tensors."""
    import torch
    T = 2
    c = _fake_comm(T, local_group)
    L = (T,) if local_group else ()
    bf = torch.bfloat16
    x = torch.zeros(L + (1, 64, 32), dtype=bf)
    w_bad = torch.zeros(L + (48, 64), dtype=bf)
    with pytest.raises(tpf.ShapeError, match=r"ag_gemm w: shape .*\(.*48, 64\).* expected .*32, 64"):
        c.ag_gemm(x, w_bad, torch.zeros(L + (1, 128, 64)))
    w = torch.zeros(L + (32, 64), dtype=bf)
    with pytest.raises(tpf.ShapeError, match="ag_gemm out"):
        c.ag_gemm(x, w, torch.zeros(L + (1, 64, 64)))  # needs (1, 128, 64)
    with pytest.raises(tpf.ShapeError, match="dtype"):
        c.ag_gemm(x.float(), w, torch.zeros(L + (1, 128, 64)))
    with pytest.raises(tpf.ShapeError, match="contiguous"):
        wt = torch.zeros(L + (64, 32), dtype=bf).transpose(-1, -2)
        c.ag_gemm(x, wt, torch.zeros(L + (1, 128, 64)))
    c.device = torch.device("cuda", 0)
    with pytest.raises(tpf.ShapeError, match="is on cpu"):
        c.ag_gemm(x, w, torch.zeros(L + (1, 128, 64)))
    c.device = torch.device("cpu")
    with pytest.raises(tpf.ShapeError, match="gemm_rs out"):
        c.gemm_rs(torch.zeros(L + (1, 64, 32), dtype=bf), w, torch.zeros(L + (1, 64, 64)))  # needs S/T = 32
    with pytest.raises(tpf.ShapeError, match="gemm_rs w"):
        c.gemm_rs(torch.zeros(L + (1, 64, 16), dtype=bf), w, torch.zeros(L + (1, 32, 64)))
    with pytest.raises(tpf.ShapeError, match="dp_grad_rs dW"):
        c.dp_grad_rs(torch.zeros(L + (16, 32), dtype=bf), torch.zeros(L + (16, 8), dtype=bf), torch.zeros(L + (32, 8)))
    with pytest.raises(tpf.ShapeError, match="dp_param_ag_gemm out"):
        c.dp_param_ag_gemm(torch.zeros(L + (16, 32), dtype=bf), torch.zeros(L + (8, 32), dtype=bf),
                           torch.zeros(L + (16, 8)))
    q = torch.zeros(L + (4, 256, 128), dtype=bf)
    with pytest.raises(tpf.ShapeError, match="head rows"):
        c.attention_a2a(q, q, q, torch.zeros(L + (1, 128, 1024), dtype=bf), 1, 2)
    with pytest.raises(tpf.ShapeError, match="attention_a2a out"):
        c.attention_a2a(q, q, q, torch.zeros(L + (1, 128, 512), dtype=bf), 1, 4)
    with pytest.raises(tpf.ShapeError, match="query_split_attention w_o"):
        c.query_split_attention(q, q, q, torch.zeros(L + (256, 64), dtype=bf), torch.zeros(L + (1, 128, 64)), 1, 4)
    with pytest.raises(tpf.ShapeError, match="ulysses_a2a q_out"):
        o = torch.zeros(L + (4, 256, 128), dtype=bf)
        c.ulysses_a2a(q, q, q, o, o, o, 1, 4)
    with pytest.raises(tpf.ShapeError, match="ulysses_attention out"):
        c.ulysses_attention(q, q, q, torch.zeros(L + (1, 256, 256), dtype=bf), 1, 4)
    with pytest.raises(tpf.ShapeError, match="must be on a CUDA device"):
        tpf.gemm(torch.zeros((8, 16), dtype=bf), torch.zeros((16, 8), dtype=bf), torch.zeros((8, 8)))
    with pytest.raises(tpf.ShapeError, match="shape mismatch"):
        tpf.gemm(torch.zeros((8, 16), dtype=bf), torch.zeros((24, 8), dtype=bf), torch.zeros((8, 8)))
    with pytest.raises(tpf.ShapeError, match="swiglu gu: tensor must be on a CUDA device"):
        tpf.swiglu(torch.zeros((8, 16), dtype=bf), torch.zeros((8, 8), dtype=bf))


def test_group_error_carries_the_failing_rank():
    e = tpf.GroupError("rank 3 failed: peer flag wait timed out (rank 0 gave up at step 2, tile 5)")
    assert e.failing_rank() == 3
    assert tpf.GroupError("x", 5).failing_rank() == 5


def test_split_group_without_device_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    hs = (C.c_void_p * 2)()
    assert tpf.lib().tpf_comm_create_split_group(2, 1 << 22, hs) == tpf.E_CUDA
    assert tpf.lib().tpf_comm_create_split_group(9, 1 << 22, hs) == tpf.E_INVALID
