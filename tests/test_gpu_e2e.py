"""bench.py's e2e timed region (e2e_pipeline) computes the right thing: with two distinct pinned
inputs in its double buffer, every step's result copied back to the host equals the
device-resident MLP block of that step's input. This checks the H2D / compute / D2H stream and
event ordering that the e2e number depends on. It uses the bench's own calls (AG-GEMM with fused
SwiGLU, then GEMM-RS) at T = 1, at a small shape."""
import os
import sys

import pytest
import torch

import paper_2604_24013_b200 as tpf

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def test_e2e_pipeline_outputs_match_device_resident_block():
    S, D, F = 1024, 512, 1024
    g = torch.Generator(device=DEV).manual_seed(4)
    w_gu = tpf.interleave_gate_up((torch.randn((D, F), device=DEV, generator=g) / 32).to(torch.bfloat16),
                                  (torch.randn((D, F), device=DEV, generator=g) / 32).to(torch.bfloat16)).contiguous()
    w_dn = (torch.randn((F, D), device=DEV, generator=g) / 32).to(torch.bfloat16)
    act = torch.empty((1, S, F), device=DEV, dtype=torch.bfloat16)
    one = tpf.Communicator.create(0, 1, 0)
    stream = torch.cuda.current_stream(DEV)

    def block(xin, yout):
        one.ag_gemm(xin, w_gu, act, act=tpf.ACT_SWIGLU, stream=stream)
        one.gemm_rs(act, w_dn, yout, stream=stream)

    xs = [torch.randn((1, S, D), device=DEV, generator=g).to(torch.bfloat16) for _ in range(2)]
    want = []
    for xv in xs:
        yv = torch.empty((1, S, D), device=DEV, dtype=torch.bfloat16)
        block(xv, yv)
        want.append(yv.cpu())
    x_host = [xv.cpu().pin_memory() for xv in xs]
    y_host = [torch.full((1, S, D), float("nan"), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    x_dev = [torch.empty_like(xs[0]) for _ in range(2)]
    y_dev = [torch.empty_like(xs[0]) for _ in range(2)]
    for n in (1, 2, 7):
        ms = bench.e2e_pipeline(torch, n, x_host, y_host, x_dev, y_dev, block, stream, DEV)
        assert ms > 0
        for b in range(min(n, 2)):
            assert torch.equal(y_host[b], want[b]), (n, b)
    one.sync()
    one.close()
