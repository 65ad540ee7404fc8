"""Kernel-level GPU tests through the C-ABI test hooks: the tcgen05 GEMM (every
epilogue, ragged M / N tails, the BN choices) against a plain fp32 torch reference of
the same op on the same bf16 operands."""
import ctypes

import pytest

from paper_2511_07399_b200.sdv2 import lib

P = ctypes.c_void_p


def _gemm(A, W, bias, out, M, N, K, epi, mod=None, e0=None, gate_row=0, L=1):
    import torch
    L_ = lib()
    L_.sdv2_debug_gemm.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P,
                                   ctypes.c_int32, ctypes.c_int32, P]
    L_.sdv2_debug_gemm.restype = ctypes.c_int
    st = L_.sdv2_debug_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), M, N, K, epi,
                            mod.data_ptr() if mod is not None else None, e0.data_ptr() if e0 is not None else None,
                            gate_row, L, torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (1560, 4608, 1536), (1560, 1536, 1536), (1560, 8960, 1536),
                                   (1560, 1536, 8960), (32, 384, 128), (200, 144, 192), (6240, 1536, 1536)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_tc_gemm(M, N, K, epi):
    import torch
    if epi >= 2 and N % 32:
        N += 32 - N % 32     # residual epilogues stage 32-column boxes (library shapes: N = d)
    torch.manual_seed(M + N + K + epi)
    A = (torch.randn(M, K, device="cuda") * 0.5).bfloat16()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda")
    ref = A.float() @ W.float().T + bias
    L = max(1, M // 4)
    if epi in (0, 1):
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        _gemm(A, W, bias, out, M, N, K, epi)
        if epi == 1:
            ref = torch.nn.functional.gelu(ref, approximate="tanh")
        err = (out.float() - ref).norm() / ref.norm()
        assert err < 8e-3, err
    else:
        x0 = torch.randn(M, N, device="cuda")
        out = x0.clone()
        mod = torch.randn(6, N, device="cuda")
        nent = (M + L - 1) // L
        e0 = torch.randn(nent, 6, N, device="cuda")
        _gemm(A, W, bias, out, M, N, K, epi, mod, e0, 2, L)
        if epi == 2:
            ent = torch.arange(M, device="cuda") // L
            g = mod[2][None, :] + e0[ent, 2, :]
            ref = x0 + g * ref
        else:
            ref = x0 + ref
        err = (out - ref).norm() / ref.norm()
        assert err < 1e-5, err


@pytest.mark.gpu
@pytest.mark.parametrize("Lq,Lk,H,hd", [(16, 48, 2, 64), (1560, 7800, 2, 128), (1560, 512, 3, 128), (128, 128, 1, 128), (1560, 7800, 12, 128), (300, 1000, 5, 64),
                                        (200, 300, 2, 64), (1024, 5120, 2, 128),
                                        # hybrid schedule: 384 units = one whole-unit round + a split
                                        # of the remaining 236; 148 units (split only)
                                        (4096, 1024, 12, 128), (4736, 256, 4, 128),
                                        # cross-attention shape at n = 1 (156 units of 4 key tiles)
                                        (1560, 512, 12, 128)])
def test_tc_attention(Lq, Lk, H, hd):
    import torch
    L_ = lib()
    L_.sdv2_debug_attention.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        P, P]
    L_.sdv2_debug_attention.restype = ctypes.c_int
    torch.manual_seed(Lq + Lk)
    q = torch.randn(Lq, H * hd, device="cuda").bfloat16()
    k = torch.randn(Lk, H * hd, device="cuda").bfloat16()
    v = torch.randn(Lk, H * hd, device="cuda").bfloat16()
    o = torch.zeros(Lq, H * hd, device="cuda", dtype=torch.bfloat16)
    scratch = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    st = L_.sdv2_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), Lq, Lk, H, hd,
                                 scratch.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert st == 0
    qh = q.float().view(Lq, H, hd).transpose(0, 1)
    kh = k.float().view(Lk, H, hd).transpose(0, 1)
    vh = v.float().view(Lk, H, hd).transpose(0, 1)
    ref = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh).transpose(0, 1).reshape(Lq, H * hd)
    err = (o.float() - ref).norm() / ref.norm()
    assert err < 1.5e-2, err
