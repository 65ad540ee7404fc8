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
                                        # cross-attention shape at n = 1 (156 units of 4 key tiles: the 8
                                        # overflow units split into 4 one-tile pieces, merged in-kernel)
                                        (1560, 512, 12, 128),
                                        # overflow splits with 3 / 2 / 4 pieces, ragged key tails
                                        (1920, 384, 10, 128), (1560, 200, 12, 128), (2048, 500, 10, 128)])
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


def _cands(M, N, K, epi):
    L_ = lib()
    L_.sdv2_debug_gemm_candidates.argtypes = [ctypes.c_int32] * 4 + [P, ctypes.c_int32, P]
    L_.sdv2_debug_gemm_candidates.restype = ctypes.c_int
    buf = (ctypes.c_int32 * 256)()
    cnt = ctypes.c_int32()
    assert L_.sdv2_debug_gemm_candidates(M, N, K, epi, buf, 64, ctypes.byref(cnt)) == 0
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(cnt.value)]


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K,epi", [(1560, 4608, 1536, 0), (1560, 1536, 1536, 2), (1560, 8960, 1536, 1),
                                       (1560, 1536, 8960, 2), (1560, 1536, 1536, 3), (6240, 1536, 1536, 2),
                                       (4096, 8960, 1536, 1), (1560, 64, 1536, 4), (6240, 5120, 5120, 0)])
def test_gemm_configs_bitwise_identical(M, N, K, epi):
    """Every configuration the create-time tuner may pick (cluster size, tile width, early
    residual fetch) reduces each output element over K in the same order, so the tuner's
    timing-dependent choice never changes results: all candidates agree bit for bit."""
    import torch
    L_ = lib()
    L_.sdv2_debug_gemm_cfg.argtypes = [P, P, P, P] + [ctypes.c_int32] * 4 + [P, P, ctypes.c_int32, ctypes.c_int32,
                                                                            P, P]
    L_.sdv2_debug_gemm_cfg.restype = ctypes.c_int
    cands = _cands(M, N, K, epi)
    assert len(cands) >= 2 and all(c[2] == 0 for c in cands)       # no stream-K on the product path
    torch.manual_seed(M + N + K)
    A = (torch.randn(M, K, device="cuda") * 0.5).bfloat16()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda")
    L = 1560
    mod = torch.randn(6, N, device="cuda")
    e0 = torch.randn((M + L - 1) // L, 6, N, device="cuda")
    x0 = torch.randn(M, N, device="cuda")
    ref = None
    for c in cands:
        if epi in (2, 3):
            out = x0.clone()
        elif epi == 4:
            out = torch.zeros(M, N, device="cuda")
        else:
            out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        cfg = (ctypes.c_int32 * 4)(*c)
        st = L_.sdv2_debug_gemm_cfg(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), M, N, K, epi,
                                    mod.data_ptr(), e0.data_ptr(), 2, L, cfg, torch.cuda.current_stream().cuda_stream)
        assert st == 0, c
        torch.cuda.synchronize()
        if ref is None:
            ref = out
            exp = A.float() @ W.float().T + bias
            if epi == 1:
                exp = torch.nn.functional.gelu(exp, approximate="tanh")
            if epi == 2:
                exp = x0 + (mod[2][None, :] + e0[torch.arange(M, device="cuda") // L, 2, :]) * exp
            if epi == 3:
                exp = x0 + exp
            assert ((out.float() - exp).norm() / exp.norm()).item() < 8e-3
        else:
            assert torch.equal(out, ref), (c, cands[0])


@pytest.mark.gpu
def test_attention_rescale_rows_disagree():
    """Regression: rows of one softmax warp whose running max grows by more than 2^8 at
    different key tiles (odd rows find a dominant key in tile 3, even rows never do).  The
    lazy O rescale touches TMEM with warp-synchronous instructions, so its decision must be
    warp-uniform; a per-row branch hung here.  Must finish and match SDPA."""
    import torch
    L_ = lib()
    L_.sdv2_debug_attention.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        P, P]
    L_.sdv2_debug_attention.restype = ctypes.c_int
    torch.manual_seed(7)
    Lq, Lk, H, hd = 256, 1024, 2, 128
    k = torch.randn(Lk, H * hd, device="cuda")
    v = torch.randn(Lk, H * hd, device="cuda")
    q = 0.1 * torch.randn(Lq, H * hd, device="cuda")
    q[1::2] = 4.0 * k[400]                       # odd rows: a dominant key in key tile 3
    q, k, v = q.bfloat16(), k.bfloat16(), v.bfloat16()
    o = torch.zeros(Lq, H * hd, device="cuda", dtype=torch.bfloat16)
    scratch = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    st = L_.sdv2_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), Lq, Lk, H, hd,
                                 scratch.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()
    qh = q.float().view(Lq, H, hd).transpose(0, 1)
    kh = k.float().view(Lk, H, hd).transpose(0, 1)
    vh = v.float().view(Lk, H, hd).transpose(0, 1)
    ref = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh).transpose(0, 1).reshape(Lq, H * hd)
    err = (o.float() - ref).norm() / ref.norm()
    assert err < 1.5e-2, err
