"""Stream-VAE stand-in on the GPU vs the oracle: 3 chunks
of 4 frames streamed through the library's encoder and decoder (tensor-core implicit-GEMM
causal convs with per-conv feature caches) == the oracle's full-sequence causal VAE
(== its chunked run, pinned in tests/test_vae_oracle.py).  bf16 activations through ~15
conv layers: rel-L2 <= 2e-2.  Also the conv kernel alone on Wan shapes vs torch."""
import ctypes
import dataclasses

import numpy as np
import pytest

import synthgen as sg
from oracle import vae as V

from gpu_harness import rel_l2


@pytest.mark.gpu
@pytest.mark.parametrize("dims,H,W", [((96, 192, 384), 16, 24), ((64, 128, 128), 32, 136)])
def test_stream_vae_parity(dims, H, W):
    import torch
    from paper_2511_07399_b200.sdv2 import StreamVAE
    vd = dataclasses.replace(sg.VAE, dims=dims)
    Wt = sg.gen_vae_weights(vd)
    n = 3
    video = sg.gen_video(vd, 4 * n, H, W)
    lat_ref = V.encode_full(video, Wt, vd)
    vid_ref = V.decode_full(lat_ref, Wt, vd)
    vae = StreamVAE(vd, H, W, Wt)
    vae.reset()
    lat = torch.zeros((vd.latent_channels, 1, H // 8, W // 8), dtype=torch.float32, device="cuda")
    rec = torch.zeros((3, 4, H, W), dtype=torch.float32, device="cuda")
    lats, recs = [], []
    for i in range(n):
        v = torch.from_numpy(np.ascontiguousarray(video[:, 4 * i:4 * i + 4])).cuda()
        vae.encode_chunk(v.data_ptr(), lat.data_ptr())
        torch.cuda.synchronize()
        lats.append(lat.cpu().numpy().copy())
    # decode the ORACLE latents (isolates the decoder's error)
    for i in range(n):
        li = torch.from_numpy(np.ascontiguousarray(lat_ref[:, i:i + 1]).astype(np.float32)).cuda()
        vae.decode_chunk(li.data_ptr(), rec.data_ptr())
        torch.cuda.synchronize()
        recs.append(rec.cpu().numpy().copy())
    vae.close()
    for i in range(n):
        e = rel_l2(lats[i], lat_ref[:, i:i + 1])
        d = rel_l2(recs[i], vid_ref[:, 4 * i:4 * i + 4])
        print(f"chunk {i}: encoder rel-L2 {e:.2e}, decoder rel-L2 {d:.2e}")
        assert e <= 2e-2 and d <= 2e-2, (i, e, d)


@pytest.mark.gpu
def test_vae_reset_restarts_stream():
    """After reset the caches are zero again: re-encoding chunk 0 reproduces the first output
    bit for bit (cache frames carried across chunks otherwise change it)."""
    import torch
    from paper_2511_07399_b200.sdv2 import StreamVAE
    vd = dataclasses.replace(sg.VAE, dims=(64, 64, 64))
    Wt = sg.gen_vae_weights(vd)
    video = sg.gen_video(vd, 8, 16, 16)
    vae = StreamVAE(vd, 16, 16, Wt)
    lat = torch.zeros((vd.latent_channels, 1, 2, 2), device="cuda")
    v0 = torch.from_numpy(np.ascontiguousarray(video[:, :4])).cuda()
    v1 = torch.from_numpy(np.ascontiguousarray(video[:, 4:])).cuda()
    vae.reset()
    vae.encode_chunk(v0.data_ptr(), lat.data_ptr())
    torch.cuda.synchronize()
    first = lat.cpu().numpy().copy()
    vae.encode_chunk(v0.data_ptr(), lat.data_ptr())      # same frames, but now with a cache
    torch.cuda.synchronize()
    assert not np.array_equal(lat.cpu().numpy(), first)
    vae.encode_chunk(v1.data_ptr(), lat.data_ptr())
    vae.reset()
    vae.encode_chunk(v0.data_ptr(), lat.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(lat.cpu().numpy(), first)
    vae.close()
