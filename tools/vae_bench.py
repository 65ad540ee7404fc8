"""Stream-VAE stand-in timing ("the VAE accounts for ~30% of
the time"): encode and decode one 4-frame chunk at 480p (Wan-VAE channel shapes), CUDA
events around each call on the VAE's stream, after warm-up; algorithmic conv FLOPs from
the layer list (logical channels) -> achieved TFLOP/s vs the measured bf16 peak.

  python tools/vae_bench.py out.json [H W chunks]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthgen as sg  # noqa: E402


def conv_flops(vd, H, W):
    """2 T H W Cout 27 Cin per causal conv, encoder and decoder, one 4-frame chunk."""
    c1, c2, c3 = vd.dims
    cl, cv = vd.latent_channels, vd.video_channels
    enc = [(4, H, W, cv, c1), (4, H, W, c1, c1), (4, H, W, c1, c1), (4, H // 2, W // 2, c1, c2),
           (4, H // 2, W // 2, c2, c2), (4, H // 2, W // 2, c2, c2), (2, H // 4, W // 4, c2, c3),
           (2, H // 4, W // 4, c3, c3), (2, H // 4, W // 4, c3, c3), (1, H // 8, W // 8, c3, c3),
           (1, H // 8, W // 8, c3, c3), (1, H // 8, W // 8, c3, cl)]
    dec = [(1, H // 8, W // 8, cl, c3), (1, H // 8, W // 8, c3, c3), (1, H // 8, W // 8, c3, c3),
           (2, H // 4, W // 4, c3, c3), (2, H // 4, W // 4, c3, c3), (2, H // 4, W // 4, c3, c3),
           (4, H // 2, W // 2, c3, c2), (4, H // 2, W // 2, c2, c2), (4, H // 2, W // 2, c2, c2),
           (4, H, W, c2, c1), (4, H, W, c1, c1), (4, H, W, c1, c1), (4, H, W, c1, cv)]
    f = lambda L: sum(2.0 * T * h * w * co * 27 * ci for T, h, w, ci, co in L)
    return f(enc), f(dec)


def main():
    import torch
    from bench import ClockSampler, measured_peaks
    from paper_2511_07399_b200.sdv2 import StreamVAE
    out = sys.argv[1]
    H, W = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (480, 832)
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 12
    vd = sg.VAE
    vae = StreamVAE(vd, H, W, sg.gen_vae_weights(vd))
    s = vae.stream
    vid = torch.from_numpy(np.ascontiguousarray(sg.gen_video(vd, 4, H, W))).cuda()
    lat = torch.zeros((vd.latent_channels, 1, H // 8, W // 8), device="cuda")
    rec = torch.zeros((3, 4, H, W), device="cuda")
    torch.cuda.synchronize()
    vae.reset()
    for _ in range(3):
        vae.encode_chunk(vid.data_ptr(), lat.data_ptr())
        vae.decode_chunk(lat.data_ptr(), rec.data_ptr())
    torch.cuda.synchronize()
    clk = ClockSampler(0)
    clk.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n + 1)]
    ev[0].record(s)
    l0 = vae.launches()
    for i in range(n):
        vae.encode_chunk(vid.data_ptr(), lat.data_ptr())
        ev[2 * i + 1].record(s)
        vae.decode_chunk(lat.data_ptr(), rec.data_ptr())
        ev[2 * i + 2].record(s)
    torch.cuda.synchronize()
    clocks = clk.stop()
    enc_ms = float(np.median([ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(n)]))
    dec_ms = float(np.median([ev[2 * i + 1].elapsed_time(ev[2 * i + 2]) for i in range(n)]))
    fe, fd = conv_flops(vd, H, W)
    peaks, src = measured_peaks()
    peak = peaks["bf16_tflops_sustained"]
    res = {"workload": f"stream_vae {H}x{W}, 4 frames per chunk, dims {vd.dims}",
           "encode_ms_per_chunk": enc_ms, "decode_ms_per_chunk": dec_ms,
           "encode_tflop": fe / 1e12, "decode_tflop": fd / 1e12,
           "encode_tflops": fe / (enc_ms * 1e-3) / 1e12, "decode_tflops": fd / (dec_ms * 1e-3) / 1e12,
           "roofline": {"bound": "tensor", "peak": peak, "peak_source": f"{src} bf16_tflops_sustained",
                        "frac_encode": fe / (enc_ms * 1e-3) / 1e12 / peak,
                        "frac_decode": fd / (dec_ms * 1e-3) / 1e12 / peak},
           "launches_per_chunk_pair": (vae.launches() - l0) / n, "clocks": clocks}
    vae.close()
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
