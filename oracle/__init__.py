"""CPU oracle for the StreamDiffusionV2 stream-batched causal-DiT hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or call
anything in this package.  The product path (``paper_2511_07399_b200``) never
imports it and fails loudly when its CUDA library is missing.

The oracle is a plain, slow, step-by-step NumPy restatement of SURVEY.md §8(c)
(model card C.1–C.8 and stream algorithm O1–O7), which itself restates the
paper (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):

* motion-aware noise controller  P:205–219 (§3.1 "Motion-aware noise scheduler")
* adaptive sink refresh           P:188–190 (§3.1 "Adaptive sink and RoPE refresh")
* RoPE phase reset
* rolling KV cache with sinks     P:472, P:490 (Fig. kv_cache caption)
* stream batch / pipeline         P:164, P:222–227 (§3.2)
* DiT block scheduler             P:231–233 (§3.3)
* causal DiT (Wan2.1 + CausVid)   P:246 — the paper never defines the block; the
  model card (SURVEY.md §8(c) C.1–C.8) is an external reading, listed in DESIGN.md.

It shares no code with the CUDA path.  Floating point runs in a caller-chosen
dtype (float64 for the parity pins, float32 = the north-star "fp32 oracle");
sinusoid / RoPE tables / Box–Muller / cosines / motion statistics are fp64.

Parity status per function (DESIGN.md §3 names the pin of every function):
  pinned:   philox (Random123 KAT), motion controller (SPEC worked examples and
            closed forms), sink refresh, rope_position, ring/sink metadata
            (Appendix A trace), partition (brute force + SPEC examples), norms /
            activations / attention (torch library routines + closed forms),
            patchify/unpatchify (torch conv3d / einsum), RoPE (relative
            invariance, identity at 0, the per-group frequency law at hand-computed
            angles, interleaved pair rotation), token positions (height/width on a
            non-square latent, tied to patchify), rms_g over the full dim,
            time embedding (closed form with one-hot weights: t = 1000 sigma, SiLU
            placement, cos-first sinusoid, [6, d] view), text embedding / prompt K,V
            (closed form), block wiring (modulation row order, gates, ungated cross
            residual, norm3 affine, cross q RMS: closed forms), head (shift/scale
            rows), sampler (perfect-denoiser closed form), residual wiring
            (identity block), streaming cache == brute-force full attention,
            stream-level RoPE-reset invariance with m = 0 (P2(iii)), pipelined ==
            sequential (order independence), causality.  tests/test_oracle_mutations.py
            shows every closed-form pin fails under its plausible misreadings.
  parity unpinned: the full random-init model output as a whole (no trained
            weights or published tensors exist); it is the composition of the
            pinned functions, checked only oracle <-> GPU.
"""
