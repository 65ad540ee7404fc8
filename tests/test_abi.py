"""The C-ABI library builds, loads without a GPU and exports every symbol include/sdv2.h
declares (no compute calls here)."""
import ctypes
import os
import re

from paper_2511_07399_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sdv2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdv2_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    build.build()
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2511_07399_b200", "libsdv2.so"))
    syms = declared_symbols()
    assert "sdv2_create" in syms and "sdv2_denoise_chunk" in syms and len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    ctl = ctypes.CDLL(os.path.join(ROOT, "paper_2511_07399_b200", "libsdv2_ctl.so"))
    assert hasattr(ctl, "sdv2_partition")


def test_workspace_sizing_and_validation():
    import synthgen as sg
    from paper_2511_07399_b200.sdv2 import lib, model_desc_c, geometry_c, PipelineC, SDV2_BF16, SDV2_FP32
    L = lib()
    cfg = sg.CONFIGS["tiny"]
    md, g = model_desc_c(cfg.model), geometry_c(cfg.geom)
    n32 = L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(g), None, SDV2_FP32)
    n16 = L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(g), None, SDV2_BF16)
    assert n32 > n16 > 0
    # 1.3B 480p n=1 and 14B n=4 fit one B200 (180 GB)
    for name in ("wan13_480p_1step", "wan14_480p_4step"):
        c = sg.CONFIGS[name]
        nb = L.sdv2_workspace_bytes(ctypes.byref(model_desc_c(c.model)), ctypes.byref(geometry_c(c.geom)), None,
                                    SDV2_BF16)
        assert 0 < nb < 150e9
    # a pipeline stage needs fewer bytes than the whole model
    pp = PipelineC(2, 0, 0, 1)
    assert 0 < L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(g), ctypes.byref(pp), SDV2_BF16) < n16 + (1 << 22)
    # invalid shapes are rejected (odd head dim, K > blocks, bad window)
    bad = model_desc_c(cfg.model)
    bad.num_heads = 3
    assert L.sdv2_workspace_bytes(ctypes.byref(bad), ctypes.byref(g), None, SDV2_BF16) == 0
    g0 = geometry_c(cfg.geom)
    g0.window_chunks = 0
    assert L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(g0), None, SDV2_BF16) == 0
    pp = PipelineC(3, 0, 0, 1)
    assert L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(g), ctypes.byref(pp), SDV2_BF16) == 0


def test_clean_rerun_mode_validation():
    """kv_mode 1 (clean-context re-run) is accepted for n = 1 on one stage, rejected
    otherwise; any other kv_mode is rejected."""
    import dataclasses
    import synthgen as sg
    from paper_2511_07399_b200.sdv2 import lib, model_desc_c, geometry_c, PipelineC, SDV2_BF16
    L = lib()
    cfg = sg.CONFIGS["tiny"]
    md = model_desc_c(cfg.model)
    ok = geometry_c(dataclasses.replace(cfg.geom, steps=1, kv_mode=1))
    assert L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(ok), None, SDV2_BF16) > 0
    two = geometry_c(dataclasses.replace(cfg.geom, steps=2, kv_mode=1))
    assert L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(two), None, SDV2_BF16) == 0
    pp = PipelineC(2, 0, 0, 1)
    assert L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(ok), ctypes.byref(pp), SDV2_BF16) == 0
    bad = geometry_c(dataclasses.replace(cfg.geom, kv_mode=2))
    assert L.sdv2_workspace_bytes(ctypes.byref(md), ctypes.byref(bad), None, SDV2_BF16) == 0
