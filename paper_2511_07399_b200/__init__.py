"""B200-native (sm_100a) StreamDiffusionV2 stream-batched causal-DiT hot path.

The product is the C-ABI library ``libsdv2.so`` (include/sdv2.h); ``sdv2`` is its thin
ctypes binding and ``pipeline`` the torch.distributed stage transport.  Nothing here
imports the CPU oracle (``oracle/`` is test infrastructure only)."""
from .sdv2 import SDV2_BF16, SDV2_FP32, SDV2Error, Stage, lib, partition  # noqa: F401
