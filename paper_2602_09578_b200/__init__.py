"""B200-native micro-batch policy-update hot path of FlexMARL (arXiv 2602.09578).

Layers:
  * ``include/flexmarl/cabi.h`` + ``csrc/`` — the C ABI and the sm_100a
    kernels (tcgen05 GEMMs, TMA-staged fused loss, fused Adam, gather, GRPO);
  * :mod:`.engine` — host mirror of the reference's ExperienceStore /
    TrainingEngine / group_advantages interfaces over that ABI;
  * :mod:`.workload` — synthetic experience for the benchmark configs.
"""
from ._lib import FlexMarlError, LIB_PATH  # noqa: F401

__all__ = ["FlexMarlError", "LIB_PATH"]
