"""B200-native data-parallel hot path of Grendel's distributed 3DGS training step
(arXiv 2406.18533): libgs (CUDA sm_100a + NCCL) behind the C ABI in include/gs.h, a thin
ctypes binding (_lib) and the step driver (engine)."""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgs.so")


def build(force: bool = False) -> str:
    from .build import build as _b
    return _b(force=force)
