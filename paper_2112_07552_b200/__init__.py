"""B200-native TCUDB hot path: join + group-by aggregate as a tensor-core GEMM.

    SELECT A.g, B.h, SUM(A.v*B.w) | COUNT(*) FROM A JOIN B ON A.k = B.k GROUP BY A.g, B.h

The computation lives in libtcudb.so (hand-written sm_100a CUDA behind the C
ABI in include/tcudb.h). This package is the thin Python binding (`Engine`)
plus the multi-GPU row-sharding driver (`shard`).
"""
from ._lib import (COUNT, FORCE_DENSE, FORCE_SPARSE, FORCE_WIDE, GATHER_NONE, SUM, Engine, TcudbError,  # noqa: F401
                   load, LIB_PATH, EXPORTS)

__all__ = ["Engine", "TcudbError", "load", "LIB_PATH", "EXPORTS", "FORCE_DENSE", "FORCE_SPARSE", "FORCE_WIDE", "GATHER_NONE"]
