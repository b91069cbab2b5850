"""B200-native PagedEviction engine (arXiv 2509.04377).

The hot path — prefill prune+pack (K1), decode append (K0), decode block
eviction (K2/K2c) and paged decode attention (K3) — runs in hand-written
sm_100a CUDA behind the C-ABI in include/pe.h (libpe_b200.so). This
package is the Python mirror of the reference's cache-manager interface over
that C-ABI; it has no CPU fallback.
"""
from .engine import (  # noqa: F401
    BudgetInvalid,
    CudaError,
    EmptyCache,
    EngineGeometry,
    Error,
    Granularity,
    IndexOutOfRange,
    InvalidArgument,
    InvalidState,
    LengthMismatch,
    NoDevice,
    PagedEvictionEngine,
    PolicyConfig,
    PolicyKind,
    PoolExhausted,
    ScoreMode,
    TokenRule,
    parse_policy_kind,
    to_string,
    DTYPE_BF16,
    DTYPE_F32,
)

__all__ = [n for n in dir() if not n.startswith("_")]
