"""B200-native SiDP decode hot path (WaS / CaS) — Python binding of libsidp.so.

The product is the C-ABI library built from ``csrc/`` (declared in ``include/sidp.h``);
this package only marshals arguments.  It never imports ``oracle/``.
"""
from . import _abi  # noqa: F401
from ._abi import (WAS, CAS, REPLICATED, ORDER_EXEC, ORDER_PAPER, POOL_LAYER, POOL_FFN,  # noqa: F401
                   FETCH_SM, FETCH_CE, SidpError)
from .api import Context, KVCache, PagedKVCache, prefill, test_gemm, test_gemm_qkv, test_gemm_resid_norm, test_mlp_fused, test_gen  # noqa: F401
