"""B200-native paged-KV hot path behind the microserving sub-request APIs
(arXiv 2412.12488).  See DESIGN.md; the C ABI is include/microkv.h."""
from .kvcache import (ApplyStatus, BatchEntry, ErrorCode, FillState, ForwardPlan, KVAddrInfo,
                      KVCache, PrepRecvResult, SplitserveError, load_library, PRODUCT_LIB,
                      EXPORTED_SYMBOLS, DEFAULT_HASH_SEED)

__all__ = ["ApplyStatus", "BatchEntry", "ErrorCode", "FillState", "ForwardPlan", "KVAddrInfo",
           "KVCache", "PrepRecvResult", "SplitserveError", "load_library", "PRODUCT_LIB",
           "EXPORTED_SYMBOLS", "DEFAULT_HASH_SEED"]
