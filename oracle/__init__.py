"""TEST INFRASTRUCTURE ONLY: CPU restatements of the reference (the checker).

oracle/hashmodel.c (+ hashmodel.py)   toy-model hash contract, hash_model.cc
oracle/kvcache_oracle.py              KVCache/RadixTree/KVAddrInfo bookkeeping, kv_cache.cc
oracle/ref_capi.cc + Makefile         the unmodified reference compiled behind include/microkv.h
                                       -> oracle/_ref/libmicrokv_ref.so (pins the restatement)

Importable only from tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs.  The product (paper_2412_12488_b200) never imports it.
"""
from pathlib import Path

REF_LIB = Path(__file__).resolve().parent / "_ref" / "libmicrokv_ref.so"
HASH_LIB = Path(__file__).resolve().parent / "_build" / "libhashoracle.so"
