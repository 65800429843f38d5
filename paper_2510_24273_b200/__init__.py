"""B200-native SALS decode-attention hot path (arXiv 2510.24273).

The product is the C-ABI library ``libsals.so`` (include/sals.h); ``sals`` is
its ctypes binding, ``sharded`` the sequence-sharded orchestration over
torch.distributed, ``traffic`` the roofline byte accounting.
"""
