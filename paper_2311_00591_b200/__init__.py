"""coop-b200: B200-native hot path of Coop (arXiv 2311.00591).

The product is libcoop.so (CUDA kernels for sm_100a behind the C ABI in include/coop.h);
`paper_2311_00591_b200.coop` is its thin ctypes binding.
"""
__all__ = ["coop"]
