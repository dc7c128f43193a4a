"""libpcpp: Partially Conditioned Patch Parallelism (arXiv 2412.02962) on B200.

The product is the C-ABI library libpcpp.so (include/pcpp.h, csrc/); ``pcpp`` is its ctypes
binding.  ``inputs`` holds the seeded synthetic input generators shared with the tests.
"""
