"""B200-native collaborative texture filtering (arXiv 2506.17770) hot path.

The product is libctf.so (CUDA kernels for sm_100a behind the C ABI in
include/ctf.h); `ctf` is its thin Python binding and `dist` the multi-GPU
frame-sharding driver (NCCL only for the statistics gather).
"""
__all__ = ["ctf", "dist", "build"]
