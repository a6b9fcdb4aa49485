"""B200-native X-MeshGraphNet processor hot path (arXiv 2411.17164).

``xmgn``      -- ctypes binding of libxmgn.so (include/xmgn.h)
``processor`` -- per-GPU driver over partitions (marshalling only)
``build``     -- nvcc build of libxmgn.so for sm_100a
"""
