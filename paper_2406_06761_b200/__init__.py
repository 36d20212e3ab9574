"""B200-native Wally server hot path (arXiv 2406.06761): per-cluster encrypted
dot products (coefficient-packed BFV ct x pt products, inverse NTT and RNS
modulus switch) as sm_100a CUDA kernels behind a C ABI (include/wally.h).

`paper_2406_06761_b200.wally` is the ctypes binding (imports libwally.so;
raises if it is missing -- there is no CPU fallback);
`paper_2406_06761_b200.build` compiles the library in-tree.
"""
