"""B200-native sliding super-point path (arXiv 1805.09246).

The product is the CUDA library behind include/srlg.h (built in-tree to
paper_1805_09246_b200/_lib/libsrlg.so) and the C++ drop-in of the reference
estimator API (include/slidecard/). This Python package is the host-side
binding used by the tests and the benchmark.
"""
