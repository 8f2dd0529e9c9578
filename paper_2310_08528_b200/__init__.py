"""B200-native 4D Gaussian Splatting forward path (arXiv 2310.08528).

Importing the package is cheap: the CUDA library (libfgs.so) is loaded lazily by
`paper_2310_08528_b200.fgs` the first time a binding is called.
"""
__all__ = ["inputs", "fgs"]
