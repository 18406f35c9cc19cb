"""B200-native GEM training step (arXiv 2509.25075): C-ABI CUDA library + thin binding.

Submodules: ``synth`` (seeded workload generator, no CUDA needed),
``binding`` (ctypes marshalling of libgem.so), ``gem`` (GemStep / DP wrapper).
The CUDA library is loaded lazily so that ``synth`` imports on CPU-only hosts.
"""
__all__ = ["synth", "binding", "gem"]
