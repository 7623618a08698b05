"""B200-native memory-step engine for online video-inpainting transformers (arXiv 2403.16161).

The compute path is libvi.so (csrc/, sm_100a kernels behind the C-ABI in include/vi.h);
``vi`` is the ctypes binding.  Build with ``python -m paper_2403_16161_b200.build``.
"""
__all__ = ["vi"]
