"""B200-native DRCE tensor-parallel GPT layer stack (arXiv 2209.02341, EnergonAI sec 4.1.3 + 4.3).

The product is the C-ABI CUDA library ``lib/libenergon.so`` (sources in ``csrc/``, ABI in
``include/energon.h``); ``energon`` is its thin ctypes binding.
"""
from . import energon  # noqa: F401
from .build import build  # noqa: F401
