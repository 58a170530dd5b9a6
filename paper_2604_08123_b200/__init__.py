"""B200-native denoise step of LegoDiffusion's shared base model (arXiv 2604.08123).

The compute lives in libdit.so (include/dit.h, csrc/); this package is the thin
Python binding.  See DESIGN.md.
"""
from .dit import DiT, DitError, load_library  # noqa: F401
from .synthetic import SyntheticDiT  # noqa: F401
