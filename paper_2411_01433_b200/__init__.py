"""B200-native mixed-precision MoE expert layer (HOBBIT, arXiv 2411.01433).

The product is libhobbit.so (include/hobbit.h); this package is its thin
Python binding.  Importing a submodule that talks to the library raises if the
library is not built: there is no CPU fallback.
"""
__all__ = ["hobbit", "build"]
