"""B200-native FP64 LGDM K/R assembly (arXiv 2301.06503) -- Python binding of liblgdm.so.

The product is the C-ABI library ``liblgdm.so`` (header ``include/lgdm.h``; sources in
``csrc/``).  This package is argument marshalling (``lgdm``), the slab partition helper
(``slabs``) and the build driver (``build``).
"""
from .lgdm import (BAR2, HEX8, KERNEL_AUTO, KERNEL_GENERAL, KERNEL_SWEEP, QUAD4, LGDMError, Material,
                   Mesh, load, material)

__all__ = ["BAR2", "QUAD4", "HEX8", "KERNEL_AUTO", "KERNEL_GENERAL", "KERNEL_SWEEP", "LGDMError",
           "Material", "Mesh", "load", "material"]
