"""paper_2507_04775_b200 -- B200-native hybrid key switching (FIDESlib hot path, arXiv 2507.04775).

The product is the C-ABI library ``libhks.so`` (``include/hks.h``) built from ``csrc/`` for
sm_100a; ``hks`` is its argument-marshalling binding.  Nothing here imports ``oracle/``.
"""
from . import hks
from .hks import (Context, HksError, automorph, bconv, keyswitch, ksk_inner_product, moddown, modup,
                  ntt_fwd, ntt_inv, relinearize, rotate_hoisted)

__all__ = ["hks", "Context", "HksError", "ntt_fwd", "ntt_inv", "bconv", "modup", "ksk_inner_product",
           "moddown", "keyswitch", "relinearize", "automorph", "rotate_hoisted"]
