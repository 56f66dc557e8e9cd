"""B200-native matrix-free sum-factorisation Laplace operator (deal.II, arXiv 1910.13247).

The product is libmf_b200.so (C ABI in include/mf.h, CUDA sm_100a kernels);
this package is its thin ctypes binding.  See DESIGN.md."""
from .mf import HangingNodeOperator, HexOperator, MFError, Multigrid, Operator, hex_number_dofs, load  # noqa: F401

__all__ = ["Operator", "Multigrid", "HangingNodeOperator", "HexOperator", "hex_number_dofs", "MFError", "load"]
