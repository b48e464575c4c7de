"""B200-native (sm_100a) hot path of the convex-hull preconditioner of
arXiv 1505.00914: Algorithm 1's per-column min/max reduction, the
skip-invalid compaction into the Lemma-1 chain, and the exact hull, behind
the reference's chp::reducer / chp::hulls interface.

Layers:
  include/chp_b200.h            C ABI (the drop-in boundary), libchp_b200.so
  include/chp/*.hpp             C++ drop-in of the reference headers
  paper_1505_00914_b200.device  torch-tensor API (device-resident buffers)
  paper_1505_00914_b200.reducer / .hulls / .kernels   Python mirror of the
                                reference entry points (host buffers)
"""
from ._lib import ChpError, load  # noqa: F401  (fails loudly without the .so)

__all__ = ["ChpError", "load"]
