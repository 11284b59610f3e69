"""B200-native MR-SP (arXiv 2507.07966): the encode+prefill hot path.

The product is libmrsp_b200.so (csrc/, C-ABI in include/mrsp_c.h); this
package is the host-side mirror of the reference's lvrl::mrsp interface.
"""
__all__ = ["mrsp"]
