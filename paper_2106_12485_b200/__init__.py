"""B200-native hot path of the ZPIC em2d EM-PIC time step (arxiv 2106.12485).

The product is libzpic_b200.so (C ABI in include/zpic.h, sm_100a kernels in csrc/); this
package is its thin Python binding.  See DESIGN.md.
"""
from .zpic import *  # noqa: F401,F403
from .zpic import Simulation, ZpicError  # noqa: F401
