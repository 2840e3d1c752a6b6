"""B200-native (sm_100a) hot path of Sprout (arXiv 2403.12900): the
trace-driven directive-optimiser + carbon-accounting sweep behind the C ABI
in include/sprout.h (libsprout.so).  See DESIGN.md.

    from paper_2403_12900_b200 import sprout     # ctypes binding (needs libsprout.so)
    from paper_2403_12900_b200.runner import Sweep
"""
__all__ = ["sprout", "runner", "build"]
