"""B200-native kFkB pipeline executor (Ada-Grouper, arXiv 2303.01675).

The C++ planner/simulator/tuner and the sm_100a stage kernels live in
libptk.so (built by paper_2303_01675_b200/build.py); this package holds the
ctypes binding of its C ABI and the Python mirror of the pipetune API.
"""
__all__ = ["_lib"]
