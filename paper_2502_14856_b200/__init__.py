"""B200-native FR-Spec drafting hot path (arxiv 2502.14856).

``paper_2502_14856_b200.api`` mirrors the reference's vocab / drafting / verification API;
all compute runs in the sm_100a library ``libfrspec_cuda.so`` (include/frspec_cuda.h).
"""
from ._lib import LIB_PATH, lib  # noqa: F401

__version__ = "0.1.0"
