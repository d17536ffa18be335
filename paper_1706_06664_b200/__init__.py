"""B200-native ACE hot path (arXiv 1706.06664): SRP hashing, L x 2^K count
arrays, scoring and the mu-sigma / mu-alpha anomaly decisions on sm_100a.

Public API: paper_1706_06664_b200.ace (mirror of the reference C++ API).
Synthetic workloads: paper_1706_06664_b200.workloads.
"""
from . import ace  # noqa: F401
