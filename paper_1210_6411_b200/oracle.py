"""Drop-in name of the reference module ``lfsrcycles.oracle`` (oracle.py:141-283): the
exhaustive mini-cipher analysis, computed on the GPU by ``ground_truth`` /
``csrc/bruteforce.cu``.  (Not to be confused with the repository's top-level ``oracle/``
test checker, which the package never imports.)"""

from .ground_truth import CycleInfo, GroundTruth, brute_force_analysis  # noqa: F401

__all__ = ["GroundTruth", "CycleInfo", "brute_force_analysis"]
