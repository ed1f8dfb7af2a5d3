"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the PHub method (no chunking, no sums,
no optimizer).  It provides only:

* ``manifests``  -- layer-size recipes (key sizes, in fp32 elements) shaped like
  the paper's Table 5 networks (recipes in SURVEY.md App. A).
* ``generate``   -- a counter-based generator (splitmix64) with a numpy host
  implementation and a torch implementation that produce bit-identical fp32
  values, so either side can materialise any element of any stream on demand.
"""
from .manifests import MANIFESTS, manifest, config_names  # noqa: F401
from .generate import (  # noqa: F401
    grad_stream, weight_stream, momentum_stream, values_np, values_torch,
    dyadic_np,
)
