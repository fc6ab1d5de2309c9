"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the SiDP method (no norms, no matmuls, no
schedules).  It only defines

* the workload shapes (``configs``): the BASELINE.json configurations, as
  model dimensions and batch/context recipes;
* the counter-based generator (``gen``): every synthetic value is a pure
  function of (seed, tensor id, layer, logical index), so the CUDA init kernel
  (K12, ``paper_2605_28095_b200/csrc/kernels/init.cu``) re-implements the same
  generator on device and both sides see bit-identical inputs without sharing
  code.
"""
from .configs import ModelDims, MODELS, get_model, Workload, WORKLOADS  # noqa: F401
from . import gen  # noqa: F401
