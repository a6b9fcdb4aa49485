"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no MLP, LayerNorm,
aggregation or gradient code).  It produces only what the processor consumes:

* ``geometry``  -- point clouds on a unit sphere (CFG1) and on a closed
  car-proxy superellipsoid (CFG2-5), nested across levels
  (Sec. III-C).
* ``graph``     -- per-level kNN (k=6), symmetrised, union over
  levels, CSR by destination.
* ``partition`` -- recursive coordinate bisection (stand-in for METIS,
  PAPER.md:172) and BFS halo rings of depth L.
* ``tensors``   -- counter-based hash values for parameters, h0, e0 and the
  upstream gradient g, rounded to BF16-representable floats.
* ``configs``   -- the five BASELINE.json configurations and a disk cache.
"""
from . import geometry, graph, partition, tensors, configs  # noqa: F401
