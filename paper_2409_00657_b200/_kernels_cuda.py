"""gnnsim backend module: the reference operator layer on the B200 library.

``gnnsim.kernels`` (kernels.py:14-34) picks ``_kernels_nb`` or ``_kernels_np``
from ``GNNSIM_KERNELS`` and re-exports four functions; this module has the
same four with the same signatures and results, computed by libhopgnn.so
(sample_frontier, feature_rows, pick_k_smallest, sbm_edges).  A gnnsim
checkout would import it for ``GNNSIM_KERNELS=cuda``;
``install(gnnsim.kernels)`` rebinds an already-imported reference to it
(what tests/test_gnnsim_dropin_gpu.py does to run gnnsim's own tests and
trainer on the GPU kernels).  No CPU fallback: every call runs on the GPU.
"""
from __future__ import annotations

from .kernels import feature_rows, pick_k_smallest, probability_threshold, sample_frontier, sbm_edges

BACKEND = "cuda"

__all__ = ["sbm_edges", "sample_frontier", "pick_k_smallest", "feature_rows", "BACKEND",
           "install"]


def install(kernels_module) -> None:
    """Point a reference ``gnnsim.kernels`` module at this backend (its callers
    read the functions through the module attribute: sampler.py:97, 118,
    featstore.py:167, graph.py:207)."""
    kernels_module.sample_frontier = sample_frontier
    kernels_module.feature_rows = feature_rows
    kernels_module.pick_k_smallest = pick_k_smallest
    kernels_module.sbm_edges = sbm_edges
    kernels_module.BACKEND = BACKEND
