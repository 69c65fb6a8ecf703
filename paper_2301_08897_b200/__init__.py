"""B200-native ScaDLES gradient-aggregation hot path (arXiv 2301.08897).

Modules
  comm      drop-in for ``streamsgd.comm`` (Top-k, gate, weighted aggregation on the GPU)
  nn        drop-in for the optimizer entries of ``streamsgd.nn`` (momentum SGD kernel)
  streams   the streaming sampler: contiguous-range StreamBuffer + device batch staging
  exchange  the per-GPU batched step (k workers) with the NCCL exchange protocol
  kernels   torch-tensor wrappers over the C-ABI (``include/scadles_b200.h``)
  dropin    install/uninstall into a reference ``streamsgd.engine`` module
  build     in-tree nvcc build of ``libscadles_b200.so`` for sm_100a
"""

__version__ = "0.1.0"
