"""B200-native executor for DiffusionPipe-style pipelined diffusion training.

Subpackages:
  pipefill   — planner API (stage partitioning, FIFO-1F1B simulation, bubble
               filling), restated from the reference `pipefill` package.
  ops        — torch wrappers over libdpipe.so (hand-written sm_100a kernels).
"""

__version__ = "0.1.0"
