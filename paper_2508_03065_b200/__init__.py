"""B200-native moving-source synthesis (arXiv 2508.03065 hot path).

Drop-in for the reference package `moverb`'s render path: the public names
mirror moverb (render, prepare_streams, synthesize, SynthesisConfig, Room,
MicPosition, Trajectory, FarrowFilter, enumerate_images, ...), while every
computation runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/mvb.h (libmvb.so).  There is no CPU fallback: calling a compute
entry point without the built library or without a GPU raises.
"""

from .farrow import FarrowFilter, hann_sinc, split_delay

__version__ = "0.1.0"
