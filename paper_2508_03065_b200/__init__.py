"""B200-native moving-source synthesis (arXiv 2508.03065 hot path).

Drop-in for the render path of the reference package `moverb`: the public
names mirror moverb (render, prepare_streams, synthesize, SynthesisConfig,
Room, MicPosition, Trajectory, FarrowFilter, enumerate_images, ...), and
every computation runs in hand-written sm_100a CUDA kernels behind the C ABI
in include/mvb.h (libmvb.so).  There is no CPU fallback: a compute entry
point called without the built library or without a GPU raises.
"""

from ._lib import MvbError
from .farrow import FarrowFilter, branch_filter, delay_stream, hann_sinc, split_delay
from .room import ImageSourceSpec, MicPosition, Room, attenuation, enumerate_images, image_count
from .synth import (BudgetError, DelayStreams, SynthesisConfig, cost_report,
                    full_rate_moving_oracle, high_order_distances, low_order_distances,
                    merge_streams, prepare_streams, render, render_jobs, synthesize)
from .trajectory import Trajectory, bandlimited_upsample, bandwidth_estimate, decimate
from .plan import RenderPlan
from .reference import (ComparisonReport, StaticRIR, compare, splice_baseline, static_render,
                        static_rir)

__version__ = "0.1.0"

__all__ = [
    "BudgetError", "ComparisonReport", "DelayStreams", "RenderPlan", "StaticRIR", "compare",
    "splice_baseline", "static_render", "static_rir", "FarrowFilter", "ImageSourceSpec", "MicPosition", "MvbError",
    "Room", "SynthesisConfig", "Trajectory", "bandlimited_upsample", "cost_report", "decimate",
    "enumerate_images", "full_rate_moving_oracle", "hann_sinc", "image_count", "prepare_streams",
    "render", "render_jobs", "split_delay", "synthesize", "__version__", "attenuation",
    "bandwidth_estimate", "branch_filter", "delay_stream", "high_order_distances",
    "low_order_distances", "merge_streams",
]
