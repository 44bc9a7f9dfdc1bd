"""B200-native Winograd / Toom-Cook convolution with the reference toolkit's API.

Drop-in names of the reference package `toomcook` (its __init__.py:4-27), with
every compute function executed by libwino (generated sm_100a CUDA) -- plus the
layer-level entry point `conv2d_layer` that the reference lacks.
"""

from .engine import (
    ConvConfig,
    EvalLeaf,
    EvalNode,
    channel_reduce,
    conv_1d,
    conv_2d,
    conv_direct,
    direct_products,
    dot_with_order,
    hadamard_1d,
    hadamard_2d,
    huffman_order,
    linear_order,
    output_1d,
    output_2d,
    pairwise_sum,
    row_trees,
    tree_depth,
    tree_leaves,
)
from .exact import INFINITY, Point, Polynomial, parse_points, poly_product, to_nearest_float
from .exact_rational import check_exactness, conv_1d_exact, conv_2d_exact, conv_direct_exact
from .harness import DirectSpec, ErrorReport, compare_reports, measure_error, measure_variants, trial_inputs
from .layer import HostPipeline, LayerOp, conv2d_layer, direct_layer_f64, layer_error_stats, layer_op
from .pointsets import curated_points, curated_transform
from .tensor_io import convolve, load_tensor, save_tensor
from .transforms import (
    MultCount,
    TransformSet,
    build_modified,
    build_toom_cook,
    build_transforms,
    chebyshev_points,
    mult_count,
    read_transform_json,
    transform_set_from_json,
)

__version__ = "0.1.0"
