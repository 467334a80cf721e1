"""B200-native depthwise-convolution training layer (arXiv 1803.09926 hot path).

The compute lives in ``libdwconv.so`` (C ABI: include/dwconv.h, CUDA for
sm_100a); this package is its thin Python binding.  See DESIGN.md.
"""
from ._lib import BF16, F32, NCHW, NHWC, PASS_BWD, PASS_BWD_DATA, PASS_BWD_FILTER, PASS_FWD, DwconvError  # noqa: F401
from .ops import (  # noqa: F401
    DepthwiseConv2d,
    DepthwiseConv2dFn,
    bwd,
    bwd_data,
    bwd_filter,
    desc_for,
    dwconv_bwd,
    dwconv_bwd_data,
    dwconv_bwd_filter,
    dwconv_bwd_filter_workspace_bytes,
    dwconv_bwd_workspace_bytes,
    dwconv_fwd,
    dwconv_plan,
    dwconv_set_variant_override,
    dwconv_workspace_init,
    fwd,
    make_desc,
    output_shape,
)
