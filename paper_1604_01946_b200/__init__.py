"""B200-native (sm_100a) multi-layer LSTM forward/backward behind the rnnwave API.

The compute path is librnnwave_sm100.so (hand-written tcgen05/TMA/TMEM kernels, see
DESIGN.md); this package is the host-side mirror of the reference interface.
"""
from .engine import (  # noqa: F401
    BackwardState, Engine, ForwardResult, ForwardTape, Gradients, LadderConfig, LayerParams,
    flop_count, gate_count, init_params, make_dy, make_input, pretranspose, random_matrix,
    splitmix_symmetric,
)
from . import param_io  # noqa: F401  (reference parameter files, param_io.hpp)
from .cells import gemm, pointwise_backward, pointwise_forward  # noqa: F401  (free functions)
