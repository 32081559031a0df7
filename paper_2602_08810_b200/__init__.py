"""lrx-b200: B200-native (sm_100a) drop-in for the hot path of `linrec`
(arxiv 2602.08810): the diagonal linear-recurrence scan, forward and backward,
for S4D / S5 / LRU / S6 / RG-LRU, behind the reference's layer and operator
API.  Kernels live in liblrx.so (include/lrx.h); this package is the host-side
mirror of the reference interface.  There is no CPU fallback.
"""
from .numerics import (REAL_DTYPES, ComplexPair, Rng, ShapeError, alloc, allocation_count, as_tensor, complex_dtype,
                       complex_exp, real_dtype, sigmoid, softplus)
from .discretize import (NonMonotoneTimestamps, SingularBilinear, deltas_from_timestamps, discretize,
                         discretize_bilinear, discretize_dirac, discretize_zoh, scheme_factors)
from .scan import (MIN_CHUNK_LEN, StepState, combine, identity_element, init_step_state, plan_chunks, scan_parallel,
                   scan_sequential, step)
from .autograd import (FiniteDiffReport, GradBundle, RecomputeTape, Tape, TapeConsumed, check_layer_gradients,
                       finite_diff_check, layer_backward, scan_backward, scan_forward, scheme_partials)
from .layers import (LAYER_KINDS, LRU, RGLRU, S4D, S5, S6, SCHEMES_BY_KIND, LayerConfig, LayerStepState, StepGraph,
                     LinearRecurrence, UnknownLayer, init_layer, layer_step, lti_forward, ltv_forward, make_layer)

__version__ = "0.1.0"
